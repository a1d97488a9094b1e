// launch_overhead.cu -- what a K1-shaped launch costs before any work: 148 CTAs x 480 threads with (a) no
// dynamic SMEM, (b) 220 KB dynamic SMEM, (c) + TMEM alloc/dealloc of 512 columns, (d) + griddepcontrol
// (launched with programmatic stream serialization).  100 back-to-back launches between one event pair
// and, separately, one event pair per launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/launch_overhead tools/launch_overhead.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"
using namespace csenc;

template <int MODE>
__global__ void __launch_bounds__(480, 1) k(int* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    if (MODE >= 2) {
        const int warp = threadIdx.x >> 5;
        if (warp == 13) { ptx::tmem_alloc(sb, 512); ptx::tmem_relinquish(); }
        ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
        if (MODE >= 3) { ptx::grid_dep_launch(); ptx::grid_dep_wait(); }
        uint32_t tb;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tb) : "r"(sb));
        __syncthreads();
        if (warp == 13) ptx::tmem_dealloc(tb, 512);
    }
    if (sink == (int*)1) sink[0] = 1;
}

template <int MODE>
void run(const char* name, int smem, bool pdl) {
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(480); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    int* sink = nullptr;
    for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, k<MODE>, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int R = 200;
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) cudaLaunchKernelEx(&cfg, k<MODE>, sink);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    float tot = 0;
    for (int i = 0; i < R; ++i) {
        cudaEventRecord(e0); cudaLaunchKernelEx(&cfg, k<MODE>, sink); cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float m; cudaEventElapsedTime(&m, e0, e1); tot += m;
    }
    // events queued ahead (not synchronised per launch), as bench.py does
    cudaEvent_t ev[2 * 50];
    for (auto& e : ev) cudaEventCreate(&e);
    for (int i = 0; i < 50; ++i) { cudaEventRecord(ev[2 * i]); cudaLaunchKernelEx(&cfg, k<MODE>, sink); cudaEventRecord(ev[2 * i + 1]); }
    cudaDeviceSynchronize();
    float tq = 0;
    for (int i = 0; i < 50; ++i) { float m; cudaEventElapsedTime(&m, ev[2 * i], ev[2 * i + 1]); tq += m; }
    printf("%-44s back-to-back %6.2f us/launch | event pair, synced %6.2f us | event pair, queued %6.2f us  %s\n", name,
           ms * 1e3 / R, tot * 1e3 / R, tq * 1e3 / 50, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<0>("empty, no dynamic smem", 0, false);
    run<1>("empty, 220 KB dynamic smem", 220 * 1024, false);
    run<2>("220 KB + TMEM alloc/dealloc", 220 * 1024, false);
    run<3>("220 KB + TMEM + griddepcontrol, PDL launch", 220 * 1024, true);
    run<2>("220 KB + TMEM, PDL attr but no griddepcontrol", 220 * 1024, true);
    return 0;
}
