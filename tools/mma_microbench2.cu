// mma_microbench2.cu -- straight-line tcgen05.mma issue (compile-time shapes, no per-MMA address
// arithmetic) to separate instruction-issue cost from tensor-core execution time on sm_100a.
#include <cstdio>
#include <cstdint>
#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"
using namespace csenc;

template <int MM, int N, bool TS, int NMMA>
__global__ void bench(long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    const uint32_t bar = sb, slot = sb + 8;
    const uint32_t a_s = sb + 1024, b_s = a_s + 32768;
    for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a_s + 4 * i), "r"(0x3C003C00u));
    if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbarrier_init(); }
    if (threadIdx.x < 32) { ptx::tmem_alloc(slot, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    uint32_t tb;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tb) : "r"(slot));
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
        const uint64_t b0 = ptx::smem_desc_noswizzle(b_s, N * 16, 128);
        const uint64_t a0 = ptx::smem_desc_noswizzle(a_s, MM * 16, 128);
        long long t0 = clock64();
#pragma unroll
        for (int i = 0; i < NMMA; ++i) {
            const uint32_t ks = i & 7;
            if (TS) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             :: "r"(tb + 256), "r"(tb + ks * 8), "l"(b0 + ks * (2 * N * 16 >> 4)), "r"(idesc), "r"(i > 0 ? 1u : 0u) : "memory");
            } else {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             :: "r"(tb + 256), "l"(a0 + ks * (2 * MM * 16 >> 4)), "l"(b0 + ks * (2 * N * 16 >> 4)), "r"(idesc), "r"(i > 0 ? 1u : 0u) : "memory");
            }
        }
        long long t1 = clock64();
        ptx::tc_commit(bar);
        ptx::mbar_wait(bar, 0);
        out[0] = t1 - t0;
        out[1] = clock64() - t0;
    }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tb, 512);
}

template <int MM, int N, bool TS>
void run(long long* d) {
    constexpr int NM = 64;
    const int smem = 1024 + 32768 + 65536 + 1024;
    cudaFuncSetAttribute(bench<MM, N, TS, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<MM, N, TS, NM><<<1, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("M=%3d N=%3d %s  issue %7.1f  total %7.1f cyc/mma  %s\n", MM, N, TS ? "TS" : "SS", (double)h[0] / NM,
           (double)h[1] / NM, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    run<128, 16, true>(d); run<128, 64, true>(d); run<128, 128, true>(d); run<128, 256, true>(d);
    run<128, 16, false>(d); run<128, 64, false>(d); run<128, 128, false>(d); run<128, 256, false>(d);
    run<64, 16, false>(d); run<64, 64, false>(d); run<64, 128, false>(d); run<64, 256, false>(d);
    run<64, 16, true>(d); run<64, 64, true>(d);
    return 0;
}
