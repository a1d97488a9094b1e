// mma_microbench3.cu -- does a second issuing warp raise the tcgen05.mma rate for small-N TS MMAs?
// NW warps (1 or 2) each issue NMMA straight-line kind::f16 TS MMAs (M = 128, N = 64, K = 16) into their own
// accumulator; time from the first issue to the completion of all of them (per-warp commit -> one mbarrier).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_microbench3 tools/mma_microbench3.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"
using namespace csenc;

template <int N, int NMMA, bool TS>
__global__ void bench(int nw, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    const uint32_t bar = sb, slot = sb + 8;
    const uint32_t a_s = sb + 1024, b_s = a_s + 32768;
    for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a_s + 4 * i), "r"(0x3C003C00u));
    if (threadIdx.x == 0) { ptx::mbar_init(bar, nw); ptx::fence_mbarrier_init(); }
    if (threadIdx.x < 32) { ptx::tmem_alloc(slot, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    uint32_t tb;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tb) : "r"(slot));
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && w < nw) {
        constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t b0 = ptx::smem_desc_noswizzle(b_s, N * 16, 128);
        const uint64_t a0 = ptx::smem_desc_noswizzle(a_s, 128 * 16, 128);
        const uint32_t d = tb + 256 + (uint32_t)w * N;
        long long t0 = clock64();
#pragma unroll
        for (int i = 0; i < NMMA; ++i) {
            const uint32_t ks = i & 7;
            if (TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             :: "r"(d), "r"(tb + ks * 8 + w * 64), "l"(b0 + ks * (2 * N * 16 >> 4)), "r"(idesc), "r"(i > 0 ? 1u : 0u) : "memory");
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             :: "r"(d), "l"(a0 + ks * (2 * 128 * 16 >> 4)), "l"(b0 + ks * (2 * N * 16 >> 4)), "r"(idesc), "r"(i > 0 ? 1u : 0u) : "memory");
        }
        long long t1 = clock64();
        ptx::tc_commit(bar);
        ptx::mbar_wait(bar, 0);
        out[2 * w] = t1 - t0;
        out[2 * w + 1] = clock64() - t0;
    }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tb, 512);
}

template <int N, bool TS>
void run(long long* d, int nw) {
    constexpr int NM = 64;
    const int smem = 1024 + 32768 + 65536 + 1024;
    cudaFuncSetAttribute(bench<N, NM, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(d, 0, 64);
    bench<N, NM, TS><<<1, 128, smem>>>(nw, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("N=%3d %s warps=%d  warp0: issue %6.1f total %6.1f | warp1: issue %6.1f total %6.1f cyc per (own) mma  %s\n", N,
           TS ? "TS" : "SS", nw, (double)h[0] / NM, (double)h[1] / NM, (double)h[2] / NM, (double)h[3] / NM,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    for (int nw = 1; nw <= 2; ++nw) {
        run<16, true>(d, nw); run<64, true>(d, nw); run<128, true>(d, nw); run<256, true>(d, nw);
        run<64, false>(d, nw); run<128, false>(d, nw);
    }
    return 0;
}
