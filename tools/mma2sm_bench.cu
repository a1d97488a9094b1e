// mma2sm_bench.cu -- throughput of tcgen05.mma kind::f16 SS with SW128 K-major operands: one SM
// (cta_group::1, M = 128) vs a CTA pair (cta_group::2, M = 256, issued by the leader), N = 128 / 256.
// Cycles per MMA from the first issue to the commit's completion, 2048 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma2sm_bench tools/mma2sm_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"

using namespace csenc;

__global__ void __cluster_dims__(2, 1, 1) bench(int two_sm, int N, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    const uint32_t bar = sb, slot = sb + 8;
    const uint32_t a_s = sb + 1024;            // 128 rows x 128 B (SW128)
    const uint32_t b_s = a_s + 16384;          // up to 256 rows x 128 B
    const int rank = (int)ptx::cluster_ctarank();
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a_s + 4 * i), "r"(0x3C003C00u));
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        if (two_sm) {
            ptx::tmem_alloc_2sm(slot, 512);
            ptx::tmem_relinquish_2sm();
        } else {
            ptx::tmem_alloc(slot, 512);
            ptx::tmem_relinquish();
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    uint32_t tbase;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(slot));
    const int Mm = two_sm ? 256 : 128;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(Mm >> 4) << 24);
    const uint64_t ad = ptx::smem_desc_swizzled(a_s, 128u, 1024u);
    const uint64_t bd = ptx::smem_desc_swizzled(b_s, 128u, 1024u);
    const bool issuer = two_sm ? rank == 0 : true;
    if (threadIdx.x == 0 && issuer) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int ks = i & 3;
            const uint32_t d = tbase + (uint32_t)((i >> 2) & 1) * 256u;
            if (two_sm)
                ptx::mma_f16_ss_2sm(d, ad + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc, ks ? 1u : 0u);
            else
                ptx::mma_f16_ss(d, ad + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc, ks ? 1u : 0u);
        }
        if (two_sm)
            ptx::tc_commit_2sm_mc(bar, 0x3);
        else
            ptx::tc_commit(bar);
        ptx::mbar_wait(bar, 0);
        if (rank == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
    }
    if (two_sm && rank == 1 && threadIdx.x == 0) ptx::mbar_wait(bar, 0);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) {
        if (two_sm)
            ptx::tmem_dealloc_2sm(tbase, 512);
        else
            ptx::tmem_dealloc(tbase, 512);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    const int smem = 1024 + 16384 + 32768 + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2048;
    printf("mode     N   cyc/MMA   flop/cyc/SM\n");
    for (int two : {0, 1})
        for (int N : {128, 256}) {
            bench<<<2, 128, smem>>>(two, N, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double cyc = (double)h / iters;
            const double flop_per_sm = 2.0 * 128 * N * 16;   // per SM per MMA (2-SM: 128 rows each)
            printf("%s %4d  %8.1f  %10.0f\n", two ? "2SM M256" : "1SM M128", N, cyc, flop_per_sm / cyc);
        }
    return 0;
}
