// mma_microbench.cu -- measure tcgen05.mma.kind::f16 throughput on sm_100a for the shapes the
// encoder uses: A from TMEM (TS) vs A from SMEM (SS), N in {16..256}, 1 vs several independent
// accumulators.  One CTA, one issuing thread, clock64 from first issue to commit completion.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_microbench tools/mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"

using namespace csenc;

__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
    return pred != 0;
}

// variant 0: lane 0 only, generic loop (as in the kernel v2)
// variant 1: whole warp runs the loop (uniform values), MMA under elect.sync
// variant 2: whole warp, descriptor increments, unrolled by 8
__global__ void bench(int mode, int N, int chains, int iters, int variant, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    const uint32_t bar = sb, slot = sb + 8;
    const uint32_t a_s = sb + 1024;
    const uint32_t b_s = a_s + 32768;
    for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a_s + 4 * i), "r"(0x3C003C00u));
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbarrier_init();
    }
    if (threadIdx.x < 32) {
        ptx::tmem_alloc(slot, 512);
        ptx::tmem_relinquish();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    uint32_t tbase;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(slot));
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a_lbo = 128 * 16, b_lbo = (uint32_t)N * 16;
    const uint32_t a_tm = tbase;
    const uint32_t d_tm = tbase + 256;
    if (variant == 0) {
        if (threadIdx.x == 0) {
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const int ks = i & 7;
                const uint32_t d = d_tm + (uint32_t)((i % chains) * N);
                const uint64_t bdesc = ptx::smem_desc_noswizzle(b_s + ks * 2 * b_lbo, b_lbo, 128);
                if (mode == 0) {
                    ptx::mma_f16_ts(d, a_tm + ks * 8, bdesc, idesc, i >= chains ? 1u : 0u);
                } else {
                    const uint64_t adesc = ptx::smem_desc_noswizzle(a_s + ks * 2 * a_lbo, a_lbo, 128);
                    mma_f16_ss(d, adesc, bdesc, idesc, i >= chains ? 1u : 0u);
                }
            }
            long long t1 = clock64();
            ptx::tc_commit(bar);
            ptx::mbar_wait(bar, 0);
            out[0] = t1 - t0;
            out[1] = clock64() - t0;
        }
    } else if (threadIdx.x < 32) {
        long long t0 = clock64();
        const uint64_t b0 = ptx::smem_desc_noswizzle(b_s, b_lbo, 128);
        const uint64_t a0 = ptx::smem_desc_noswizzle(a_s, a_lbo, 128);
        const uint64_t bstep = (2 * b_lbo) >> 4, astep = (2 * a_lbo) >> 4;
        if (variant == 1) {
            for (int i = 0; i < iters; ++i) {
                const int ks = i & 7;
                const uint32_t d = d_tm + (uint32_t)((i % chains) * N);
                const uint64_t bdesc = b0 + ks * bstep;
                if (elect_one()) {
                    if (mode == 0) ptx::mma_f16_ts(d, a_tm + ks * 8, bdesc, idesc, i >= chains ? 1u : 0u);
                    else mma_f16_ss(d, a0 + ks * astep, bdesc, idesc, i >= chains ? 1u : 0u);
                }
                __syncwarp();
            }
        } else {
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint32_t d = d_tm + (uint32_t)((ks & (chains - 1)) * N);
                    if (elect_one()) {
                        if (mode == 0) ptx::mma_f16_ts(d, a_tm + ks * 8, b0 + ks * bstep, idesc, (i + ks) >= chains ? 1u : 0u);
                        else mma_f16_ss(d, a0 + ks * astep, b0 + ks * bstep, idesc, (i + ks) >= chains ? 1u : 0u);
                    }
                    __syncwarp();
                }
            }
        }
        long long t1 = clock64();
        if (elect_one()) ptx::tc_commit(bar);
        __syncwarp();
        ptx::mbar_wait(bar, 0);
        if (threadIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = clock64() - t0;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    const int smem = 1024 + 32768 + 65536 + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 1024;
    printf("var mode N chains  issue_cyc/mma  total_cyc/mma  ideal(N/2)\n");
    for (int variant = 0; variant < 3; ++variant)
    for (int mode = 0; mode < 2; ++mode)
        for (int N : {16, 64, 128, 256})
            for (int chains : {1, 4}) {
                if (chains * N > 256) continue;
                bench<<<1, 128, smem>>>(mode, N, chains, iters, variant, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[2];
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                printf("v%d %s %3d %d  %8.1f  %8.1f  %5d\n", variant, mode ? "SS" : "TS", N, chains, (double)h[0] / iters,
                       (double)h[1] / iters, N / 2);
            }
    return 0;
}
