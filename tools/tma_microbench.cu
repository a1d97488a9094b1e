// tma_microbench.cu -- streaming HBM -> SMEM throughput of the TMA engine on sm_100a:
// 1-D cp.async.bulk vs 2-D tensor-map tile loads, copy size, ring depth, L2 cache hint.
// grid = #SMs, one producer thread fills a ring of S slots, a consumer warp releases each slot as
// soon as it lands.  Reports GB/s over a 512 MiB buffer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_microbench tools/tma_microbench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1311_1419_b200/csrc/ptx_sm100.cuh"
using namespace csenc;

struct Args {
    const uint8_t* src;
    size_t bytes;
    int mode;        // 0 bulk, 1 bulk+hint, 2 tensor 2D (rows of 256 B), 3 bulk split in `parts`
    uint32_t slot;   // bytes per slot
    int stages;
    int parts;       // mode 3: parts per slot; mode 4: producer warps
    long long* issue_cyc;
};

__global__ void __launch_bounds__(256, 1) kern(const __grid_constant__ CUtensorMap tm, const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = (ptx::smem_addr(smem) + 1023u) & ~1023u;
    const uint32_t full = sb, empty = sb + 256, data = sb + 1024;  // <= 32 slots
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.stages; ++i) {
            ptx::mbar_init(full + 8 * i, 1);
            ptx::mbar_init(empty + 8 * i, 1);
        }
        ptx::fence_mbarrier_init();
    }
    __syncthreads();
    const size_t n_slots_total = a.bytes / a.slot;
    if (a.mode == 4) {
        // P producer warps (0..P-1, lane 0) and P consumer lanes (warp P+q, lane 0); producer q owns
        // slots [q*stages, (q+1)*stages) and items i = blockIdx.x + (j*P + q)*gridDim.x
        const int P = a.parts;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0 && w < 2 * P) {
            const int q = w % P;
            const bool prod = w < P;
            int st = 0;
            uint32_t ph = 0;
            long long cyc = 0;
            for (size_t i = blockIdx.x + (size_t)q * gridDim.x; i < n_slots_total; i += (size_t)P * gridDim.x) {
                const int slot = q * a.stages + st;
                if (prod) {
                    ptx::mbar_wait(empty + 8 * slot, ph ^ 1u);
                    ptx::mbar_arrive_expect_tx(full + 8 * slot, a.slot);
                    long long c0 = clock64();
                    ptx::bulk_load(data + (uint32_t)slot * a.slot, a.src + i * a.slot, a.slot, full + 8 * slot);
                    cyc += clock64() - c0;
                } else {
                    ptx::mbar_wait(full + 8 * slot, ph);
                    ptx::mbar_arrive(empty + 8 * slot);
                }
                if (++st == a.stages) { st = 0; ph ^= 1u; }
            }
            if (prod && blockIdx.x == 0 && q == 0) a.issue_cyc[0] = cyc;
        }
        __syncthreads();
        return;
    }
    if (threadIdx.x == 0) {
        long long cyc = 0;
        uint64_t pol = ptx::policy_evict_first();
        int st = 0;
        uint32_t ph = 0;
        for (size_t i = blockIdx.x; i < n_slots_total; i += gridDim.x) {
            ptx::mbar_wait(empty + 8 * st, ph ^ 1u);
            ptx::mbar_arrive_expect_tx(full + 8 * st, a.slot);
            const uint32_t dst = data + (uint32_t)st * a.slot;
            const uint8_t* src = a.src + i * a.slot;
            long long c0 = clock64();
            if (a.mode == 0) {
                ptx::bulk_load(dst, src, a.slot, full + 8 * st);
            } else if (a.mode == 5) {
                ptx::prefetch_l2(src, a.slot);
                ptx::bulk_load(dst, src, a.slot, full + 8 * st);
            } else if (a.mode == 1) {
                ptx::bulk_load_hint(dst, src, a.slot, full + 8 * st, pol);
            } else if (a.mode == 2) {
                // rows of 256 B: box {256, rows} with rows = slot/256 (<= 256)
                const int row0 = (int)(i * (a.slot / 256));
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                    ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(row0), "r"(full + 8 * st) : "memory");
            } else {
                const uint32_t part = a.slot / a.parts;
                for (int q = 0; q < a.parts; ++q) ptx::bulk_load(dst + q * part, src + q * part, part, full + 8 * st);
            }
            cyc += clock64() - c0;
            if (++st == a.stages) { st = 0; ph ^= 1u; }
        }
        if (blockIdx.x == 0) a.issue_cyc[0] = cyc;
    } else if (threadIdx.x == 32) {
        int st = 0;
        uint32_t ph = 0;
        for (size_t i = blockIdx.x; i < n_slots_total; i += gridDim.x) {
            ptx::mbar_wait(full + 8 * st, ph);
            ptx::mbar_arrive(empty + 8 * st);
            if (++st == a.stages) { st = 0; ph ^= 1u; }
        }
    }
    __syncthreads();
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t bytes = 512ull << 20;
    uint8_t* buf;
    cudaMalloc(&buf, bytes + (1 << 20));
    cudaMemset(buf, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    PFN_encodeTiled enc = (PFN_encodeTiled)fp;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long long* issue;
    cudaMalloc(&issue, 8);
    printf("mode slotKB stages parts  GB/s  issue_cyc/copy(cta0)\n");
    struct C { int mode, kb, stages, parts; };
    C cs[] = {{0, 4, 8, 1}, {0, 8, 8, 1}, {0, 16, 8, 1}, {0, 32, 6, 1}, {5, 16, 8, 1}, {5, 32, 6, 1},
              {4, 8, 4, 2}, {4, 8, 2, 4}, {4, 16, 4, 2}, {4, 16, 2, 4}, {4, 4, 4, 4}, {4, 8, 3, 4}};
    for (auto c : cs) {
        Args a{buf, bytes, c.mode, (uint32_t)c.kb * 1024u, c.stages, c.parts, issue};
        CUtensorMap tm;
        cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 256)};
        cuuint64_t str[1] = {256};
        cuuint32_t box[2] = {256, (cuuint32_t)(a.slot / 256 > 256 ? 256 : a.slot / 256)};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (c.mode == 2 && a.slot / 256 > 256) continue;
        const int slots = (c.mode == 4) ? c.stages * c.parts : c.stages;
        int smem = 1024 + a.slot * slots + 1024;
        if (smem > 227 * 1024) continue;
        if (slots > 32) continue;
        for (int rep = 0; rep < 2; ++rep) kern<<<sms, 64, smem>>>(tm, a);
        cudaEventRecord(e0);
        const int R = 5;
        for (int rep = 0; rep < R; ++rep) kern<<<sms, 64, smem>>>(tm, a);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long ic = 0;
        cudaMemcpy(&ic, issue, 8, cudaMemcpyDeviceToHost);
        const double copies = (double)(bytes / a.slot) / sms / (c.mode == 4 ? c.parts : 1);
        printf("%d %3d %2d %d  %8.1f  %8.1f %s\n", c.mode, c.kb, c.stages, c.parts, R * bytes / (ms * 1e-3) / 1e9,
               ic / copies, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
