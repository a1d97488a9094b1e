// cs_adjoint_kernel.cuh -- K3: block back-projection x0 = Phi^T y.
//
// SPEC.md:145-153 adjoint(A, v) = A^T v; the decoder's start point x = A^T y.  With
// the block-based Phi of the north star (BASELINE.json:5) it is, for every block b of every frame,
// x_b = Phi^T y_b (N = B*B outputs from M measurements), written back into the frame layout
// x[frame][H][W] (the inverse of the a2 tiling; pixels of padded blocks outside the frame dropped).
//
// A dense contraction, so it runs on the tensor cores: D[128 blocks x Nc pixels] (+)=
// Y[128 blocks x K] * Phi^T[K x Nc], tcgen05.mma kind::tf32, fp32 accumulation in TMEM.  Phi is
// fp16, exactly representable in tf32; y is fp32, split y = hi + lo with hi = y with the low 13
// mantissa bits cleared (exactly tf32) and lo = y - hi (exact), two MMAs per K step, so the result
// carries ~22 bits of y (the single-tf32 product would carry 11).
//
// Roles (10 warps):
//   warps 0..3  converters: split each landed Y K-chunk in place (hi) and into the lo buffer,
//               fence.proxy.async, arrive.
//   warps 4..7  epilogue: tcgen05.ld of one pixel row (B columns) per block (lane = block), a 32-row
//               swizzled SMEM stage, coalesced st.global.v4 of the warp's 32*B contiguous floats of
//               that frame row.
//   warp 8      producer: per stage one TMA 2-D box of Y (128 rows x Kc floats, hardware swizzle
//               32/64/128 B = the UMMA K-major swizzled layout) + one bulk copy of the Phi^T chunk.
//   warp 9      MMA issuer + TMEM allocator.
// Work unit = (frame, block row, part of the row) = up to 128 consecutive blocks; item = one chunk
// of Nc <= 256 output columns (B = 32: 4 chunks of 8 pixel rows); stage = one K chunk of an item.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "ptx_sm100.cuh"

namespace csenc {
namespace adj {

constexpr int kConvWarps = 4;
constexpr int kEpiWarp0 = 4;
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kThreads = 10 * 32;
constexpr int kMaxStages = 8;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOffEpi = 1024;                 // 4 warps x 4 KB epilogue stage
constexpr uint32_t kOffStage = 1024 + 4 * 4096;    // stages (1024-aligned)

struct AParams {
    CUtensorMap ymap;         // y as 2-D [rows = n_frames * nblk][M] fp32, box [128][Kc], swizzle Kc*4 B
    const uint8_t* phiT;      // device: [n_nc][n_kc] chunks of chunk_bytes, no-swizzle K-major tf32
    float* x;                 // device: [n_frames][H][W]
    int W, H, M, nbx, nby, nblk;
    int parts, L;             // tiles per block row, blocks per tile (<= 128)
    // flat != 0 (nbx % 32 == 0): a tile is 128 consecutive blocks of the frame's raster order, across
    // block rows (each epilogue warp's 32 blocks still lie in one block row); tiles_pf per frame
    int flat, tiles_pf;
    // programmatic dependent launch (as K1): 0 = the whole kernel waits for the stream's previous kernel before
    // touching global memory; 1 (cs_encoder_set_stable_inputs: y and Phi^T not written by that kernel) = only
    // the epilogue warps wait, before their first store
    int pdl_early;
    int Kc, n_kc;             // K per stage (8/16/32), K chunks
    int Nc, n_nc;             // output columns per item (<= 256), items per tile
    uint32_t a_bytes, chunk_bytes, stage_bytes;
    int n_stages;
    int n_units;
    uint32_t idesc, b_lbo, a_sbo;
    long long x_floats;
    uint32_t smem_bytes;      // dynamic SMEM from the aligned base (CSENC_CHECKS)
};

// Staged store of one pixel row of a warp's 32 blocks: lane r holds its block's 4*CPR floats (w);
// the warp's output is 32 * 4*CPR contiguous floats at dst, of which the first `valid` are stored.
template <int CPR>
__device__ __forceinline__ void row_store(const uint32_t* w, uint32_t tile, uint32_t lane, float* dst, int valid) {
    constexpr uint32_t PITCH = CPR * 16;
#pragma unroll
    for (int q = 0; q < CPR; ++q) {
        const int f = (CPR == 8) ? (int)(lane & 7u) : (CPR == 4 ? (int)((lane >> 1) & 3u) : (int)((lane >> 2) & 1u));
        ptx::sts128(tile + lane * PITCH + (uint32_t)(q ^ f) * 16u, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < CPR; ++it) {
        const uint32_t o = (uint32_t)it * 512u + lane * 16u;   // byte offset in the warp's contiguous output
        const int r = (int)(o / PITCH), c = (int)((o % PITCH) / 16u);
        const int f = (CPR == 8) ? (r & 7) : (CPR == 4 ? ((r >> 1) & 3) : ((r >> 2) & 1));
        uint4 t = ptx::lds128(tile + (uint32_t)r * PITCH + (uint32_t)(c ^ f) * 16u);
        if ((int)(o / 4u) < valid) ptx::stg128(dst + o / 4u, t.x, t.y, t.z, t.w);
    }
    __syncwarp();
}

template <int B>
__global__ void __launch_bounds__(kThreads, 1) cs_adjoint_kernel(const __grid_constant__ AParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31u;

    const uint32_t bar_full = sbase;                       // [kMaxStages]
    const uint32_t bar_conv = sbase + 8 * kMaxStages;      // [kMaxStages]
    const uint32_t bar_empty = sbase + 16 * kMaxStages;    // [kMaxStages]
    const uint32_t bar_dfull = sbase + 24 * kMaxStages;    // [2]
    const uint32_t bar_dempty = bar_dfull + 16;            // [2]
    const uint32_t tmem_slot = bar_dempty + 16;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(bar_full + 8 * i, 1);
            ptx::mbar_init(bar_conv + 8 * i, kConvWarps);
            ptx::mbar_init(bar_empty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_dfull + 8 * i, 1);
            ptx::mbar_init(bar_dempty + 8 * i, 4);
        }
        ptx::fence_mbarrier_init();
    }
    if (warp == kMmaWarp) {
        ptx::tmem_alloc(tmem_slot, kTmemCols);
        ptx::tmem_relinquish();
    }
    if (warp == kProducerWarp && lane == 0) ptx::prefetch_tmap(&p.ymap);
    CS_CHECK(kOffStage + (uint32_t)p.n_stages * p.stage_bytes <= p.smem_bytes);
    CS_CHECK(2u * p.a_bytes + p.chunk_bytes <= p.stage_bytes && p.n_stages <= kMaxStages && p.Nc <= 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    ptx::grid_dep_launch();
    if (!p.pdl_early) ptx::grid_dep_wait();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));

    const int per_frame = p.flat ? p.tiles_pf : p.nby * p.parts;

    if (warp == kProducerWarp) {
        // ================================================================ producer
        int st = 0;
        uint32_t ph = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            const int f = u / per_frame, rem = u - f * per_frame;
            const int by = rem / p.parts, part = rem - by * p.parts;
            const int row0 = p.flat ? f * p.nblk + rem * 128 : f * p.nblk + by * p.nbx + part * p.L;
            for (int nc = 0; nc < p.n_nc; ++nc) {
                for (int kc = 0; kc < p.n_kc; ++kc) {
                    ptx::mbar_wait(bar_empty + 8 * st, ph ^ 1u);
                    if (lane == 0) {
                        const uint32_t sa = sbase + kOffStage + (uint32_t)st * p.stage_bytes;
                        ptx::mbar_arrive_expect_tx(bar_full + 8 * st, p.a_bytes + p.chunk_bytes);
                        ptx::tma_load_2d(sa, &p.ymap, bar_full + 8 * st, kc * p.Kc, row0);
                        ptx::bulk_load(sa + 2 * p.a_bytes, p.phiT + (size_t)(nc * p.n_kc + kc) * p.chunk_bytes,
                                       p.chunk_bytes, bar_full + 8 * st);
                    }
                    __syncwarp();
                    if (++st == p.n_stages) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp < kConvWarps) {
        // ================================================================ hi/lo split
        int st = 0;
        uint32_t ph = 0;
        const int n16 = (int)(p.a_bytes / 16u);
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            for (int i = 0; i < p.n_nc * p.n_kc; ++i) {
                ptx::mbar_wait(bar_full + 8 * st, ph);
                const uint32_t sa = sbase + kOffStage + (uint32_t)st * p.stage_bytes;
                for (int c = (int)threadIdx.x; c < n16; c += kConvWarps * 32) {
                    const uint4 v = ptx::lds128(sa + (uint32_t)c * 16u);
                    const uint32_t h0 = v.x & 0xFFFFE000u, h1 = v.y & 0xFFFFE000u;
                    const uint32_t h2 = v.z & 0xFFFFE000u, h3 = v.w & 0xFFFFE000u;
                    const uint32_t l0 = __float_as_uint(__uint_as_float(v.x) - __uint_as_float(h0));
                    const uint32_t l1 = __float_as_uint(__uint_as_float(v.y) - __uint_as_float(h1));
                    const uint32_t l2 = __float_as_uint(__uint_as_float(v.z) - __uint_as_float(h2));
                    const uint32_t l3 = __float_as_uint(__uint_as_float(v.w) - __uint_as_float(h3));
                    ptx::sts128(sa + (uint32_t)c * 16u, h0, h1, h2, h3);
                    ptx::sts128(sa + p.a_bytes + (uint32_t)c * 16u, l0, l1, l2, l3);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_conv + 8 * st);
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ================================================================ MMA issuer
        int st = 0;
        uint32_t ph = 0;
        int db = 0;
        uint32_t dph = 0;
        const uint32_t span = (uint32_t)p.Kc * 4u;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            for (int nc = 0; nc < p.n_nc; ++nc) {
                ptx::mbar_wait(bar_dempty + 8 * db, dph ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d_tm = tmem_base + (uint32_t)db * 256u;
                for (int kc = 0; kc < p.n_kc; ++kc) {
                    ptx::mbar_wait(bar_conv + 8 * st, ph);
                    ptx::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = sbase + kOffStage + (uint32_t)st * p.stage_bytes;
                        const uint64_t ahi = ptx::smem_desc_swizzled(sa, span, p.a_sbo);
                        const uint64_t alo = ptx::smem_desc_swizzled(sa + p.a_bytes, span, p.a_sbo);
                        const uint64_t bd = ptx::smem_desc_noswizzle(sa + 2 * p.a_bytes, p.b_lbo, 128u);
                        for (int ks = 0; ks < p.Kc / 8; ++ks) {
                            // K step of 8 tf32: +32 B inside the swizzled row; +2 core matrices (2 LBO) in B
                            const uint64_t ka = (uint64_t)(ks * 2), kb = (uint64_t)(ks * 2) * (p.b_lbo >> 4);
                            ptx::mma_tf32_ss(d_tm, ahi + ka, bd + kb, p.idesc, (kc | ks) != 0 ? 1u : 0u);
                            ptx::mma_tf32_ss(d_tm, alo + ka, bd + kb, p.idesc, 1u);
                        }
                        ptx::tc_commit(bar_empty + 8 * st);
                        if (kc == p.n_kc - 1) ptx::tc_commit(bar_dfull + 8 * db);
                    }
                    __syncwarp();
                    if (++st == p.n_stages) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
                if (++db == 2) {
                    db = 0;
                    dph ^= 1u;
                }
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ================================================================ epilogue
        if (p.pdl_early) ptx::grid_dep_wait();
        const int ew = warp - kEpiWarp0;   // == warp % 4: TMEM lanes 32*ew .. 32*ew+31
        const uint32_t lane_bits = (uint32_t)(ew * 32) << 16;
        const uint32_t tile = sbase + kOffEpi + (uint32_t)ew * 4096u;
        const int rows_per_chunk = p.Nc / B;
        int db = 0;
        uint32_t dph = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            const int f = u / per_frame, rem = u - f * per_frame;
            int by, bx0, nv;   // block row, first block of this warp, blocks of this warp (may be <= 0)
            if (p.flat) {
                const int b0 = rem * 128 + ew * 32;
                by = b0 / p.nbx;
                bx0 = b0 - by * p.nbx;
                nv = min(32, p.nblk - b0);
            } else {
                by = rem / p.parts;
                const int part = rem - by * p.parts;
                bx0 = part * p.L + ew * 32;
                nv = min(32, min(p.L - ew * 32, p.nbx - bx0));
            }
            const int col0 = bx0 * B;
            const int valid = nv > 0 ? min(nv * B, p.W - col0) : 0;
            for (int nc = 0; nc < p.n_nc; ++nc) {
                ptx::mbar_wait(bar_dfull + 8 * db, dph);
                ptx::tc_fence_after();
                const uint32_t d_tm = tmem_base + lane_bits + (uint32_t)db * 256u;
                // one 32-column TMEM load covers 32 / B pixel rows (B = 8: 4 rows, B = 16: 2, B = 32: 1)
                constexpr int kRowsPerLd = 32 / B;
                for (int pr0 = 0; pr0 < rows_per_chunk; pr0 += kRowsPerLd) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)(pr0 * B), v);
                    ptx::tc_wait_ld();
#pragma unroll
                    for (int k = 0; k < kRowsPerLd; ++k) {
                        const int Y = by * B + nc * rows_per_chunk + pr0 + k;
                        float* dst = p.x + ((long long)f * p.H + Y) * p.W + col0;
                        CS_CHECK(Y >= p.H || valid <= 0 || ((long long)f * p.H + Y) * p.W + col0 + valid <= p.x_floats);
                        if (Y < p.H && valid > 0) row_store<B / 4>(v + k * B, tile, lane, dst, valid);
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_dempty + 8 * db);
                if (++db == 2) {
                    db = 0;
                    dph ^= 1u;
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kMmaWarp) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace adj
}  // namespace csenc
