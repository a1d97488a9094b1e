// cs_measure_kernel.cuh -- K1: fused GOP residual formation + block CS measurement on sm_100a.
//
// One persistent, warp-specialised kernel per encode call.  Per work unit
// (stream s, GOP g, tile t of full-width block rows, range of CS frames of the GOP):
//
//   warp 0        TMA producer: Phi -> SMEM once; the key tile (double buffered) and the CS
//                 tiles (ring of n_stages) with 3-D tiled tensor-map loads [frame][y][x] whose
//                 out-of-bounds rows/columns are zero-filled (partial blocks, reading R10).
//   warps 4..7    converters ("im2col + residual", a2+a3): thread = TMEM lane = block of the
//                 tile.  Reads its B x B block of the CS frame and of the key frame from SMEM,
//                 forms the exact residual r = F - F_key as fp16 (magic-number trick) and
//                 writes it with tcgen05.st as the MMA A operand in TMEM (row = block, K = the
//                 row-major pixel index j = yy*B + xx, two fp16 per 32-bit column).
//   warp 1        MMA issuer (a4): D[tmem, fp32] = A[tmem, fp16] x Phi^T[smem, fp16], one
//                 tcgen05.mma.kind::f16 (M=128 lanes, N=Mpad, K=16) per 16 pixels, chained
//                 over the block; commit -> mbarriers.
//   warps 8..11   epilogue (a6): tcgen05.ld of the fp32 accumulators, vectorised stores of
//                 y[s][g][c][by][bx][0..M) (block-major, M*4 contiguous bytes per block).
//   warp 2        TMEM allocator.
//
// Pipelines (mbarrier phase/parity rings): stage_full/empty (TMA <-> converters), key_full/
// empty (double-buffered key tile), a_full/empty (converters <-> MMA, 2 TMEM A buffers),
// d_full/empty (MMA <-> epilogue, 2 TMEM accumulators).  Paper passages: Eq.(1) P:83-85,
// P:87 and Eq.(2)-(3) P:89-91 (see include/cs_encoder.h).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "ptx_sm100.cuh"

namespace csenc {

constexpr int kThreads = 384;
constexpr int kMaxFolds = 8;
constexpr int kMaxStages = 8;
constexpr uint32_t kTmemCols = 512;

struct KParams {
    float* out;
    const uint16_t* phi;      // device, canonical UMMA layout, phi_bytes
    uint32_t phi_bytes;
    int M, Mpad, N;
    int nbx, nby, nblk;
    // tiling
    int T_r, F, L, n_tiles;
    int chunk_rows, n_chunks, chunk_k;
    int box_w, n_box, box_rows, pieces;
    int single_piece;         // 1: one box row-range covers all T_r*B rows of the tile (n_chunks == 1)
    uint32_t box_bytes, stage_cs_bytes, stage_bytes, key_bytes;
    int key_resident, n_stages;
    uint32_t off_phi, off_key, off_stage;
    // work
    int G, T, gop_begin, n_gops_sel, cs_per_stream_sel, n_splits, cs_per_unit, n_units;
    // MMA
    uint32_t idesc, lbo, sbo;
    int a_cols, d_cols;
    int n_abuf, n_dbuf;       // TMEM ring depths (1 or 2)
};

struct Unit {
    int s, g, t, c0, c1;
};

__device__ __forceinline__ bool decode_unit(const KParams& p, int u, Unit& w) {
    int j = u % p.n_splits;
    int r = u / p.n_splits;
    w.t = r % p.n_tiles;
    r /= p.n_tiles;
    int gl = r % p.n_gops_sel;
    w.s = r / p.n_gops_sel;
    w.g = p.gop_begin + gl;
    int gop_len = min(p.G, p.T - w.g * p.G);
    int ncs = gop_len - 1;
    w.c0 = j * p.cs_per_unit;
    w.c1 = min(w.c0 + p.cs_per_unit, ncs);
    return w.c1 > w.c0;
}

// Issue the TMA boxes of one K-chunk of one tile of frame z into dst (layout [piece][box][rows][box_w]).
__device__ __forceinline__ void load_tile_chunk(const KParams& p, const CUtensorMap* tmap, uint32_t dst, int z,
                                                int t, int k, uint32_t bar, uint64_t policy) {
    const int B_rows_tile = p.T_r * (p.chunk_k / p.chunk_rows);  // T_r * B
    for (int pc = 0; pc < p.pieces; ++pc) {
        int y = p.single_piece ? t * B_rows_tile : (t * p.T_r + pc) * (p.chunk_k / p.chunk_rows) + k * p.chunk_rows;
        for (int b = 0; b < p.n_box; ++b) {
            ptx::tma_load_3d(dst + (uint32_t)(pc * p.n_box + b) * p.box_bytes, tmap, bar, b * p.box_w, y, z, policy);
        }
    }
}

// Converter: one block-row segment of B pixels -> B/2 fp16x2 residual words.
template <int B>
struct RowConv;

template <>
struct RowConv<8> {
    static constexpr int kWords = 4;
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w) {
        uint2 c = ptx::lds64(cs), k = ptx::lds64(key);
        ptx::residual4(c.x, k.x, w[0], w[1]);
        ptx::residual4(c.y, k.y, w[2], w[3]);
    }
};
template <>
struct RowConv<16> {
    static constexpr int kWords = 8;
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w) {
        uint4 c = ptx::lds128(cs), k = ptx::lds128(key);
        ptx::residual4(c.x, k.x, w[0], w[1]);
        ptx::residual4(c.y, k.y, w[2], w[3]);
        ptx::residual4(c.z, k.z, w[4], w[5]);
        ptx::residual4(c.w, k.w, w[6], w[7]);
    }
};
template <>
struct RowConv<32> {
    static constexpr int kWords = 16;
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w) {
        RowConv<16>::run(cs, key, w);
        RowConv<16>::run(cs + 16, key + 16, w + 8);
    }
};

template <int B>
__global__ void __launch_bounds__(kThreads, 1)
    cs_measure_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ KParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31u;

    // barrier block at sbase: [stage_full x8][stage_empty x8][key_full x2][key_empty x2]
    //                         [a_full x2][a_empty x2][d_full x2][d_empty x2][phi_full][tmem slot]
    const uint32_t bar_stage_full = sbase;
    const uint32_t bar_stage_empty = sbase + 8 * kMaxStages;
    const uint32_t bar_key_full = sbase + 16 * kMaxStages;
    const uint32_t bar_key_empty = bar_key_full + 16;
    const uint32_t bar_a_full = bar_key_full + 32;
    const uint32_t bar_a_empty = bar_key_full + 48;
    const uint32_t bar_d_full = bar_key_full + 64;
    const uint32_t bar_d_empty = bar_key_full + 80;
    const uint32_t bar_phi = bar_key_full + 96;
    const uint32_t tmem_slot = bar_key_full + 104;
    const uint32_t s_phi = sbase + p.off_phi;
    const uint32_t s_key = sbase + p.off_key;
    const uint32_t s_stage = sbase + p.off_stage;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(bar_stage_full + 8 * i, 1);
            ptx::mbar_init(bar_stage_empty + 8 * i, 4);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_key_full + 8 * i, 1);
            ptx::mbar_init(bar_key_empty + 8 * i, 4);
            ptx::mbar_init(bar_a_full + 8 * i, 4);
            ptx::mbar_init(bar_a_empty + 8 * i, 1);
            ptx::mbar_init(bar_d_full + 8 * i, 1);
            ptx::mbar_init(bar_d_empty + 8 * i, 4);
        }
        ptx::mbar_init(bar_phi, 1);
        ptx::fence_mbarrier_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc(tmem_slot, kTmemCols);
        ptx::tmem_relinquish();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));

    const uint32_t a_col0 = 0;
    const uint32_t d_col0 = (uint32_t)(p.n_abuf * p.a_cols);

    if (warp == 0) {
        // ================================================================ TMA producer
        if (lane == 0) {
            const uint64_t pol_stream = ptx::policy_evict_first();
            const uint64_t pol_key = ptx::policy_evict_last();
            ptx::mbar_arrive_expect_tx(bar_phi, p.phi_bytes);
            ptx::bulk_load(s_phi, p.phi, p.phi_bytes, bar_phi);
            int st = 0;
            uint32_t ph = 0;
            int kb = 0;
            uint32_t kph = 0;
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                Unit w;
                if (!decode_unit(p, u, w)) continue;
                const int zkey = w.s * p.T + w.g * p.G;
                if (p.key_resident) {
                    ptx::mbar_wait(bar_key_empty + 8 * kb, kph ^ 1u);
                    ptx::mbar_arrive_expect_tx(bar_key_full + 8 * kb, p.key_bytes);
                    for (int k = 0; k < p.n_chunks; ++k)
                        load_tile_chunk(p, &tmap, s_key + (uint32_t)kb * p.key_bytes + (uint32_t)k * p.stage_cs_bytes,
                                        zkey, w.t, k, bar_key_full + 8 * kb, pol_key);
                    kb ^= 1;
                    if (kb == 0) kph ^= 1u;
                }
                for (int c = w.c0; c < w.c1; ++c) {
                    const int zcs = zkey + 1 + c;
                    for (int k = 0; k < p.n_chunks; ++k) {
                        ptx::mbar_wait(bar_stage_empty + 8 * st, ph ^ 1u);
                        const uint32_t dst = s_stage + (uint32_t)st * p.stage_bytes;
                        ptx::mbar_arrive_expect_tx(bar_stage_full + 8 * st, p.stage_bytes);
                        load_tile_chunk(p, &tmap, dst, zcs, w.t, k, bar_stage_full + 8 * st, pol_stream);
                        if (!p.key_resident)
                            load_tile_chunk(p, &tmap, dst + p.stage_cs_bytes, zkey, w.t, k, bar_stage_full + 8 * st,
                                            pol_key);
                        if (++st == p.n_stages) {
                            st = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            ptx::mbar_wait(bar_phi, 0);
            ptx::tc_fence_after();
            int ab = 0, db = 0;
            uint32_t aph = 0, dph = 0;
            const int ksteps = p.chunk_k / 16;
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                Unit w;
                if (!decode_unit(p, u, w)) continue;
                for (int c = w.c0; c < w.c1; ++c) {
                    ptx::mbar_wait(bar_d_empty + 8 * db, dph ^ 1u);
                    ptx::tc_fence_after();
                    const uint32_t d_tm = tmem_base + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                    for (int k = 0; k < p.n_chunks; ++k) {
                        ptx::mbar_wait(bar_a_full + 8 * ab, aph);
                        ptx::tc_fence_after();
                        const uint32_t a_tm = tmem_base + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                        for (int f = 0; f < p.F; ++f) {
                            for (int s = 0; s < ksteps; ++s) {
                                const int kg = k * ksteps + s;  // global K step (16 pixels)
                                const uint64_t bdesc =
                                    ptx::smem_desc_noswizzle(s_phi + (uint32_t)(2 * kg) * p.lbo, p.lbo, p.sbo);
                                ptx::mma_f16_ts(d_tm + (uint32_t)(f * p.Mpad),
                                                a_tm + (uint32_t)(f * (p.chunk_k / 2) + s * 8), bdesc, p.idesc,
                                                (k > 0 || s > 0) ? 1u : 0u);
                            }
                        }
                        ptx::tc_commit(bar_a_empty + 8 * ab);
                        if (++ab == p.n_abuf) {
                            ab = 0;
                            aph ^= 1u;
                        }
                    }
                    ptx::tc_commit(bar_d_full + 8 * db);
                    if (++db == p.n_dbuf) {
                        db = 0;
                        dph ^= 1u;
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ================================================================ converters (a2 + a3)
        const int lane_idx = (warp - 4) * 32 + (int)lane;       // TMEM lane = block slot
        const uint32_t lane_bits = (uint32_t)((warp - 4) * 32) << 16;
        const int Bconst = B;
        // per-fold SMEM offset of this lane's block (row yy = 0) inside a stage
        uint32_t off[kMaxFolds];
#pragma unroll
        for (int f = 0; f < kMaxFolds; ++f) {
            off[f] = 0;
            if (f < p.F) {
                int b = f * p.L + lane_idx;
                if (lane_idx < p.L && b < p.T_r * p.nbx) {
                    int brow = b / p.nbx, bx = b % p.nbx;
                    int pc = p.single_piece ? 0 : brow;
                    int row0 = p.single_piece ? brow * Bconst : 0;
                    int x = bx * Bconst;
                    int box = x / p.box_w, xo = x % p.box_w;
                    off[f] = (uint32_t)(pc * p.n_box + box) * p.box_bytes + (uint32_t)(row0 * p.box_w + xo);
                }
            }
        }
        constexpr int kWords = RowConv<B>::kWords;      // fp16x2 words per pixel row
        constexpr int kRowsPerSt = 32 / kWords;         // rows per 32-column TMEM store
        int st = 0, ab = 0, kb = 0;
        uint32_t ph = 0, aph = 0, kph = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            if (p.key_resident) ptx::mbar_wait(bar_key_full + 8 * kb, kph);
            for (int c = w.c0; c < w.c1; ++c) {
                for (int k = 0; k < p.n_chunks; ++k) {
                    ptx::mbar_wait(bar_stage_full + 8 * st, ph);
                    ptx::mbar_wait(bar_a_empty + 8 * ab, aph ^ 1u);
                    ptx::tc_fence_after();
                    const uint32_t cs_base = s_stage + (uint32_t)st * p.stage_bytes;
                    const uint32_t key_base = p.key_resident
                                                  ? s_key + (uint32_t)kb * p.key_bytes + (uint32_t)k * p.stage_cs_bytes
                                                  : cs_base + p.stage_cs_bytes;
                    const uint32_t a_tm = tmem_base + lane_bits + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                    for (int f = 0; f < p.F; ++f) {
                        const uint32_t cs_a = cs_base + off[f], key_a = key_base + off[f];
                        const uint32_t a_f = a_tm + (uint32_t)(f * (p.chunk_k / 2));
                        for (int r0 = 0; r0 < p.chunk_rows; r0 += kRowsPerSt) {
                            uint32_t v[32];
#pragma unroll
                            for (int rr = 0; rr < kRowsPerSt; ++rr) {
                                const uint32_t ro = (uint32_t)((r0 + rr) * p.box_w);
                                RowConv<B>::run(cs_a + ro, key_a + ro, v + rr * kWords);
                            }
                            ptx::tmem_st_32x32b_x32(a_f + (uint32_t)(r0 * kWords), v);
                        }
                    }
                    ptx::tc_wait_st();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::mbar_arrive(bar_a_full + 8 * ab);
                        ptx::mbar_arrive(bar_stage_empty + 8 * st);
                    }
                    if (++ab == p.n_abuf) {
                        ab = 0;
                        aph ^= 1u;
                    }
                    if (++st == p.n_stages) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
            }
            if (p.key_resident) {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_key_empty + 8 * kb);
                kb ^= 1;
                if (kb == 0) kph ^= 1u;
            }
        }
    } else if (warp >= 8) {
        // ================================================================ epilogue (a6)
        const int lane_idx = (warp - 8) * 32 + (int)lane;
        const uint32_t lane_bits = (uint32_t)((warp - 8) * 32) << 16;
        const bool vec = (p.M & 3) == 0;
        int db = 0;
        uint32_t dph = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            const int rows_here = min(p.T_r, p.nby - w.t * p.T_r);
            const int blocks_here = rows_here * p.nbx;
            const int blk0 = w.t * p.T_r * p.nbx;
            for (int c = w.c0; c < w.c1; ++c) {
                ptx::mbar_wait(bar_d_full + 8 * db, dph);
                ptx::tc_fence_after();
                const long long cs_global = (long long)w.s * p.cs_per_stream_sel +
                                            (long long)(w.g - p.gop_begin) * (p.G - 1) + c;
                const uint32_t d_tm = tmem_base + lane_bits + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                for (int f = 0; f < p.F; ++f) {
                    const int b = f * p.L + lane_idx;
                    const bool valid = lane_idx < p.L && b < blocks_here;
                    float* dst = p.out + (cs_global * p.nblk + blk0 + b) * (long long)p.M;
                    for (int j = 0; j < p.Mpad; j += 16) {
                        uint32_t v[16];
                        ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad + j), v);
                        ptx::tc_wait_ld();
                        if (valid) {
                            const int nm = min(16, p.M - j);
                            if (vec) {
#pragma unroll
                                for (int q = 0; q < 16; q += 4)
                                    if (q < nm) ptx::stg128(dst + j + q, v[q], v[q + 1], v[q + 2], v[q + 3]);
                            } else {
#pragma unroll
                                for (int q = 0; q < 16; ++q)
                                    if (q < nm) dst[j + q] = __uint_as_float(v[q]);
                            }
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_d_empty + 8 * db);
                if (++db == p.n_dbuf) {
                    db = 0;
                    dph ^= 1u;
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace csenc
