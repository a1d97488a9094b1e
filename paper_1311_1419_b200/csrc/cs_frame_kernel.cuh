// cs_frame_kernel.cuh -- K4: paper-faithful frame-level measurement.
//
// Eq. (1), as the paper states it: one dense Gaussian A in R^{m x n}, n = W*H (
// SPEC.md:133-134), measures the whole vectorised residual of every CS frame, y = A r,
// r = vec(F_cs - F_key) row-major.  Batched over the CS frames of many GOPs this is a GEMM
//   D[128 measurements x N CS frames] += A[128 x K] * R[N x K]^T
// with K = n pixels: tensor-core bound (2 m n flop per frame against n bytes), unlike the block
// path.  tcgen05.mma kind::f16 (fp16 x fp16 -> fp32), both operands from SMEM (SS form):
//   A: TMA 2-D box [256 rows][64 fp16] of the device copy of A (SWIZZLE_128B = the UMMA K-major
//      SW128 layout); the copy's columns are permuted within groups of 4 pixels to the converters'
//      (0,2,1,3) pair order (ptx::residual4), so K index k multiplies pixel 4(k/4)+{0,2,1,3}[k%4].
//   R: TMA 2-D box [nf rows][64 bytes] of a window of whole GOPs (keys included, SWIZZLE_64B);
//      4 converter warps form the exact fp16 residual of every CS frame of the window against its
//      GOP key (same box) and write it as the SW128 K-major B operand.
// Roles (15 warps): 0-7 converters, 8-11 epilogue, 12 frames producer, 13 MMA issuer + TMEM allocator,
// 14 A producer.  The frame boxes (from HBM, needed first: by the converters) and the A tiles (from L2,
// needed last: by the MMA) run in two rings of their own depths, so the frames are fetched far ahead
// (up to 8 chunks) while A occupies only the slots the MMA is about to use.
// Unit = (window of whole GOPs, pair of 128-row m-tiles = one 256-row A box); item = one 64-pixel K
// chunk: one residual operand feeds both m-tiles' MMAs (D uses all 512 TMEM columns), halving the
// conversion work and the frame-box traffic per flop.  Work split (stream-K): the (unit, K chunk)
// sequence is cut into gridDim.x equal ranges, one per CTA, so windows can be as large as a TMA box
// allows (the per-chunk A traffic per flop falls with the window) while every SM gets the same number
// of chunks.  A piece = the part of a CTA's range inside one unit; a unit done by one CTA is written
// to y directly, the pieces of a unit cut by CTA boundaries go to per-CTA partial tiles that
// cs_frame_fixup_kernel sums in CTA order (deterministic).  The epilogue's lane = measurement, so for
// each CS frame a warp stores 32 consecutive measurements (128 B).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "ptx_sm100.cuh"

namespace csenc {
namespace frm {

#ifndef CSENC_FRAME_CONV_WARPS
#define CSENC_FRAME_CONV_WARPS 16
#endif
constexpr int kConvWarps = CSENC_FRAME_CONV_WARPS;   // residual converters (a multiple of 4)
constexpr int kConvRowGroups = kConvWarps * 4;         // 8-lane row groups: rows c = group + kConvRowGroups i
constexpr int kConvRows = (256 + kConvRowGroups - 1) / kConvRowGroups;   // CS rows per thread and chunk
constexpr int kEpiWarp0 = kConvWarps;                  // a warpgroup: TMEM lane quarters = warp % 4
constexpr int kProducerWarp = kConvWarps + 4;          // frame boxes
constexpr int kMmaWarp = kConvWarps + 5;
constexpr int kAProducerWarp = kConvWarps + 6;         // A tiles
constexpr int kThreads = (kConvWarps + 7) * 32;
constexpr int kMaxStages = 8;
constexpr int kKc = 64;                          // pixels per K chunk
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOffB = 1024;                 // two residual (B operand) buffers of b_bytes

struct FParams {
    CUtensorMap fmap;         // frames: 2-D [n_seq*T rows][n bytes], box [nf_box][64], SWIZZLE_64B
    CUtensorMap amap;         // A (permuted): 2-D [m rows][n fp16], box [256][64], SWIZZLE_128B
    float* out;               // y [n_seq*cs_s][m]
    float* part;              // partial tiles [2 * gridDim.x][256 CS][256 rows] fp32: CTA b's first piece
                              // (if partial) in tile 2b, its last partial piece in tile 2b + 1
    int n, m, G, T, cs_s;     // pixels, measurements, GOP, frames/stream, CS frames/stream
    int gw, nf_box;           // GOPs per window, frame rows of a window (= gw * G)
    int n_fbox, fbox_rows;    // TMA boxes per chunk (box dims <= 256) and rows per box (multiple of 8): the
                              // boxes land back to back, so row t of the window is at byte 64 t of the slot
    int n_win_s, n_win;       // windows per stream, all windows
    int global_win;           // T % G == 0: windows run over the concatenated GOPs of all streams
    int total_gops;           // n_seq * T / G (global_win)
    int n_mp, n_chunks;       // 256-row m-pairs, 64-pixel chunks
    int n_units;
    long long total_chunks;   // n_win * n_chunks (per m-pair): CTA b = j n_mp + mp takes m-pair mp's chunks
                              // [j C / gj, (j + 1) C / gj) of the (window, K chunk) sequence, gj = grid / n_mp
                              // (the n_mp CTAs of one j read the same frame boxes at about the same time)
    uint32_t fbox_bytes;      // the chunk's frame boxes (n_fbox * fbox_rows rows x 64 B)
    uint32_t off_a;           // A ring: n_a slots of 256 * kKc fp16 (32 KB), 1024-aligned
    int n_a;
    uint32_t stage_bytes;     // frames ring slot (fbox_bytes rounded up to 1024)
    uint32_t b_bytes;         // one residual buffer: roundup(window CS rows * 128, 1024)
    int n_b;                  // residual buffers (2..4)
    uint32_t off_stage;       // frames ring: kOffB + n_b * b_bytes
    int n_stages;             // frames ring slots
    int prefetch;             // frame boxes prefetched into L2 this many chunks ahead (0 = off)
    unsigned long long* trace;   // debug timeline (CTA 0): [4][trace_cap] clock64, nullptr = off
    int trace_cap;
    long long out_floats;     // floats in y (CSENC_CHECKS)
    uint32_t smem_bytes;      // dynamic SMEM from the aligned base (CSENC_CHECKS)
};

// trace events: 0 producer issued, 1 converter data landed, 2 converter done, 3 MMA issued
__device__ __forceinline__ void ftrace(const FParams& p, int ev, int i) {
    if (p.trace != nullptr && blockIdx.x == 0 && i < p.trace_cap) p.trace[(size_t)ev * p.trace_cap + i] = clock64();
}

struct FUnit {
    int u, s, g0, ngops, n_cs, cs0, mp, kc0, kc1;
    int slot;                 // partial tile of this piece, -1 = whole unit (written to y)
};

// Stream-K ranges (per m-pair, gj ranges): range j = chunks [cbeg(j), cbeg(j + 1)) of the (window, K chunk)
// sequence; range_of(c) = the range holding chunk c.
__device__ __forceinline__ long long cbeg(const FParams& p, long long j, long long gj) {
    return j * p.total_chunks / gj;
}
__device__ __forceinline__ int range_of(const FParams& p, long long c, long long gj) {
    return (int)(((c + 1) * gj - 1) / p.total_chunks);
}

// Unit u = win * n_mp + mp: (window, m-pair).
__device__ __forceinline__ void decode_funit(const FParams& p, int u, FUnit& w) {
    w.u = u;
    w.mp = u % p.n_mp;
    const int win = u / p.n_mp;
    w.kc0 = 0;
    w.kc1 = p.n_chunks;
    w.slot = -1;
    if (win >= p.n_win) {
        w.s = 0;
        w.g0 = 0;
        w.ngops = 0;
        w.n_cs = 0;
        w.cs0 = 0;
        return;
    }
    if (p.global_win) {
        // every stream is whole GOPs: GOP gg of the concatenation starts at frame row gg * G and
        // its CS frames are global CS rows gg * (G-1) ... (stream offsets included)
        w.s = 0;
        w.g0 = win * p.gw;
        w.ngops = min(p.gw, p.total_gops - w.g0);
        w.n_cs = w.ngops * (p.G - 1);
    } else {
        w.s = win / p.n_win_s;
        const int wi = win - w.s * p.n_win_s;
        w.g0 = wi * p.gw;
        const int n_gops = (p.T + p.G - 1) / p.G;
        w.ngops = min(p.gw, n_gops - w.g0);
        const int t_end = min(p.T, (w.g0 + w.ngops) * p.G);
        w.n_cs = (t_end - w.g0 * p.G) - w.ngops;        // frames in the window minus its keys
    }
    w.cs0 = w.g0 * (p.G - 1);
}

// The piece of CTA `cid` (m-pair mp, range [cb, ce)) that starts at chunk c: its unit and K range, and its
// partial tile when the unit is cut by a range boundary (tile 2 cid for the CTA's first piece, 2 cid + 1 else).
__device__ __forceinline__ void piece_at(const FParams& p, long long c, long long cb, long long ce, int cid, int mp,
                                         FUnit& w) {
    const int win = (int)(c / p.n_chunks);
    decode_funit(p, win * p.n_mp + mp, w);
    w.kc0 = (int)(c - (long long)win * p.n_chunks);
    w.kc1 = (int)min((long long)p.n_chunks, (long long)w.kc0 + (ce - c));
    if (w.kc0 != 0 || w.kc1 != p.n_chunks) w.slot = 2 * cid + (c == cb ? 0 : 1);
}

__global__ void __launch_bounds__(kThreads, 1) cs_frame_measure_kernel(const __grid_constant__ FParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31u;

    const uint32_t bar_full = sbase;                      // [kMaxStages] frame box landed -> converters
    const uint32_t bar_empty = sbase + 8 * kMaxStages;    // [kMaxStages] converters done -> frames producer
    const uint32_t bar_afull = sbase + 32 * kMaxStages;   // [kMaxStages] A tile landed -> MMA
    const uint32_t bar_aempty = sbase + 40 * kMaxStages;  // [kMaxStages] MMA done -> A producer
    const uint32_t bar_conv = sbase + 16 * kMaxStages;    // [4] converters -> MMA (B buffer written)
    const uint32_t bar_bempty = bar_conv + 32;            // [4] MMA -> converters (B buffer free)
    const uint32_t bar_dfull = bar_bempty + 32;
    const uint32_t bar_dempty = bar_dfull + 8;
    const uint32_t tmem_slot = bar_dempty + 8;

    const int cid = (int)blockIdx.x, n_cl = (int)gridDim.x;
    const int cmp = cid % p.n_mp;                   // this CTA's m-pair and stream-K range
    const long long gj = n_cl / p.n_mp, cj = cid / p.n_mp;
    const long long c_beg = cbeg(p, cj, gj), c_end = cbeg(p, cj + 1, gj);
    if (threadIdx.x == 0) {
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(bar_full + 8 * i, 1);
            ptx::mbar_init(bar_empty + 8 * i, kConvWarps);
        }
        for (int i = 0; i < p.n_a; ++i) {
            ptx::mbar_init(bar_afull + 8 * i, 1);
            ptx::mbar_init(bar_aempty + 8 * i, 1);
        }
        for (int i = 0; i < 4; ++i) {
            ptx::mbar_init(bar_conv + 8 * i, kConvWarps);
            ptx::mbar_init(bar_bempty + 8 * i, 1);
        }
        ptx::mbar_init(bar_dfull, 1);
        ptx::mbar_init(bar_dempty, 4);
        ptx::fence_mbarrier_init();
    }
    if (warp == kMmaWarp) {
        ptx::tmem_alloc(tmem_slot, kTmemCols);
        ptx::tmem_relinquish();
    }
    if (warp == kProducerWarp && lane == 0) {
        ptx::prefetch_tmap(&p.fmap);
        ptx::prefetch_tmap(&p.amap);
    }
    CS_CHECK(p.off_stage + (uint32_t)p.n_stages * p.stage_bytes <= p.off_a && p.n_stages <= kMaxStages);
    CS_CHECK(p.off_a + (uint32_t)p.n_a * 256u * kKc * 2u <= p.smem_bytes && p.n_a <= kMaxStages);
    CS_CHECK(p.fbox_bytes <= p.stage_bytes && p.n_b <= 4);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));

    if (warp == kProducerWarp) {
        // ================================================================ producer
        int st = 0, ntr = 0;
        uint32_t ph = 0;
        for (long long c = c_beg; c < c_end;) {
            FUnit w;
            piece_at(p, c, c_beg, c_end, cid, cmp, w);
            c += w.kc1 - w.kc0;
            const int row0 = w.s * p.T + w.g0 * p.G;
            if (lane == 0)   // frames stream from HBM: pull the first boxes of the unit into L2 early
                for (int kc = w.kc0; kc < min(w.kc1, w.kc0 + p.prefetch); ++kc)
                    ptx::tma_prefetch_2d(&p.fmap, kc * kKc, row0);
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_empty + 8 * st, ph ^ 1u);
                if (lane == 0 && p.prefetch > 0 && kc + p.prefetch < w.kc1)
                    ptx::tma_prefetch_2d(&p.fmap, (kc + p.prefetch) * kKc, row0);
                if (lane == 0) {
                    const uint32_t sf = sbase + p.off_stage + (uint32_t)st * p.stage_bytes;
                    ptx::mbar_arrive_expect_tx(bar_full + 8 * st, p.fbox_bytes);
                    for (int j = 0; j < p.n_fbox; ++j)   // rows past the tensor are zero-filled (and counted)
                        ptx::tma_load_2d(sf + (uint32_t)(j * p.fbox_rows * 64), &p.fmap, bar_full + 8 * st, kc * kKc,
                                         row0 + j * p.fbox_rows);
                    ftrace(p, 0, ntr);
                }
                ++ntr;
                __syncwarp();
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == kAProducerWarp) {
        // ================================================================ A producer
        int as = 0;
        uint32_t aph = 0;
        for (long long c = c_beg; c < c_end;) {
            FUnit w;
            piece_at(p, c, c_beg, c_end, cid, cmp, w);
            c += w.kc1 - w.kc0;
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_aempty + 8 * as, aph ^ 1u);
                if (lane == 0) {
                    const uint32_t sa = sbase + p.off_a + (uint32_t)as * (256u * kKc * 2u);
                    ptx::mbar_arrive_expect_tx(bar_afull + 8 * as, 256u * kKc * 2u);
                    ptx::tma_load_2d(sa, &p.amap, bar_afull + 8 * as, kc * kKc, w.mp * 256);
                }
                __syncwarp();
                if (++as == p.n_a) {
                    as = 0;
                    aph ^= 1u;
                }
            }
        }
    } else if (warp < kConvWarps) {
        // ================================================================ residual -> B operand
        // thread: 8-pixel group q = tid & 7 of CS rows c = tid/8 + kConvRowGroups i (i < kConvRows).  Row c of a window
        // is CS frame 1 + c % (G-1) of the window's GOP c / (G-1): frame row and key row packed.
        const int tid = (int)threadIdx.x;
        const int q = tid & 7;
        uint32_t rows[kConvRows];
#pragma unroll
        for (int i = 0; i < kConvRows; ++i) {
            const int c = (tid >> 3) + kConvRowGroups * i;
            const int gl = c / (p.G - 1), pos = c - gl * (p.G - 1);
            rows[i] = (uint32_t)(gl * p.G + 1 + pos) | ((uint32_t)(gl * p.G) << 16);
        }
        int st = 0, b = 0, ntr = 0;
        uint32_t ph = 0, bph = 0;
        for (long long c = c_beg; c < c_end;) {
            FUnit w;
            piece_at(p, c, c_beg, c_end, cid, cmp, w);
            c += w.kc1 - w.kc0;
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_full + 8 * st, ph);
                if (tid == 0) ftrace(p, 1, ntr);
                ptx::mbar_wait(bar_bempty + 8 * b, bph ^ 1u);
                const uint32_t sf = sbase + p.off_stage + (uint32_t)st * p.stage_bytes;
                const uint32_t sb = sbase + kOffB + (uint32_t)b * p.b_bytes;
                // all loads first (rows past the window read row 0: harmless, not stored), then convert
                uint2 fv[kConvRows], kv[kConvRows];
#pragma unroll
                for (int i = 0; i < kConvRows; ++i) {
                    const int c = (tid >> 3) + kConvRowGroups * i;
                    const uint32_t rr = c < w.n_cs ? rows[i] : 0u;
                    const uint32_t t = rr & 0xFFFFu, k = rr >> 16;
                    // SWIZZLE_64B box rows of 64 B: 16-B chunk (q/2) ^ ((row/2) & 3), 8-B half q & 1
                    const uint32_t ct = t * 64u + ((((uint32_t)(q >> 1)) ^ ((t >> 1) & 3u)) << 4) + (uint32_t)(q & 1) * 8u;
                    const uint32_t ck = k * 64u + ((((uint32_t)(q >> 1)) ^ ((k >> 1) & 3u)) << 4) + (uint32_t)(q & 1) * 8u;
                    fv[i] = ptx::lds64(sf + ct);
                    kv[i] = ptx::lds64(sf + ck);
                }
#pragma unroll
                for (int i = 0; i < kConvRows; ++i) {
                    const int c = (tid >> 3) + kConvRowGroups * i;
                    if (c < w.n_cs) {
                        CS_CHECK((rows[i] & 0xFFFFu) < (uint32_t)p.nf_box && (rows[i] >> 16) < (uint32_t)p.nf_box);
                        CS_CHECK((uint32_t)(c + 1) * 128u <= p.b_bytes);
                        uint32_t w0, w1, w2, w3;
                        ptx::residual4(fv[i].x, kv[i].x, w0, w1);
                        ptx::residual4(fv[i].y, kv[i].y, w2, w3);
                        // SWIZZLE_128B B rows of 128 B: 16-B chunk q ^ (c & 7)
                        ptx::sts128(sb + (uint32_t)c * 128u + ((uint32_t)(q ^ (c & 7)) << 4), w0, w1, w2, w3);
                    }
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(bar_conv + 8 * b);
                    ptx::mbar_arrive(bar_empty + 8 * st);   // frame box read (values are in registers)
                }
                if (tid == 0) ftrace(p, 2, ntr);
                ++ntr;
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
                if (++b == p.n_b) {
                    b = 0;
                    bph ^= 1u;
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ================================================================ MMA issuer
        // D: m-tile 0 at TMEM columns [0, N), m-tile 1 at [256, 256 + N); single-buffered (a unit is
        // hundreds of chunks long, the epilogue a few thousand cycles)
        int st = 0, b = 0, ntr = 0;   // st: A ring slot
        uint32_t ph = 0, bph = 0, dph = 0;
        for (long long c = c_beg; c < c_end;) {
            FUnit w;
            piece_at(p, c, c_beg, c_end, cid, cmp, w);
            c += w.kc1 - w.kc0;
            const uint32_t nmma = (uint32_t)((w.n_cs + 15) & ~15);
            const uint32_t idesc = (1u << 4) | ((nmma >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const bool two = (w.mp * 256 + 128) < p.m;          // second m-tile has rows
            ptx::mbar_wait(bar_dempty, dph ^ 1u);
            ptx::tc_fence_after();
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_afull + 8 * st, ph);
                ptx::mbar_wait(bar_conv + 8 * b, bph);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = sbase + p.off_a + (uint32_t)st * (256u * kKc * 2u);
                    const uint64_t a0 = ptx::smem_desc_swizzled(sa, 128u, 1024u);
                    const uint64_t a1 = ptx::smem_desc_swizzled(sa + 128u * 128u, 128u, 1024u);
                    const uint64_t bd = ptx::smem_desc_swizzled(sbase + kOffB + (uint32_t)b * p.b_bytes, 128u, 1024u);
#pragma unroll
                    for (int ks = 0; ks < kKc / 16; ++ks) {   // K = 16 per MMA: +32 B inside the SW128 rows
                        const uint32_t acc = (kc != w.kc0 || ks != 0) ? 1u : 0u;
                        ptx::mma_f16_ss(tmem_base, a0 + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc, acc);
                        if (two)
                            ptx::mma_f16_ss(tmem_base + 256u, a1 + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc, acc);
                    }
                    ptx::tc_commit(bar_aempty + 8 * st);
                    ptx::tc_commit(bar_bempty + 8 * b);
                    if (kc == w.kc1 - 1) ptx::tc_commit(bar_dfull);
                    ftrace(p, 3, ntr);
                }
                ++ntr;
                __syncwarp();
                if (++st == p.n_a) {
                    st = 0;
                    ph ^= 1u;
                }
                if (++b == p.n_b) {
                    b = 0;
                    bph ^= 1u;
                }
            }
            dph ^= 1u;
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ================================================================ epilogue
        const int ew = warp - kEpiWarp0;   // == warp % 4: TMEM lanes 32 ew .. 32 ew + 31
        const uint32_t lane_bits = (uint32_t)(ew * 32) << 16;
        uint32_t dph = 0;
        for (long long c = c_beg; c < c_end;) {
            FUnit w;
            piece_at(p, c, c_beg, c_end, cid, cmp, w);
            c += w.kc1 - w.kc0;
            ptx::mbar_wait(bar_dfull, dph);
            ptx::tc_fence_after();
            for (int half = 0; half < 2; ++half) {
                const int il = half * 128 + ew * 32 + (int)lane;                 // row within the m-pair
                const int i = w.mp * 256 + il;                                      // measurement index
                if (w.mp * 256 + half * 128 >= p.m) break;                        // warp-uniform
                // whole unit: y rows [cs][m]; a piece of a cut unit: its partial tile [256 CS][256 rows]
                const long long ld = w.slot < 0 ? (long long)p.m : 256LL;
                float* const dst0 = w.slot < 0 ? p.out + ((long long)w.s * p.cs_s + w.cs0) * p.m + i
                                               : p.part + (long long)w.slot * 65536LL + il;
                const uint32_t d_tm = tmem_base + lane_bits + (uint32_t)half * 256u;
                for (int j0 = 0; j0 < w.n_cs; j0 += 32) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)j0, v);
                    ptx::tc_wait_ld();
                    CS_CHECK(i >= p.m || w.slot >= 0 || ((long long)w.s * p.cs_s + w.cs0 + w.n_cs - 1) * p.m + i < p.out_floats);
                    CS_CHECK(w.slot < 2 * n_cl && w.n_cs <= 256);
                    if (i < p.m) {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (j0 + k < w.n_cs) dst0[(long long)(j0 + k) * ld] = __uint_as_float(v[k]);
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar_dempty);
            dph ^= 1u;
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kMmaWarp) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

// Units cut by stream-K range boundaries: y = the sum of their pieces' partial tiles in CTA order
// (deterministic).  Block x handles split unit units[x]; `grid` is the measurement kernel's grid.
struct FixupList {
    int n;
    int grid;
    int units[256];   // <= grid - 1 split units (grid <= SM count)
};
__global__ void __launch_bounds__(64) cs_frame_fixup_kernel(const __grid_constant__ FParams p,
                                                                const __grid_constant__ FixupList L) {
    // block (x, y): split unit units[x], CS frames y, y + gridDim.y, ...; thread: 4 rows of the m-pair
    const int u = L.units[blockIdx.x];
    FUnit w;
    decode_funit(p, u, w);
    const long long gj = L.grid / p.n_mp;
    const long long c0 = (long long)(u / p.n_mp) * p.n_chunks, c1 = c0 + p.n_chunks - 1;
    const int jf = range_of(p, c0, gj), jl = range_of(p, c1, gj);
    constexpr int kMaxPieces = 8;
    long long tile[kMaxPieces];
    const int np = min(kMaxPieces, jl - jf + 1);
    CS_CHECK(jl - jf + 1 <= kMaxPieces);
    for (int k = 0; k < np; ++k) {
        const int j = jf + k, b = j * p.n_mp + w.mp;   // range j's CTA of this m-pair; its first piece iff j starts inside u
        tile[k] = (long long)(2 * b + (cbeg(p, j, gj) >= c0 ? 0 : 1)) * 65536LL;
    }
    const int rows = min(256, p.m - w.mp * 256);
    const int il = (int)threadIdx.x * 4;
    if (il >= rows) return;
    float* const y0 = p.out + ((long long)w.s * p.cs_s + w.cs0) * p.m + (long long)w.mp * 256 + il;
    for (int cs = (int)blockIdx.y; cs < w.n_cs; cs += (int)gridDim.y) {
        float4 a = *reinterpret_cast<const float4*>(p.part + tile[0] + (long long)cs * 256 + il);
        for (int j = 1; j < np; ++j) {   // CTA order: deterministic
            const float4 b = *reinterpret_cast<const float4*>(p.part + tile[j] + (long long)cs * 256 + il);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        float* const yr = y0 + (long long)cs * p.m;
        yr[0] = a.x;
        if (il + 1 < rows) yr[1] = a.y;
        if (il + 2 < rows) yr[2] = a.z;
        if (il + 3 < rows) yr[3] = a.w;
    }
}

}  // namespace frm
}  // namespace csenc
