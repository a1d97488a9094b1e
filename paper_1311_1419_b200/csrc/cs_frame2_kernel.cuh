// cs_frame2_kernel.cuh -- K4b: frame-level measurement on CTA PAIRS with the
// 2-SM tensor-core MMA (tcgen05.mma.cta_group::2).
//
// Same operation as K4 (cs_frame_kernel.cuh): y[cs][i] = sum_j A[i][j] * (F_cs - F_key)[j].  A pair of
// CTAs on one TPC computes D[256 measurements x N CS frames] per K chunk with ONE M=256 MMA per 16-K
// step issued by the pair leader:
//   A (measurement rows): CTA r holds rows 128 r .. 128 r + 127 of the pair's 256-row tile (TMA
//     .cta_group::2: its box lands in its own SMEM, the bytes are counted on the leader's barrier);
//   B (residual of the window's CS frames): CTA r holds rows N/2 r .. N/2 r + N/2 - 1, built by its
//     own converter warps from its own frame box (its half of the window's GOPs);
//   D: CTA r's TMEM holds its 128 measurement rows x all N CS-frame columns.
// Per SM and 64-pixel chunk that is 16 KB of A + ~10 KB of frames for 128 x N x 64 MACs (K4: 32 + 11
// KB for 256 x 140 x 64), and the ~26 KB stages leave room for 7 in flight.
// Signalling: the converters and epilogue warps of both CTAs arrive on the leader's barriers (mapa +
// mbarrier.arrive.release.cluster); the leader's tcgen05.commit multicasts to both CTAs' barriers.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "ptx_sm100.cuh"

namespace csenc {
namespace frm2 {

constexpr int kConvWarps = 8;
constexpr int kEpiWarp0 = 8;
constexpr int kProducerWarp = 12;
constexpr int kMmaWarp = 13;
constexpr int kThreads = 14 * 32;
constexpr int kMaxStages = 8;
constexpr int kKc = 64;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOffB = 1024;                 // n_b residual buffers of b_bytes (this CTA's half)
constexpr int kMaxB = 4;

struct F2Params {
    CUtensorMap fmap;         // frames: 2-D [n_seq*T rows][n bytes], box [nf_box][64], SWIZZLE_64B
    CUtensorMap amap;         // A (permuted): 2-D [m rows][n fp16], box [128][64], SWIZZLE_128B
    float* out;               // y [n_seq*cs_s][m] (n_ks == 1) or partials [n_ks][...][m]
    int n, m, G, T, cs_s;
    int gw2, nf_box;          // GOPs per CTA half of a window (window = 2 * gw2 GOPs), frame rows per box
    int nhalf;                // B rows per CTA (multiple of 8); MMA N = 2 * nhalf
    int global_win, total_gops, n_win_s, n_win;
    int n_mp, n_ks, n_chunks, n_units;   // units are per pair
    uint32_t fbox_bytes, off_a, stage_bytes, b_bytes, off_stage;
    int n_stages;
    int n_b;                  // residual buffers (2..kMaxB): conversion runs n_b - 1 chunks ahead of the MMAs
    long long part_stride, out_floats;
    uint32_t smem_bytes;
    unsigned long long* trace;   // debug timeline (pair 0): [4][trace_cap] clock64, nullptr = off
    int trace_cap;
    int dbg;                  // ablations (timing only, results invalid): 1 no frame loads, 2 no A loads,
                              // 4 A by plain per-CTA TMA onto the local barrier + remote arrive
};

// events: 0 producer issued (leader), 1 leader converters done, 2 MMA saw both A halves, 3 MMA issued
__device__ __forceinline__ void f2trace(const F2Params& p, int ev, int i) {
    if (p.trace != nullptr && blockIdx.x < 2 && i < p.trace_cap) p.trace[(size_t)ev * p.trace_cap + i] = clock64();
}

struct F2Unit {
    int s, g0, n_cs, cs0;     // this CTA's half: stream, first GOP, CS frames, first CS row (global)
    int n_cs_h[2];            // CS frames of both halves (columns [0, nhalf) and [nhalf, 2 nhalf))
    long long cs0_h[2];       // first output CS row of both halves
    int mp, ks, kc0, kc1;
};

__device__ __forceinline__ void decode_half(const F2Params& p, int win, int h, int& s, int& g0, int& n_cs,
                                            long long& cs0) {
    if (win >= p.n_win) {
        s = 0;
        g0 = 0;
        n_cs = 0;
        cs0 = 0;
        return;
    }
    if (p.global_win) {
        s = 0;
        g0 = win * 2 * p.gw2 + h * p.gw2;
        const int ng = max(0, min(p.gw2, p.total_gops - g0));
        n_cs = ng * (p.G - 1);
        cs0 = (long long)g0 * (p.G - 1);
    } else {
        s = win / p.n_win_s;
        const int wi = win - s * p.n_win_s;
        g0 = wi * 2 * p.gw2 + h * p.gw2;
        const int n_gops = (p.T + p.G - 1) / p.G;
        const int ng = max(0, min(p.gw2, n_gops - g0));
        const int t_end = min(p.T, (g0 + ng) * p.G);
        n_cs = ng > 0 ? (t_end - g0 * p.G) - ng : 0;
        cs0 = (long long)s * p.cs_s + (long long)g0 * (p.G - 1);
    }
}

__device__ __forceinline__ void decode_f2(const F2Params& p, int u, int rank, F2Unit& w) {
    w.mp = u % p.n_mp;
    const int r = u / p.n_mp;
    const int win = r % p.n_win;
    w.ks = r / p.n_win;
    const int per = (p.n_chunks + p.n_ks - 1) / p.n_ks;
    w.kc0 = w.ks * per;
    w.kc1 = min(p.n_chunks, w.kc0 + per);
    int s0, g00, n0, s1, g01, n1;
    long long c0, c1;
    decode_half(p, win, 0, s0, g00, n0, c0);
    decode_half(p, win, 1, s1, g01, n1, c1);
    w.n_cs_h[0] = n0;
    w.n_cs_h[1] = n1;
    w.cs0_h[0] = c0;
    w.cs0_h[1] = c1;
    w.s = rank ? s1 : s0;
    w.g0 = rank ? g01 : g00;
    w.n_cs = rank ? n1 : n0;
    w.cs0 = (int)(rank ? c1 : c0);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    cs_frame2_kernel(const __grid_constant__ F2Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const int rank = (int)ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = (int)blockIdx.x / 2, n_cl = (int)gridDim.x / 2;

    const uint32_t bar_fullF = sbase;                       // [8] frames box landed (local)
    const uint32_t bar_fullA = sbase + 8 * kMaxStages;      // [8] both A halves landed (leader)
    const uint32_t bar_empty = sbase + 16 * kMaxStages;     // [8] stage free (both, multicast commit)
    const uint32_t bar_conv = sbase + 24 * kMaxStages;      // [kMaxB] both halves' residual written (leader)
    const uint32_t bar_bempty = bar_conv + 8 * kMaxB;       // [kMaxB] residual buffer free (both)
    const uint32_t bar_dfull = bar_bempty + 8 * kMaxB;      // [2] accumulator ready (both)
    const uint32_t bar_dempty = bar_dfull + 16;             // [2] accumulator drained by both epilogues (leader)
    const uint32_t tmem_slot = bar_dempty + 16;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(bar_fullF + 8 * i, 1);
            ptx::mbar_init(bar_fullA + 8 * i, 1);
            ptx::mbar_init(bar_empty + 8 * i, 1);
        }
        for (int i = 0; i < kMaxB; ++i) {
            ptx::mbar_init(bar_conv + 8 * i, 2 * kConvWarps);
            ptx::mbar_init(bar_bempty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_dfull + 8 * i, 1);
            ptx::mbar_init(bar_dempty + 8 * i, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {   // the same warp in both CTAs: pair allocation
        ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
        ptx::tmem_relinquish_2sm();
    }
    if (warp == kProducerWarp && lane == 0) {
        ptx::prefetch_tmap(&p.fmap);
        ptx::prefetch_tmap(&p.amap);
    }
    CS_CHECK(p.off_stage + (uint32_t)p.n_stages * p.stage_bytes <= p.smem_bytes && p.n_stages <= kMaxStages);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));
    const uint32_t lead_conv = ptx::mapa(bar_conv, 0);
    const uint32_t lead_dempty = ptx::mapa(bar_dempty, 0);

    if (warp == kProducerWarp) {
        // ================================================================ producer (both CTAs)
        int st = 0, ntr = 0;
        uint32_t ph = 0;
        for (int u = cid; u < p.n_units; u += n_cl) {
            F2Unit w;
            decode_f2(p, u, rank, w);
            const int row0 = w.s * p.T + w.g0 * p.G;
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_empty + 8 * st, ph ^ 1u);
                if (lane == 0) {
                    const uint32_t sf = sbase + p.off_stage + (uint32_t)st * p.stage_bytes;
                    const bool has = w.n_cs > 0 && !(p.dbg & 1);
                    ptx::mbar_arrive_expect_tx(bar_fullF + 8 * st, has ? p.fbox_bytes : 0u);
                    if (has) ptx::tma_load_2d(sf, &p.fmap, bar_fullF + 8 * st, kc * kKc, row0);
                    if (p.dbg & 2) {
                        if (leader) ptx::mbar_arrive(bar_fullA + 8 * st);
                    } else {
                        if (leader) ptx::mbar_arrive_expect_tx(bar_fullA + 8 * st, 2u * 128u * kKc * 2u);
                        ptx::tma_load_2d_2sm(sf + p.off_a, &p.amap, bar_fullA + 8 * st, kc * kKc, w.mp * 256 + rank * 128);
                    }
                    if (leader) f2trace(p, 0, ntr);
                }
                ++ntr;
                __syncwarp();
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp < kConvWarps) {
        // ================================================================ residual half (both CTAs)
        const int tid = (int)threadIdx.x;
        const int q = tid & 7;
        uint32_t rows[4];   // this CTA's B rows c = tid/8 + 32 i (i < 4): nhalf <= 128
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = (tid >> 3) + 32 * i;
            const int gl = c / (p.G - 1), pos = c - gl * (p.G - 1);
            rows[i] = (uint32_t)(gl * p.G + 1 + pos) | ((uint32_t)(gl * p.G) << 16);
        }
        int st = 0, b = 0, ntr = 0;
        uint32_t ph = 0, bph = 0;
        for (int u = cid; u < p.n_units; u += n_cl) {
            F2Unit w;
            decode_f2(p, u, rank, w);
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_fullF + 8 * st, ph);
                ptx::mbar_wait(bar_bempty + 8 * b, bph ^ 1u);
                if (tid == 0 && rank == 0) f2trace(p, 2, ntr);   // conversion starts
                const uint32_t sf = sbase + p.off_stage + (uint32_t)st * p.stage_bytes;
                const uint32_t sb = sbase + kOffB + (uint32_t)b * p.b_bytes;
                uint2 fv[4], kv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = (tid >> 3) + 32 * i;
                    const uint32_t rr = c < w.n_cs ? rows[i] : 0u;
                    const uint32_t t = rr & 0xFFFFu, k = rr >> 16;
                    const uint32_t ct = t * 64u + ((((uint32_t)(q >> 1)) ^ ((t >> 1) & 3u)) << 4) + (uint32_t)(q & 1) * 8u;
                    const uint32_t ck = k * 64u + ((((uint32_t)(q >> 1)) ^ ((k >> 1) & 3u)) << 4) + (uint32_t)(q & 1) * 8u;
                    fv[i] = ptx::lds64(sf + ct);
                    kv[i] = ptx::lds64(sf + ck);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = (tid >> 3) + 32 * i;
                    if (c < w.n_cs) {
                        CS_CHECK((rows[i] & 0xFFFFu) < (uint32_t)p.nf_box && (uint32_t)(c + 1) * 128u <= p.b_bytes);
                        uint32_t w0, w1, w2, w3;
                        ptx::residual4(fv[i].x, kv[i].x, w0, w1);
                        ptx::residual4(fv[i].y, kv[i].y, w2, w3);
                        ptx::sts128(sb + (uint32_t)c * 128u + ((uint32_t)(q ^ (c & 7)) << 4), w0, w1, w2, w3);
                    }
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (leader)
                        ptx::mbar_arrive(bar_conv + 8 * b);                       // local barrier
                    else
                        ptx::mbar_arrive_cluster(lead_conv + 8u * (uint32_t)b);   // release at cluster scope
                }
                if (tid == 0 && rank == 0) f2trace(p, 1, ntr);
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
    } else if (warp == kMmaWarp && leader) {
        // ================================================================ MMA issuer (pair leader)
        const uint32_t nmma = (uint32_t)(2 * p.nhalf);
        const uint32_t idesc = (1u << 4) | ((nmma >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
        int st = 0, b = 0, db = 0, ntr = 0;
        uint32_t ph = 0, bph = 0, dph = 0;
        for (int u = cid; u < p.n_units; u += n_cl) {
            F2Unit w;
            decode_f2(p, u, rank, w);
            ptx::mbar_wait_cluster(bar_dempty + 8 * db, dph ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d_tm = tmem_base + (uint32_t)db * 256u;
            for (int kc = w.kc0; kc < w.kc1; ++kc) {
                ptx::mbar_wait(bar_fullA + 8 * st, ph);
                ptx::mbar_wait_cluster(bar_conv + 8 * b, bph);   // the peer's half: release.cluster arrivals
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = sbase + p.off_stage + (uint32_t)st * p.stage_bytes + p.off_a;
                    const uint64_t ad = ptx::smem_desc_swizzled(sa, 128u, 1024u);
                    const uint64_t bd = ptx::smem_desc_swizzled(sbase + kOffB + (uint32_t)b * p.b_bytes, 128u, 1024u);
#pragma unroll
                    for (int ks = 0; ks < kKc / 16; ++ks)
                        ptx::mma_f16_ss_2sm(d_tm, ad + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc,
                                            (kc != w.kc0 || ks != 0) ? 1u : 0u);
                    ptx::tc_commit_2sm_mc(bar_empty + 8 * st, 0x3);
                    ptx::tc_commit_2sm_mc(bar_bempty + 8 * b, 0x3);
                    if (kc == w.kc1 - 1) ptx::tc_commit_2sm_mc(bar_dfull + 8 * db, 0x3);
                    f2trace(p, 3, ntr);
                }
                ++ntr;
                __syncwarp();
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
                if (++b == p.n_b) {
                    b = 0;
                    bph ^= 1u;
                }
            }
            if (++db == 2) {
                db = 0;
                dph ^= 1u;
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ================================================================ epilogue (both CTAs)
        const int ew = warp - kEpiWarp0;   // == warp % 4: TMEM lanes 32 ew .. 32 ew + 31
        const uint32_t lane_bits = (uint32_t)(ew * 32) << 16;
        int db = 0;
        uint32_t dph = 0;
        for (int u = cid; u < p.n_units; u += n_cl) {
            F2Unit w;
            decode_f2(p, u, rank, w);
            ptx::mbar_wait(bar_dfull + 8 * db, dph);
            ptx::tc_fence_after();
            const int i = w.mp * 256 + rank * 128 + ew * 32 + (int)lane;   // measurement row of this lane
            const uint32_t d_tm = tmem_base + lane_bits + (uint32_t)db * 256u;
            if (w.mp * 256 + rank * 128 < p.m) {   // this CTA's 128 rows exist (warp-uniform)
                for (int h = 0; h < 2; ++h) {
                    float* const dst0 = p.out + (long long)w.ks * p.part_stride + w.cs0_h[h] * p.m + i;
                    const int nh = w.n_cs_h[h];
                    for (int j0 = 0; j0 < nh; j0 += 32) {
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)(h * p.nhalf + j0), v);
                        ptx::tc_wait_ld();
                        CS_CHECK(i >= p.m || (w.cs0_h[h] + nh - 1) * p.m + i < p.out_floats);
                        if (i < p.m) {
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (j0 + k < nh) dst0[(long long)(j0 + k) * p.m] = __uint_as_float(v[k]);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(lead_dempty + 8u * (uint32_t)db);
            if (++db == 2) {
                db = 0;
                dph ^= 1u;
            }
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();   // no CTA exits (or frees TMEM) while the pair still works
    ptx::tc_fence_after();
    if (warp == kMmaWarp) ptx::tmem_dealloc_2sm(tmem_base, kTmemCols);
}

}  // namespace frm2
}  // namespace csenc
