// cs_encoder.cu -- libcsenc.so, the north-star path (K1): planner, launch and the C ABI of the
// block-based encoder (create/destroy, autotune, encode calls and their f1 / f4 variants, the
// host-buffer pipeline, CR accounting).  The f2 / f3 / f4-codec host code is in cs_frame.cu,
// cs_adjoint.cu and cs_keys.cu; shared declarations in cs_internal.h.
//
// Host logic only; the device work is the kernel in cs_measure_kernel.cuh.  No CPU fallback exists:
// every encode runs the sm_100a kernel or returns an error.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "cs_internal.h"
#include "cs_measure_kernel.cuh"

using csenc::KParams;

#ifndef CSENC_SWIZZLE_DEFAULT
#define CSENC_SWIZZLE_DEFAULT 1   // KEY_CHUNK strips through the 128-B-swizzled 5-D box when the shape allows
#endif

namespace csenc {
namespace host {

// key_mode: 0 = key strip streamed with every item, 1 = resident in SMEM (double-buffered),
//           2 = in converter registers (arrives once per unit through a ring slot),
//           3 = chunk-outer order (KEY_CHUNK): per K-chunk the key chunk arrives once through a ring
//               slot into converter registers and every CS frame of the unit follows against it, each
//               into its own TMEM accumulator (unit frames <= n_dbuf); Phi resident, or (phi_stream)
//               its K-slice loaded once per chunk into a double-buffered region.
// a_pref (key_mode 3 only): TMEM A-operand buffers; the rest of TMEM goes to accumulators.
bool try_plan(const Geometry& g, int T_r, int chunk_rows, int key_mode, int smem_limit, Plan& p, int phi_stream = 0,
              int a_pref = 2) {
    const bool key_res = key_mode == 1;
    const bool key_chunk = key_mode == 3;
    p = Plan();
    const int words = g.B / 2;          // fp16x2 columns per pixel row
    const int rows_per_st = 32 / words;
    if (g.B % chunk_rows != 0 || chunk_rows % rows_per_st != 0) return false;
    if ((chunk_rows * g.B) % 16 != 0) return false;
    if (key_chunk && g.B != 32) return false;   // instantiated for B = 32 (the config it exists for: C3)
    const int tile_blocks = T_r * g.nbx;
    p.T_r = T_r;
    p.F = cdiv(tile_blocks, 128);
    if (p.F > csenc::kMaxFolds) return false;
    p.L = cdiv(tile_blocks, p.F);
    p.n_tiles = cdiv(g.nby, T_r);
    p.chunk_rows = chunk_rows;
    p.n_chunks = g.B / chunk_rows;
    p.chunk_k = chunk_rows * g.B;
    p.a_cols = p.F * p.chunk_k / 2;
    p.d_cols = p.F * g.Mpad;
    // TMEM rings: A buffers (converter -> MMA) and accumulators (MMA -> epilogue).  Deeper rings
    // decouple the converter and epilogue latencies (measured: with 2+2 a slow converter OR a
    // slow epilogue stalls the chain).  Prefer (3+, 3+), then (2, 2).  (Dependent MMAs into one
    // accumulator issue back to back -- tools/mma_microbench*.cu -- so no split-K chains.)
    // KEY_CHUNK: a_pref A buffers and as many accumulators as fit (they bound the unit's frames).
    if (key_chunk) {
        p.n_abuf = a_pref;
        p.n_dbuf = std::min(csenc::kMaxTmemBufs, ((int)csenc::kTmemCols - a_pref * p.a_cols) / p.d_cols);
        if (p.n_dbuf < 2) return false;
    } else {
        const int dc = p.d_cols;
        const int cands[][2] = {{4, 4}, {4, 3}, {3, 4}, {3, 3}, {4, 2}, {3, 2}, {2, 3}, {2, 2}, {2, 1}, {1, 1}};
        p.n_abuf = 0;
        for (auto& c : cands)
            if (c[0] * p.a_cols + c[1] * dc <= (int)csenc::kTmemCols) {
                p.n_abuf = c[0];
                p.n_dbuf = c[1];
                break;
            }
        if (p.n_abuf == 0) return false;
#if CSENC_TUNING
        if (const char* e = std::getenv("CSENC_TMEM_BUFS")) {  // experiment knob "A,D"
            int a = 0, d = 0;
            if (std::sscanf(e, "%d,%d", &a, &d) == 2 && a >= 1 && d >= 1 && a <= 4 && d <= 4 &&
                a * p.a_cols + d * dc <= (int)csenc::kTmemCols) {
                p.n_abuf = a;
                p.n_dbuf = d;
            }
        }
#endif
    }
    p.tmem_cols = p.n_abuf * p.a_cols + p.n_dbuf * p.d_cols;
    if (p.tmem_cols > (int)csenc::kTmemCols) return false;
    const double ring_q = std::min(p.n_abuf, 3) * std::min(p.n_dbuf, 3) / 9.0;  // prefer 3+3
    // Stage layout: [piece][piece_rows][W] -- each piece is one contiguous strip of full-width
    // frame rows, moved by a single bulk copy.
    if (p.n_chunks == 1) {
        p.pieces = 1;
        p.single_piece = 1;
        p.piece_rows = T_r * g.B;
    } else {
        p.pieces = T_r;
        p.piece_rows = chunk_rows;
    }
    p.piece_bytes = align_up((uint32_t)(p.piece_rows * g.W), 128);
    p.stage_cs_bytes = (uint32_t)p.pieces * p.piece_bytes;
    p.key_resident = key_res ? 1 : 0;
    p.key_regs = key_mode == 2 ? 1 : 0;
    p.key_chunk = key_chunk ? 1 : 0;
    const int groups_per_fold = chunk_rows / rows_per_st;
    if (p.key_regs || key_chunk) {
        // each converter warpgroup holds <= 2 row groups (16 u8 words each) of the key
        if (p.F * groups_per_fold > 4) return false;
        if (p.key_regs && (g.B == 32 || p.n_chunks != 1)) return false;
    }
    p.key_bytes = key_res ? (uint32_t)p.n_chunks * p.stage_cs_bytes : 0;
    p.stage_bytes = (key_res || p.key_regs || key_chunk) ? p.stage_cs_bytes : 2 * p.stage_cs_bytes;
    uint32_t phi_bytes = (uint32_t)g.Mpad * (uint32_t)g.N * 2u;
    if (phi_stream) {
        if (p.n_chunks < 2 || p.key_regs || key_res) return false;
        p.phi_stream = 1;
        p.phi_slice_bytes = phi_bytes / (uint32_t)p.n_chunks;
        if (key_chunk) {
            // the chunk's K-slice of Phi: once per (unit, chunk) into a double-buffered region (at off_key)
            p.key_bytes = align_up(p.phi_slice_bytes, 1024);
        } else {
            // Phi's K-slice for the chunk rides in every stage (the canonical layout keeps a chunk's
            // chunk_k / 8 K-groups contiguous); nothing of Phi stays resident
            p.stage_phi_off = align_up(p.stage_bytes, 128);
            p.stage_bytes = align_up(p.stage_phi_off + p.phi_slice_bytes, 128);
        }
        phi_bytes = 0;
    }
    p.off_tab = 1024;  // barriers live in the first KB, then the converter offset table (1 KB per fold)
    p.off_epi = 1024 + (uint32_t)p.F * 1024u;  // epilogue staging tiles (4 warps x 4 KB)
    p.off_phi = p.off_epi + 16384;
    p.off_key = align_up(p.off_phi + phi_bytes, 1024);
    p.off_stage = align_up(p.off_key + 2 * p.key_bytes, 1024);
    const long avail = (long)smem_limit - 1024 /*alignment slack*/ - (long)p.off_stage;
    if (avail < (long)p.stage_bytes * 2) return false;
    p.n_stages = (int)std::min<long>(csenc::kMaxStages, avail / p.stage_bytes);
    if (key_chunk && p.n_stages < 3) return false;   // key item + at least two frames in flight
    p.smem_bytes = p.off_stage + (uint32_t)p.n_stages * p.stage_bytes + 1024;
    p.prefetch_items = 0;  // (L2 prefetch of future strips measured no benefit; kept in the plan info as 0)
    // Score = modelled pixels per cycle of one SM, calibrated on B200 measurements
    // (tools/trace_timeline.py, tools/sweep*.sh): an item costs a fixed ~700
    // cycles of pipeline handoffs plus ~150 per bulk copy, overlapped with the slowest of
    //   converters ~350 cycles per row group per warpgroup, loads at ~32 B/cycle,
    //   MMA issue ~48 cycles per tcgen05.mma.
    const int groups_per_wg = (p.F * groups_per_fold + 1) / 2;
    const double px = (double)tile_blocks * p.chunk_k;
    const double item_bytes = (double)p.stage_bytes;
    const bool box = p.pieces > 1 && !p.key_regs && !key_res && g.H % g.B == 0;   // 4-D TMA strips
    const int strip_copies = box ? 1 : p.pieces;
    const int copies = strip_copies * ((key_res || p.key_regs || key_chunk) ? 1 : 2) + (key_chunk ? 0 : p.phi_stream);
    const double conv = 350.0 * groups_per_wg;
    const double load = item_bytes / 32.0;
    const double mma = (double)(p.chunk_k / 16) * p.F * std::max(48.0, g.Mpad / 2.0);
    const double cycles = 700.0 + 150.0 * copies + std::max({conv, load, mma});
    double s = px / cycles;
    if (key_chunk) {   // one key item per chunk, amortised over the unit's frames (<= n_dbuf of G-1)
        const double U = std::max(1, std::min(p.n_dbuf, g.G - 1));
        const double key_item = 700.0 + 150.0 * strip_copies + (double)p.stage_cs_bytes / 32.0;
        s = px * U / (U * cycles + key_item);
    }
    // Measured (round 1, a forced-plan sweep since removed): with >= 3 ring slots the double-buffered SMEM key is ~5% faster
    // than the register key (whose load sits in the ring at every unit start); the register key
    // wins when a resident key would leave < 3 slots (C5).
    // B = 8 rows are 8-byte loads, so dropping the per-item key loads matters more there.
    if (p.key_regs) s *= (g.B == 8) ? 1.05 : 0.9;
    if (p.n_stages < 3) s *= 0.85;
    if (p.n_dbuf < 2) s *= 0.8;
    if (!key_chunk) s *= 0.85 + 0.15 * ring_q;
    p.score = s;
    return true;
}

// All feasible plans, best model score first (the autotuner times the first few).
std::vector<Plan> plan_candidates(const Geometry& g, int smem_limit) {
    std::vector<Plan> all;
    // experiment knobs (tools/sweep.sh): force a tile-row count / chunk size / key residency
    const int f_tr = env_int("CSENC_TILE_ROWS", 0), f_cr = env_int("CSENC_CHUNK_ROWS", 0);
    const int f_kr = env_int("CSENC_KEY_RESIDENT", -1), f_st = env_int("CSENC_STAGES", 0);
    const int f_ps = env_int("CSENC_PHI_STREAM", -1);
    for (int T_r = 1; T_r <= g.nby; ++T_r) {
        if (T_r * g.nbx > 128 * csenc::kMaxFolds) break;
        if (f_tr && T_r != f_tr) continue;
        for (int cr = g.B; cr >= 1; --cr) {
            if (f_cr && cr != f_cr) continue;
            for (int kr = 3; kr >= 0; --kr) {
                if (f_kr >= 0 && kr != f_kr) continue;
                for (int ps = 0; ps <= 1; ++ps) {
                    if (f_ps >= 0 && ps != f_ps) continue;
                    for (int ap = 2; ap <= (kr == 3 ? 3 : 2); ++ap) {
                        Plan p;
                        if (!try_plan(g, T_r, cr, kr, smem_limit, p, ps, ap)) continue;
                        if (f_st > 0 && f_st < p.n_stages) {
                            p.smem_bytes -= (uint32_t)(p.n_stages - f_st) * p.stage_bytes;
                            p.n_stages = f_st;
                        }
                        all.push_back(p);
                    }
                }
            }
        }
    }
    std::stable_sort(all.begin(), all.end(), [](const Plan& a, const Plan& b) { return a.score > b.score; });
    return all;
}

bool make_plan(const Geometry& g, int smem_limit, Plan& best) {
    std::vector<Plan> all = plan_candidates(g, smem_limit);
    if (all.empty()) return false;
    best = all[0];
    return true;
}

struct WorkSplit {
    int n_splits, cs_per_unit, n_units;
};

WorkSplit choose_split(const Geometry& g, const Plan& p, int n_seq, int n_gops_sel, int sms) {
    const long base = (long)n_seq * n_gops_sel * p.n_tiles;
    WorkSplit best{1, std::max(1, g.G - 1), (int)base};
    if (g.G <= 1) return best;
    double best_cost = 1e300;
    const double key_cost = (p.key_resident || p.key_regs || p.key_chunk) ? 1.0 : 0.0;
    if (p.key_chunk) best = WorkSplit{cdiv(g.G - 1, p.n_dbuf), p.n_dbuf, (int)(base * cdiv(g.G - 1, p.n_dbuf))};
    for (int ns = 1; ns <= g.G - 1; ++ns) {
        int cpu = cdiv(g.G - 1, ns);
        if (ns > 1 && cdiv(g.G - 1, cpu) != ns) continue;  // identical to a smaller ns
        if (p.key_chunk && cpu > p.n_dbuf) continue;        // a unit's frames each own an accumulator
        long units = base * ns;
        if (units > (1L << 30)) break;
        double rounds = std::ceil((double)units / sms);
        double cost = rounds * (cpu + key_cost);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = WorkSplit{ns, cpu, (int)units};
        }
    }
    return best;
}

int validate(int W, int H, int gop, int B, int M, const uint16_t* phi) {
    if (W < 1 || H < 1 || gop < 1 || M < 1) return fail(CS_ERR_ARG, "W, H, gop and M must be >= 1");
    if (B != 8 && B != 16 && B != 32) return fail(CS_ERR_UNSUPPORTED, "B must be 8, 16 or 32");
    if (M > B * B) return fail(CS_ERR_ARG, "M must be <= N = B*B");
    if (M > 256) return fail(CS_ERR_UNSUPPORTED, "M must be <= 256 (UMMA N limit)");
    if (W % 16 != 0) return fail(CS_ERR_UNSUPPORTED, "W must be a multiple of 16 (16-byte aligned bulk-copy rows)");
    if ((long long)W * H > (1LL << 31)) return fail(CS_ERR_UNSUPPORTED, "frame too large");
    if (phi) {
        for (long i = 0; i < (long)M * B * B; ++i) {
            float v = half_bits_to_float(phi[i]);
            if (!std::isfinite(v) || std::fabs(v) > 2048.0f)
                return fail(CS_ERR_PHI, "Phi entries must be finite with |Phi| <= 2048");
        }
    }
    return CS_OK;
}

Geometry make_geometry(int W, int H, int gop, int B, int M) {
    Geometry g;
    g.W = W;
    g.H = H;
    g.G = gop;
    g.B = B;
    g.M = M;
    g.N = B * B;
    g.Mpad = std::max(16, (M + 15) / 16 * 16);
    g.nbx = cdiv(W, B);
    g.nby = cdiv(H, B);
    g.nblk = g.nbx * g.nby;
    return g;
}

double cr_formula(const Geometry& g, int T, double key_cr, int bits) {
    if (T == 0) T = g.G;
    const long long n_key = cdiv(T, g.G);
    const long long n_cs = (long long)T - n_key;
    const double orig = (double)T * g.W * g.H * 8.0;
    const double key_bits = (double)n_key * g.W * g.H * 8.0 / key_cr;
    const double meas_bits = (double)n_cs * g.nblk * g.M * (double)bits;
    return orig / (key_bits + meas_bits);
}

}  // namespace host
}  // namespace csenc

// ====================================================================================== encoder
using namespace csenc::host;

namespace {

// f1 epilogue arguments (qmode 0 = fp32 output)
struct QArgs {
    const uint8_t* keys = nullptr;   // f4: decoded key frames [n_seq][ceil(T/G)][H][W]
    int chained = 0;                 // f4 variant: previous-frame reference (needs a KEY_STREAMED plan)
    const Plan* plan = nullptr;      // plan override (default e->plan)
    int qmode = 0;
    int16_t* codes = nullptr;
    uint32_t* amax = nullptr;
    float* scales = nullptr;
};

int launch(cs_encoder* e, const uint8_t* frames, int n_seq, int T, int g0, int g1, float* out, cudaStream_t stream,
           const QArgs& q = QArgs()) {
    const Geometry& g = e->geo;
    const Plan& pl = q.plan ? *q.plan : e->plan;
    if (g1 <= g0 || g.G == 1) return CS_OK;
    if (cs_frames_in_gops(T, g.G, g0, g1) == 0) return CS_OK;
    KParams kp;
    std::memset(&kp, 0, sizeof(kp));
    kp.frames = frames;
    kp.zeros = (const uint8_t*)e->zeros_dev;
    kp.out = out;
    kp.W = g.W;
    kp.H = g.H;
    kp.phi = (const uint16_t*)e->phi_dev;
    kp.phi_bytes = e->phi_bytes;
    kp.M = g.M;
    kp.Mpad = g.Mpad;
    kp.N = g.N;
    kp.nbx = g.nbx;
    kp.nby = g.nby;
    kp.nblk = g.nblk;
    kp.T_r = pl.T_r;
    kp.F = pl.F;
    kp.L = pl.L;
    kp.Lq = env_int("CSENC_LANE_SPREAD", 1) ? (pl.L + 3) / 4 : 32;   // spread the tile's lanes over the 4 quarters
    kp.n_tiles = pl.n_tiles;
    kp.chunk_rows = pl.chunk_rows;
    kp.n_chunks = pl.n_chunks;
    kp.chunk_k = pl.chunk_k;
    kp.pieces = pl.pieces;
    kp.piece_rows = pl.piece_rows;
    kp.single_piece = pl.single_piece;
    kp.piece_bytes = pl.piece_bytes;
    kp.set_bytes = (uint32_t)pl.pieces * (uint32_t)pl.piece_rows * (uint32_t)g.W;
    kp.smem_bytes = pl.smem_bytes - 1024;
    kp.out_floats = (long long)n_seq * cs_frames_in_gops(T, g.G, g0, g1) * g.nblk * g.M;
    kp.frames_bytes = (long long)n_seq * T * g.W * g.H;
    kp.stage_cs_bytes = pl.stage_cs_bytes;
    kp.phi_stream = pl.phi_stream;
    kp.phi_slice_bytes = pl.phi_slice_bytes;
    kp.stage_phi_off = pl.stage_phi_off;
    kp.stage_bytes = pl.stage_bytes;
    kp.key_bytes = pl.key_bytes;

    kp.n_stages = pl.n_stages;
    kp.off_phi = pl.off_phi;
    kp.off_key = pl.off_key;
    kp.off_stage = pl.off_stage;
    kp.G = g.G;
    kp.T = T;
    kp.gop_begin = g0;
    kp.n_gops_sel = g1 - g0;
    kp.cs_per_stream_sel = (int)cs_frames_in_gops(T, g.G, g0, g1);
    {
        WorkSplit ws = choose_split(g, pl, n_seq, g1 - g0, e->sms);
        kp.n_splits = ws.n_splits;
        kp.cs_per_unit = ws.cs_per_unit;
        kp.n_units = ws.n_units;
    }
    kp.idesc = e->idesc;
    kp.lbo = e->lbo;
    kp.sbo = e->sbo;
    kp.a_cols = pl.a_cols;
    kp.d_cols = pl.d_cols;
    kp.n_abuf = pl.n_abuf;
    kp.n_dbuf = pl.n_dbuf;
    kp.off_tab = pl.off_tab;
    kp.off_epi = pl.off_epi;
    kp.dbg_load_only = env_int("CSENC_DBG_LOAD_ONLY", 0);
    kp.dbg_flags = env_int("CSENC_DBG_FLAGS", 0);
    kp.trace = e->trace;
    kp.trace_cap = e->trace_cap;
    // loads before the previous kernel completes: only when the caller vouches for the inputs, and never when
    // the keys come from the key-codec kernel or a trace buffer is shared between launches
    kp.pdl_early = ((e->stable_inputs & CS_STABLE_FRAMES) && q.keys == nullptr && e->trace == nullptr) ? 1 : 0;
    kp.keys = q.keys;
    kp.keys_bytes = (long long)n_seq * cdiv(T, g.G) * g.W * g.H;
    kp.chained = q.chained;
    kp.phis = (const uint16_t*)e->phis_dev;
    kp.n_phis = e->n_phis;
    // per-GOP Phi resident in SMEM: a second slot behind the ring (one stage fewer if it does not fit), so the
    // next GOP's matrix loads while the current one is in use
    uint32_t smem_launch = pl.smem_bytes;
    kp.off_phi2 = 0;
    if (e->n_phis > 0 && !pl.phi_stream) {
        for (int ns = pl.n_stages; ns >= std::max(2, pl.n_stages - 1) && kp.off_phi2 == 0; --ns) {
            const uint32_t off2 = align_up(pl.off_stage + (uint32_t)ns * pl.stage_bytes, 1024);
            if (off2 + e->phi_bytes + 1024 <= (uint32_t)e->smem_limit) {
                kp.off_phi2 = off2;
                kp.n_stages = ns;
                smem_launch = off2 + e->phi_bytes + 1024;
            }
        }
    }
    kp.smem_bytes = smem_launch - 1024;
    kp.n_gops_T = cdiv(T, g.G);
    kp.qmode = q.qmode;
    kp.codes = q.codes;
    kp.amax = q.amax;
    kp.scales = q.scales;
    // multi-piece strips by one 4-D TMA box (H % B == 0 so block rows never run into the next frame;
    // the box's inner extent W/4 u32 words <= 256; pieces packed back to back in the stage)
    csenc::KParamsTS kpt;
    std::memset(&kpt, 0, sizeof(kpt));
    static_cast<KParams&>(kpt) = kp;
    if (!pl.key_regs && !pl.key_resident && pl.pieces > 1 && !pl.single_piece && g.H % g.B == 0 && g.W % 4 == 0 && g.W / 4 <= 256 &&
        pl.piece_bytes == (uint32_t)(pl.piece_rows * g.W) && env_int("CSENC_TMA_STRIPS", 1)) {
        PFN_encodeTiled enc = get_encode_tiled();
        if (enc) {
            cuuint64_t dims[4] = {(cuuint64_t)(g.W / 4), (cuuint64_t)g.B, (cuuint64_t)g.nby, (cuuint64_t)n_seq * T};
            cuuint64_t strides[3] = {(cuuint64_t)g.W, (cuuint64_t)g.B * g.W, (cuuint64_t)g.H * g.W};
            cuuint32_t box[4] = {(cuuint32_t)(g.W / 4), (cuuint32_t)pl.chunk_rows, (cuuint32_t)pl.T_r, 1u};
            cuuint32_t estr[4] = {1, 1, 1, 1};
            CUresult r = enc(&kpt.smap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint8_t*>(frames), dims, strides,
                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            kpt.tma_strips = (r == CUDA_SUCCESS && pl.T_r <= 256) ? 1 : 0;
            // KEY_CHUNK (B = 32), W a multiple of 128 and 1024-B stages: the same box as 128-B lines
            // [W/128][128 B] written with the 128-B swizzle, so the converters' reads of 32-B block rows
            // are free of bank conflicts (the SMEM image is the 4-D box's with chunk c of line L at c ^ (L & 7))
            // (decoded keys, f4, come from another buffer by plain bulk copies: unswizzled)
            if (kpt.tma_strips && pl.key_chunk && q.keys == nullptr && g.W % 128 == 0 && pl.stage_bytes % 1024 == 0 &&
                pl.off_stage % 1024 == 0 && env_int("CSENC_SWIZZLE", CSENC_SWIZZLE_DEFAULT)) {
                cuuint64_t dims5[5] = {32, (cuuint64_t)(g.W / 128), (cuuint64_t)g.B, (cuuint64_t)g.nby, (cuuint64_t)n_seq * T};
                cuuint64_t strides5[4] = {128, (cuuint64_t)g.W, (cuuint64_t)g.B * g.W, (cuuint64_t)g.H * g.W};
                cuuint32_t box5[5] = {32, (cuuint32_t)(g.W / 128), (cuuint32_t)pl.chunk_rows, (cuuint32_t)pl.T_r, 1u};
                cuuint32_t estr5[5] = {1, 1, 1, 1, 1};
                CUtensorMap m5;
                r = enc(&m5, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<uint8_t*>(frames), dims5, strides5, box5, estr5,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r == CUDA_SUCCESS) {
                    kpt.smap = m5;
                    kpt.tma_strips = 2;
                }
            }
        }
    }
#if CSENC_CHECKS
    {   // race gate: random delays after mbarrier waits (ptx::stress_point), seed from CSENC_STRESS
        static const unsigned int stress = [] {
            const char* v = std::getenv("CSENC_STRESS");
            return v ? (unsigned int)std::strtoul(v, nullptr, 10) : 0u;
        }();
        static std::once_flag once;
        std::call_once(once, [] { cudaMemcpyToSymbol(csenc::ptx::g_csenc_stress, &stress, sizeof(stress)); });
    }
#endif
    int grid = std::max(1, std::min(e->sms, kp.n_units));
    cudaError_t err, launch_err = cudaSuccess;
    const int km = pl.key_chunk ? csenc::KEY_CHUNK
                   : pl.key_regs ? csenc::KEY_REGS : (pl.key_resident ? csenc::KEY_RESIDENT : csenc::KEY_STREAMED);
    // KEY_STREAMED / KEY_CHUNK kernels take KParamsTS (with the strip tensor map), the others KParams
    auto go = [&](auto kern) {
        // launched with programmatic stream serialization: the kernel's prologue may overlap the tail of
        // the stream's previous kernel (it waits, griddepcontrol.wait, before touching global memory)
        auto run = [&](auto& prm) {
            cudaLaunchConfig_t cfg;
            std::memset(&cfg, 0, sizeof(cfg));
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3((unsigned)(km == csenc::KEY_CHUNK ? csenc::kThreadsChunk : csenc::kThreads));
            cfg.dynamicSmemBytes = smem_launch;
            cfg.stream = stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = CSENC_PDL ? 1 : 0;
            launch_err = cudaLaunchKernelEx(&cfg, kern, prm);
        };
        if constexpr (std::is_invocable_v<decltype(kern), const csenc::KParamsTS&> &&
                      !std::is_invocable_v<decltype(kern), const csenc::KParams&>)
            run(kpt);
        else
            run(kp);
    };
    int epi = q.qmode ? csenc::EPI_Q16 : csenc::EPI_F32;
    if (q.qmode == csenc::Q_STOREMAX) epi = csenc::EPI_F32A;
    if (q.qmode == csenc::Q_ROW)
        epi = (pl.F != 1 || g.Mpad != g.M || pl.T_r > csenc::kRowRegRows || g.Mpad > 64) ? csenc::EPI_Q16R
              : g.Mpad <= 32 ? csenc::EPI_Q16RR : csenc::EPI_Q16RR64;
#define CSENC_CASE(B_, K_)                                                                                \
    case (B_ * 4 + K_) * 8 + csenc::EPI_F32: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_F32>); break;   \
    case (B_ * 4 + K_) * 8 + csenc::EPI_Q16: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16>); break;   \
    case (B_ * 4 + K_) * 8 + csenc::EPI_Q16R: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16R>); break; \
    case (B_ * 4 + K_) * 8 + csenc::EPI_Q16RR: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16RR>); break; \
    case (B_ * 4 + K_) * 8 + csenc::EPI_Q16RR64: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16RR64>); break; \
    case (B_ * 4 + K_) * 8 + csenc::EPI_F32A: go(csenc::cs_measure_kernel<B_, K_, csenc::EPI_F32A>); break;
    switch ((g.B * 4 + km) * 8 + epi) {
        CSENC_CASE(8, csenc::KEY_STREAMED) CSENC_CASE(8, csenc::KEY_RESIDENT) CSENC_CASE(8, csenc::KEY_REGS)
        CSENC_CASE(16, csenc::KEY_STREAMED) CSENC_CASE(16, csenc::KEY_RESIDENT) CSENC_CASE(16, csenc::KEY_REGS)
        CSENC_CASE(32, csenc::KEY_STREAMED) CSENC_CASE(32, csenc::KEY_RESIDENT) CSENC_CASE(32, csenc::KEY_CHUNK)
        default: return fail(CS_ERR_UNSUPPORTED, "no kernel instantiation for this plan");
    }
#undef CSENC_CASE
    err = cudaGetLastError();
    if (err == cudaSuccess) err = launch_err;
    if (err != cudaSuccess) return cuda_fail(err, "kernel launch");
    return CS_OK;
}

cudaError_t set_smem_attr_all(int bytes) {
    cudaError_t e = cudaSuccess, r;
#define CSENC_ATTR(B_, K_)                                                                               \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_F32>,                           \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;                                                                          \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16>,                           \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;                                                                          \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16R>,                          \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;                                                                          \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16RR>,                         \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;                                                                          \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_Q16RR64>,                       \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;                                                                          \
    r = cudaFuncSetAttribute(csenc::cs_measure_kernel<B_, K_, csenc::EPI_F32A>,                          \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);                         \
    if (r != cudaSuccess) e = r;
    CSENC_ATTR(8, csenc::KEY_STREAMED) CSENC_ATTR(8, csenc::KEY_RESIDENT) CSENC_ATTR(8, csenc::KEY_REGS)
    CSENC_ATTR(16, csenc::KEY_STREAMED) CSENC_ATTR(16, csenc::KEY_RESIDENT) CSENC_ATTR(16, csenc::KEY_REGS)
    CSENC_ATTR(32, csenc::KEY_STREAMED) CSENC_ATTR(32, csenc::KEY_RESIDENT) CSENC_ATTR(32, csenc::KEY_CHUNK)
#undef CSENC_ATTR
    r = adjoint_set_smem_attr(bytes);
    if (r != cudaSuccess) e = r;
    return e;
}


// Phi -> canonical no-swizzle K-major UMMA layout, zero-padded to Mpad rows:
//   byte(n, k) = (k/8)*LBO + (n/8)*SBO + (n%8)*16 + (k%8)*2.
// The converters emit each group of four pixels j = 4q..4q+3 of a block row in K order
// (4q, 4q+2, 4q+1, 4q+3) (see ptx::residual4), so MMA K index k holds pixel
// j = 4(k/4) + {0,2,1,3}[k%4]; Phi's column k must be pixel j's column.
std::vector<uint16_t> arrange_phi(const Geometry& g, uint32_t lbo, uint32_t sbo, const uint16_t* phi_fp16) {
    static const int kPerm[4] = {0, 2, 1, 3};
    std::vector<uint16_t> arranged((size_t)g.Mpad * g.N, 0);
    for (int n = 0; n < g.M; ++n)
        for (int k = 0; k < g.N; ++k) {
            const int j = (k & ~3) | kPerm[k & 3];
            size_t byte = (size_t)(k / 8) * lbo + (size_t)(n / 8) * sbo + (size_t)(n % 8) * 16 + (size_t)(k % 8) * 2;
            arranged[byte / 2] = phi_fp16[(size_t)n * g.N + j];
        }
    return arranged;
}

}  // namespace

cudaError_t csenc::host::scratch_alloc(cs_encoder* e, void** ptr, size_t bytes, cudaStream_t st) {
    {
        std::lock_guard<std::mutex> lk(e->pool_mu);
        if (!e->pool) {
            cudaMemPoolProps props;
            std::memset(&props, 0, sizeof(props));
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = e->device;
            cudaError_t err = cudaMemPoolCreate(&e->pool, &props);
            if (err != cudaSuccess) {
                e->pool = nullptr;
                return err;
            }
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(e->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    return cudaMallocFromPoolAsync(ptr, bytes, e->pool, st);
}

namespace {

// f1, per-frame scale from stored y (8 M < N): codes = rint(y * inv), inv = 1 / (amax / 32767) of the
// frame -- the same expressions as the K1 epilogue (q16_bits / q16_scale / q16_inv), so the codes are
// bitwise those of the two-pass path.  8 measurements per thread and step (two 16-B loads, one 16-B
// store); per_frame (= nblk * M) is a multiple of 8.
// y is walked from its END: the measurement kernel wrote it front to back, so its last tens of MB are
// still in L2 and are re-read from there; every fully consumed 128-B line of y is then discarded
// (discard.global.L2: no write-back of a workspace nobody reads again).  y must be 128-B aligned.
__global__ void q16_requant_kernel(const float4* __restrict__ y, const uint32_t* __restrict__ amax,
                                   uint4* __restrict__ codes, long long n8, long long per8, int discard) {
    const long long step = (long long)gridDim.x * blockDim.x;
    const int lane = (int)(threadIdx.x & 31u);
    const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long rounds = (n8 + step - 1) / step;   // every thread runs the same trip count (warp-uniform loop)
    for (long long r = 0; r < rounds; ++r) {
        const long long i = n8 - 1 - (start + r * step);   // descending with the lane inside a warp
        if (i >= 0) {
            const float inv = csenc::q16_inv(csenc::q16_scale(__ldg(amax + i / per8)));
            const float4 a = y[2 * i], b = y[2 * i + 1];
            uint4 w;
            w.x = csenc::q16_pack(__float_as_uint(a.x), __float_as_uint(a.y), inv);
            w.y = csenc::q16_pack(__float_as_uint(a.z), __float_as_uint(a.w), inv);
            w.z = csenc::q16_pack(__float_as_uint(b.x), __float_as_uint(b.y), inv);
            w.w = csenc::q16_pack(__float_as_uint(b.z), __float_as_uint(b.w), inv);
            codes[i] = w;
        }
        __syncwarp();   // the warp's loads have returned (their values were used)
        // line i/4 (groups i..i+3, 128 B) was read by this lane and its three lower lanes
        if (discard && i >= 0 && (i & 3) == 0 && lane >= 3 && i + 3 < n8)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(y + 2 * i) : "memory");
    }
}

// f1, per-frame scale: amax bits (pass 1) -> fp32 scales in place, after pass 2 has read them.
__global__ void q16_finalize_kernel(uint32_t* amax, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) amax[i] = __float_as_uint(csenc::q16_scale(amax[i]));
}

}  // namespace

// ============================================================================================ ABI
extern "C" {


int cs_validate_config(int W, int H, int gop, int B, int M, const uint16_t* phi_fp16) {
    return validate(W, H, gop, B, M, phi_fp16);
}

double cs_total_cr(int G, double key_cr, double cs_cr) {
    if (G < 1 || !(key_cr > 0) || !(cs_cr > 0)) return -1.0;
    return (double)G / (1.0 / key_cr + (double)(G - 1) / cs_cr);
}

double cs_compression_ratio_cfg(int W, int H, int gop, int B, int M, int T, double key_cr, int bits) {
    if (W < 1 || H < 1 || gop < 1 || B < 1 || M < 1 || T < 0 || !(key_cr > 0) || bits < 1) return -1.0;
    return cr_formula(make_geometry(W, H, gop, B, M), T, key_cr, bits);
}

int64_t cs_measurement_count_cfg(int W, int H, int gop, int B, int M, int n_seq, int T) {
    if (W < 1 || H < 1 || gop < 1 || B < 1 || M < 1 || n_seq < 0 || T < 0) return -1;
    Geometry g = make_geometry(W, H, gop, B, M);
    return (int64_t)n_seq * cs_frames_per_stream(T, gop) * g.nblk * M;
}

int cs_encoder_create(int W, int H, int gop, int B, int M, const uint16_t* phi_fp16, cs_encoder** out) {
    if (!out) return fail(CS_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!phi_fp16) return fail(CS_ERR_ARG, "phi is NULL");
    int rc = validate(W, H, gop, B, M, phi_fp16);
    if (rc != CS_OK) return rc;
    cs_encoder* e = new (std::nothrow) cs_encoder();
    if (!e) return fail(CS_ERR_OOM, "host allocation failed");
    e->geo = make_geometry(W, H, gop, B, M);
    cudaError_t err = cudaGetDevice(&e->device);
    if (err != cudaSuccess) {
        delete e;
        return cuda_fail(err, "cudaGetDevice");
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, e->device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, e->device);
    if (major != 10 || minor != 0) {
        delete e;
        return fail(CS_ERR_UNSUPPORTED, "device is not sm_100 (B200); this library is built for sm_100a only");
    }
    cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, e->device);
    cudaDeviceGetAttribute(&e->smem_limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device);
    e->candidates = plan_candidates(e->geo, e->smem_limit);
    for (size_t i = 0; i < e->candidates.size(); ++i)
        if (!e->candidates[i].key_resident && !e->candidates[i].key_regs && !e->candidates[i].key_chunk) {
            e->chained_plan = (int)i;
            break;
        }
    // f1 row scales: the best plan whose tiles have <= kRowSlots block rows (used when the current
    // plan -- model choice, autotuned or set -- has more)
    for (size_t i = 0; i < e->candidates.size(); ++i)
        if (e->candidates[i].T_r <= csenc::kRowSlots) {
            e->row_plan = (int)i;
            break;
        }
    if (!make_plan(e->geo, e->smem_limit, e->plan)) {
        delete e;
        return fail(CS_ERR_UNSUPPORTED, "no tiling fits shared memory / TMEM for this configuration");
    }
    // The attribute is per kernel (not per encoder): set the device maximum so encoders with
    // different plans can coexist.
    err = set_smem_attr_all(e->smem_limit);
    if (err != cudaSuccess) {
        delete e;
        return cuda_fail(err, "cudaFuncSetAttribute");
    }
    // Phi in the canonical UMMA layout (arrange_phi): SBO = 128, LBO = Mpad*16
    const Geometry& g = e->geo;
    e->sbo = 128;
    e->lbo = (uint32_t)g.Mpad * 16u;
    e->phi_bytes = (uint32_t)g.Mpad * (uint32_t)g.N * 2u;
    std::vector<uint16_t> arranged = arrange_phi(g, e->lbo, e->sbo, phi_fp16);
    // instruction descriptor, kind::f16: D fp32 (bit 4), A/B fp16 (0), K-major (0),
    // N>>3 at bits 17-22, M>>4 at bits 24-28 (M = 128 lanes).
    e->idesc = (1u << 4) | ((uint32_t)(g.Mpad >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    err = cudaMalloc(&e->phi_dev, e->phi_bytes);
    if (err != cudaSuccess) {
        delete e;
        return fail(CS_ERR_OOM, std::string("cudaMalloc(Phi): ") + cudaGetErrorString(err));
    }
    err = cudaMemcpy(e->phi_dev, arranged.data(), e->phi_bytes, cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
        cudaFree(e->phi_dev);
        delete e;
        return cuda_fail(err, "cudaMemcpy(Phi)");
    }
    e->zeros_bytes = (size_t)e->smem_limit;  // >= any plan's strip (strips live in SMEM)
    if ((err = cudaMalloc(&e->zeros_dev, e->zeros_bytes)) != cudaSuccess ||
        (err = cudaMemset(e->zeros_dev, 0, e->zeros_bytes)) != cudaSuccess) {
        cudaFree(e->phi_dev);
        if (e->zeros_dev) cudaFree(e->zeros_dev);
        delete e;
        return fail(CS_ERR_OOM, std::string("zero buffer: ") + cudaGetErrorString(err));
    }
    if ((rc = prepare_adjoint(e, phi_fp16)) != CS_OK) {
        cs_encoder_destroy(e);
        return rc;
    }
    *out = e;
    return CS_OK;
}

int cs_encoder_destroy(cs_encoder* e) {
    if (!e) return CS_OK;
    if (e->phi_dev) cudaFree(e->phi_dev);
    if (e->zeros_dev) cudaFree(e->zeros_dev);
    if (e->ws_frames) cudaFree(e->ws_frames);
    if (e->ws_out) cudaFree(e->ws_out);
    if (e->phiT_dev) cudaFree(e->phiT_dev);
    if (e->phis_dev) cudaFree(e->phis_dev);
    for (auto& s : e->hs)
        if (s) cudaStreamDestroy(s);
    for (auto& ev : e->hev) cudaEventDestroy(ev);
    if (e->pool) cudaMemPoolDestroy(e->pool);
    delete e;
    return CS_OK;
}

static void fill_info(const Plan& p, const Geometry& g, int sms, cs_plan_info* info) {
    info->tile_block_rows = p.T_r;
    info->folds = p.F;
    info->lanes = p.L;
    info->chunk_rows = p.chunk_rows;
    info->stages = p.n_stages;
    info->key_resident = p.key_chunk ? 3 : p.key_regs ? 2 : p.key_resident;
    info->box_w = g.W;  /* strips are full-width rows */
    info->prefetch_items = p.prefetch_items;
    info->a_bufs = p.n_abuf;
    info->d_bufs = p.n_dbuf;
    info->smem_bytes = (int)p.smem_bytes;
    info->tmem_cols = p.tmem_cols;
    info->m_pad = g.Mpad;
    info->chains = 1;
    info->phi_stream = p.phi_stream;
    info->sms = sms;
}

int cs_plan_cfg(int W, int H, int gop, int B, int M, int smem_limit, int sms, cs_plan_info* info) {
    if (!info) return fail(CS_ERR_ARG, "NULL argument");
    int rc = validate(W, H, gop, B, M, nullptr);
    if (rc != CS_OK) return rc;
    Geometry g = make_geometry(W, H, gop, B, M);
    Plan p;
    if (!make_plan(g, smem_limit, p)) return fail(CS_ERR_UNSUPPORTED, "no tiling fits shared memory / TMEM");
    fill_info(p, g, sms, info);
    return CS_OK;
}

int cs_encoder_set_trace(cs_encoder* e, unsigned long long* trace_dev, int cap) {
    if (!e || cap < 0 || (cap > 0 && !trace_dev)) return fail(CS_ERR_ARG, "bad trace buffer");
    e->trace = cap > 0 ? trace_dev : nullptr;
    e->trace_cap = cap;
    return CS_OK;
}

int cs_encoder_set_stable_inputs(cs_encoder* e, int flags) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (flags & ~(CS_STABLE_FRAMES | CS_STABLE_MEASUREMENTS)) return fail(CS_ERR_ARG, "unknown stable-input flags");
    e->stable_inputs = flags;
    return CS_OK;
}

int cs_encoder_autotune(cs_encoder* e, const uint8_t* frames, int n_seq, int T, float* out, int max_candidates,
                        int reps, cs_stream_t stream) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (max_candidates < 1 || reps < 1) return fail(CS_ERR_ARG, "max_candidates and reps must be >= 1");
    if (int rc = check_device(e->device)) return rc;
    if (cs_frames_per_stream(T, e->geo.G) * n_seq == 0) return CS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t e0, e1;
    cudaError_t err;
    if ((err = cudaEventCreate(&e0)) != cudaSuccess) return cuda_fail(err, "cudaEventCreate");
    if ((err = cudaEventCreate(&e1)) != cudaSuccess) {
        cudaEventDestroy(e0);
        return cuda_fail(err, "cudaEventCreate");
    }
    const Plan keep = e->plan;
    int best = -1;
    float best_ms = 1e30f;
    const int n = std::min<int>(max_candidates, (int)e->candidates.size());
    int rc = CS_OK;
    for (int i = 0; i < n && rc == CS_OK; ++i) {
        e->plan = e->candidates[i];
        rc = cs_encode_batch(e, frames, n_seq, T, out, stream);  // warm-up
        if (rc != CS_OK) break;
        cudaEventRecord(e0, s);
        for (int r = 0; r < reps && rc == CS_OK; ++r) rc = cs_encode_batch(e, frames, n_seq, T, out, stream);
        cudaEventRecord(e1, s);
        if ((err = cudaEventSynchronize(e1)) != cudaSuccess) {
            rc = cuda_fail(err, "autotune");
            break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_ms) {
            best_ms = ms;
            best = i;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc != CS_OK || best < 0) {
        e->plan = keep;
        return rc;
    }
    e->plan = e->candidates[best];
    e->tuned = best;
    return CS_OK;
}

int cs_encoder_num_candidates(const cs_encoder* e) { return e ? (int)e->candidates.size() : -1; }

int cs_encoder_candidate_index(const cs_encoder* e) { return e ? (e->tuned < 0 ? 0 : e->tuned) : -1; }

int cs_encoder_set_candidate(cs_encoder* e, int index) {
    if (!e || index < 0 || index >= (int)e->candidates.size()) return fail(CS_ERR_ARG, "candidate index out of range");
    e->plan = e->candidates[index];
    e->tuned = index;
    return CS_OK;
}

int cs_encoder_plan(const cs_encoder* e, cs_plan_info* info) {
    if (!e || !info) return fail(CS_ERR_ARG, "NULL argument");
    fill_info(e->plan, e->geo, e->sms, info);
    return CS_OK;
}

int64_t cs_measurement_count(const cs_encoder* e, int n_seq, int T) {
    if (!e || n_seq < 0 || T < 0) return -1;
    return (int64_t)n_seq * cs_frames_per_stream(T, e->geo.G) * e->geo.nblk * e->geo.M;
}

double cs_compression_ratio(const cs_encoder* e, int T, double key_cr, int bits) {
    if (!e || T < 0 || !(key_cr > 0) || bits < 1) return -1.0;
    return cr_formula(e->geo, T, key_cr, bits);
}

int cs_encode_batch_gops(cs_encoder* e, const uint8_t* frames, int n_seq, int T, int g0, int g1, float* out,
                         cs_stream_t stream) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    const int n_gops = cdiv(T, e->geo.G);
    if (g0 < 0 || g1 > n_gops || g0 > g1) return fail(CS_ERR_ARG, "GOP range out of bounds");
    if (n_seq == 0 || T == 0 || g0 == g1 || cs_frames_in_gops(T, e->geo.G, g0, g1) == 0) return CS_OK;
    if (!frames || !out) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(out)) return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    if (int rc = check_device(e->device)) return rc;
    return launch(e, frames, n_seq, T, g0, g1, out, (cudaStream_t)stream);
}

int cs_encode_batch(cs_encoder* e, const uint8_t* frames, int n_seq, int T, float* out, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_batch");
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (T < 0) return fail(CS_ERR_ARG, "T must be >= 0");
    return cs_encode_batch_gops(e, frames, n_seq, T, 0, cdiv(T, e->geo.G), out, stream);
}

int cs_encode_gop(cs_encoder* e, const uint8_t* frames, int n_frames, float* out, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_gop");
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_frames < 1 || n_frames > e->geo.G) return fail(CS_ERR_ARG, "n_frames must be in [1, gop]");
    return cs_encode_batch_gops(e, frames, 1, n_frames, 0, 1, out, stream);
}

int cs_encoder_set_gop_phis(cs_encoder* e, int n_phi, const uint16_t* phis) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_phi < 0 || (n_phi > 0 && !phis)) return fail(CS_ERR_ARG, "n_phi must be >= 0 and phis non-NULL");
    const Geometry& g = e->geo;
    const size_t per = (size_t)g.M * g.N;
    if (int rc = check_device(e->device)) return rc;
    for (int i = 0; i < n_phi; ++i) {
        const int rc = validate(g.W, g.H, g.G, g.B, g.M, phis + (size_t)i * per);
        if (rc != CS_OK) return rc;
    }
    if (e->phis_dev) cudaFree(e->phis_dev);
    e->phis_dev = nullptr;
    e->n_phis = 0;
    if (n_phi == 0) return CS_OK;
    cudaError_t err = cudaMalloc(&e->phis_dev, (size_t)n_phi * e->phi_bytes);
    if (err != cudaSuccess) return fail(CS_ERR_OOM, std::string("cudaMalloc(phis): ") + cudaGetErrorString(err));
    for (int i = 0; i < n_phi; ++i) {
        std::vector<uint16_t> a = arrange_phi(g, e->lbo, e->sbo, phis + (size_t)i * per);
        err = cudaMemcpy((uint8_t*)e->phis_dev + (size_t)i * e->phi_bytes, a.data(), e->phi_bytes, cudaMemcpyHostToDevice);
        if (err != cudaSuccess) {
            cudaFree(e->phis_dev);
            e->phis_dev = nullptr;
            return cuda_fail(err, "cudaMemcpy(phis)");
        }
    }
    e->n_phis = n_phi;
    return CS_OK;
}

int cs_encode_batch_chained(cs_encoder* e, const uint8_t* frames, int n_seq, int T, float* out, cs_stream_t stream) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    if (n_seq == 0 || T == 0 || cs_frames_per_stream(T, e->geo.G) == 0) return CS_OK;
    if (!frames || !out) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(out)) return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    if (e->chained_plan < 0) return fail(CS_ERR_UNSUPPORTED, "no streamed-key plan fits this configuration");
    if (int rc = check_device(e->device)) return rc;
    QArgs q;
    q.chained = 1;
    q.plan = &e->candidates[(size_t)e->chained_plan];
    return launch(e, frames, n_seq, T, 0, cdiv(T, e->geo.G), out, (cudaStream_t)stream, q);
}

int cs_encode_batch_keys(cs_encoder* e, const uint8_t* frames, int n_seq, int T, const uint8_t* keys, float* out,
                         cs_stream_t stream) {
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    if (n_seq == 0 || T == 0 || cs_frames_per_stream(T, e->geo.G) == 0) return CS_OK;
    if (!frames || !keys || !out) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(keys) || !aligned16(out)) return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    if (int rc = check_device(e->device)) return rc;
    QArgs q;
    q.keys = keys;
    return launch(e, frames, n_seq, T, 0, cdiv(T, e->geo.G), out, (cudaStream_t)stream, q);
}

int64_t cs_q16_scale_count(const cs_encoder* e, int n_seq, int T, int granularity) {
    if (!e || n_seq < 0 || T < 0) return -1;
    const long long n_cs = (long long)n_seq * cs_frames_per_stream(T, e->geo.G);
    if (granularity == CS_Q16_FRAME) return n_cs;
    if (granularity == CS_Q16_ROW) return n_cs * e->geo.nby;
    return -1;
}

int cs_encode_batch_q16(cs_encoder* e, const uint8_t* frames, int n_seq, int T, int granularity, int16_t* codes,
                        float* scales, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_batch_q16");
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    if (granularity != CS_Q16_FRAME && granularity != CS_Q16_ROW) return fail(CS_ERR_ARG, "bad granularity");
    const Geometry& g = e->geo;
    const long long n_cs = (long long)n_seq * cs_frames_per_stream(T, g.G);
    if (n_cs == 0) return CS_OK;
    if (!frames || !codes || !scales) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(codes) || (reinterpret_cast<uintptr_t>(scales) & 3u))
        return fail(CS_ERR_ARG, "frames/codes must be 16-byte aligned, scales 4-byte aligned");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    if (int rc = check_device(e->device)) return rc;
    const int n_gops = cdiv(T, g.G);
    const cudaStream_t st = (cudaStream_t)stream;
    QArgs q;
    q.codes = codes;
    if (granularity == CS_Q16_ROW) {
        if (e->plan.T_r > csenc::kRowSlots) {   // the current plan's tiles are too tall: the best one that fits
            if (e->row_plan < 0)
                return fail(CS_ERR_UNSUPPORTED, "row-scale quantisation: no plan with <= 40 block rows per tile fits");
            q.plan = &e->candidates[(size_t)e->row_plan];
        }
        q.qmode = csenc::Q_ROW;
        q.scales = scales;
        return launch(e, frames, n_seq, T, 0, n_gops, nullptr, st, q);
    }
    // per-frame scale: zero the |y| maxima, then either
    //  (a) 8 M < N: one measurement pass storing fp32 y in a stream-ordered workspace + the maxima,
    //      and a re-quantisation pass over y (8 B per measurement moved instead of re-reading the
    //      frames, N / M B per measurement), or
    //  (b) an absmax pass and a codes pass, both measuring (no y round trip);
    // then finalize (maxima -> scales in place).
    q.amax = reinterpret_cast<uint32_t*>(scales);
    cudaError_t err = cudaMemsetAsync(scales, 0, (size_t)n_cs * sizeof(float), st);
    if (err != cudaSuccess) return cuda_fail(err, "cudaMemsetAsync");
    const long long per_frame = (long long)g.nblk * g.M;
    const int store_knob = env_int("CSENC_Q16_STORE", 1);   // (TUNING builds: 0 = never, 2 = for every M)
    if ((8 * g.M <= g.N || store_knob == 2) && per_frame % 8 == 0 && store_knob) {
        float* ybuf = nullptr;
        err = scratch_alloc(e, (void**)&ybuf, (size_t)(n_cs * per_frame) * sizeof(float), st);
        if (err == cudaSuccess) {
            q.qmode = csenc::Q_STOREMAX;
            int rc = launch(e, frames, n_seq, T, 0, n_gops, ybuf, st, q);
            if (rc == CS_OK) {
                const long long n8 = n_cs * per_frame / 8;
                const unsigned blocks = (unsigned)std::min<long long>((n8 + 255) / 256, (long long)e->sms * 16);
                q16_requant_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(ybuf), q.amax,
                                                          reinterpret_cast<uint4*>(codes), n8, per_frame / 8,
                                                          (reinterpret_cast<uintptr_t>(ybuf) & 127u) == 0 ? 1 : 0);
                err = cudaGetLastError();
                if (err == cudaSuccess) {
                    q16_finalize_kernel<<<(unsigned)((n_cs + 255) / 256), 256, 0, st>>>(q.amax, n_cs);
                    err = cudaGetLastError();
                }
                rc = err == cudaSuccess ? CS_OK : cuda_fail(err, "re-quantisation launch");
            }
            cudaFreeAsync(ybuf, st);
            return rc;
        }
        cudaGetLastError();   // no workspace: fall back to measuring twice
    }
    q.qmode = csenc::Q_ABSMAX;
    int rc = launch(e, frames, n_seq, T, 0, n_gops, nullptr, st, q);
    if (rc != CS_OK) return rc;
    q.qmode = csenc::Q_FRAME;
    rc = launch(e, frames, n_seq, T, 0, n_gops, nullptr, st, q);
    if (rc != CS_OK) return rc;
    q16_finalize_kernel<<<(unsigned)((n_cs + 255) / 256), 256, 0, st>>>(q.amax, n_cs);
    err = cudaGetLastError();
    return err == cudaSuccess ? CS_OK : cuda_fail(err, "finalize launch");
}

}  // extern "C"

namespace {

// Host-buffer pipeline shared by the fp32 and q16 host calls.  granularity < 0: fp32 measurements into
// outs_host[k] (float); otherwise int16 codes into outs_host[k] and fp32 scales into scales_host[k].
// Groups are chunks of streams (n_seq > 1) or of whole GOPs of the single stream; a GOP range of one
// stream is itself a stream of whole GOPs starting at a key frame, so every group is one ordinary
// device-buffer call on a sub-batch.  Copy-in of group i+1 overlaps the encodes of group i and the
// copy-outs of group i-1; each frame group crosses PCIe once whatever the number of encoders.
int host_pipeline(cs_encoder* const* encs, int n_enc, const uint8_t* frames_host, int n_seq, int T, int granularity,
                  void* const* outs_host, float* const* scales_host) {
    if (!encs || n_enc < 1) return fail(CS_ERR_ARG, "encoders: need at least one");
    for (int k = 0; k < n_enc; ++k) {
        if (!encs[k]) return fail(CS_ERR_ARG, "encoder is NULL");
        for (int j = 0; j < k; ++j)
            if (encs[j] == encs[k]) return fail(CS_ERR_ARG, "the same encoder twice");
        const Geometry& a = encs[0]->geo;
        const Geometry& c = encs[k]->geo;
        if (c.W != a.W || c.H != a.H || c.G != a.G || encs[k]->device != encs[0]->device)
            return fail(CS_ERR_ARG, "encoders must share W, H, gop and device");
    }
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    const bool q16 = granularity >= 0;
    if (q16 && granularity != CS_Q16_FRAME && granularity != CS_Q16_ROW) return fail(CS_ERR_ARG, "bad granularity");
    cs_encoder* const e = encs[0];   // frames workspace, streams and events
    const Geometry& g = e->geo;
    const long long cs_s = cs_frames_per_stream(T, g.G);
    if (n_seq == 0 || T == 0 || cs_s == 0) return CS_OK;
    if (!frames_host || !outs_host || (q16 && !scales_host)) return fail(CS_ERR_ARG, "NULL buffer");
    for (int k = 0; k < n_enc; ++k)
        if (!outs_host[k] || (q16 && !scales_host[k])) return fail(CS_ERR_ARG, "NULL output buffer");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    DeviceGuard dev_guard(e->device);   // synchronous host call: run on the encoders' device
    if (!dev_guard.ok) return fail(CS_ERR_CUDA, "cannot switch to the encoder's device");
    const size_t frame_bytes = (size_t)g.W * g.H;
    const size_t in_bytes = (size_t)n_seq * T * frame_bytes;
    const size_t n_cs = (size_t)n_seq * cs_s;
    const size_t elem = q16 ? sizeof(int16_t) : sizeof(float);
    // workspaces are per encoder: lock them in address order (no deadlock between concurrent callers)
    std::vector<cs_encoder*> order(encs, encs + n_enc);
    std::sort(order.begin(), order.end());
    std::vector<std::unique_lock<std::mutex>> locks;
    for (cs_encoder* x : order) locks.emplace_back(x->ws_mu);
    cudaError_t err;
    if (e->ws_frames_bytes < in_bytes) {
        if (e->ws_frames) cudaFree(e->ws_frames);
        e->ws_frames = nullptr;
        e->ws_frames_bytes = 0;
        if ((err = cudaMalloc(&e->ws_frames, in_bytes)) != cudaSuccess)
            return fail(CS_ERR_OOM, std::string("workspace: ") + cudaGetErrorString(err));
        e->ws_frames_bytes = in_bytes;
    }
    // per encoder: [measurements or codes][scales] (scales at a 256-byte aligned offset)
    std::vector<size_t> sc_off(n_enc, 0), sc_per_cs(n_enc, 0);
    for (int k = 0; k < n_enc; ++k) {
        cs_encoder* x = encs[k];
        const size_t meas_bytes = n_cs * (size_t)x->geo.nblk * x->geo.M * elem;
        sc_per_cs[k] = !q16 ? 0 : (granularity == CS_Q16_ROW ? (size_t)x->geo.nby : 1);
        sc_off[k] = (meas_bytes + 255) / 256 * 256;
        const size_t out_bytes = sc_off[k] + n_cs * sc_per_cs[k] * sizeof(float);
        if (x->ws_out_bytes < out_bytes) {
            if (x->ws_out) cudaFree(x->ws_out);
            x->ws_out = nullptr;
            x->ws_out_bytes = 0;
            if ((err = cudaMalloc(&x->ws_out, out_bytes)) != cudaSuccess)
                return fail(CS_ERR_OOM, std::string("workspace: ") + cudaGetErrorString(err));
            x->ws_out_bytes = out_bytes;
        }
    }
    for (auto& st : e->hs)
        if (!st && (err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(err, "cudaStreamCreate");
    struct Grp {
        int s0, s1, g0, g1;
    };
    std::vector<Grp> groups;
    const int n_gops = cdiv(T, g.G);
    if (n_seq > 1) {
        const int per = std::max(1, n_seq / 8);
        for (int s = 0; s < n_seq; s += per) groups.push_back({s, std::min(n_seq, s + per), 0, n_gops});
    } else {
        const int per = std::max(1, n_gops / 8);
        for (int gg = 0; gg < n_gops; gg += per) groups.push_back({0, 1, gg, std::min(n_gops, gg + per)});
    }
    const size_t n_ev = groups.size() * (size_t)(1 + n_enc);
    while (e->hev.size() < n_ev) {
        cudaEvent_t ev;
        if ((err = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(err, "cudaEventCreate");
        e->hev.push_back(ev);
    }
    cudaStream_t s_in = e->hs[0], s_run = e->hs[1], s_out = e->hs[2];
    int rc = CS_OK;
    for (size_t i = 0; i < groups.size() && rc == CS_OK; ++i) {
        const Grp& gr = groups[i];
        // the group as a sub-batch: streams [s0, s1) x all T frames, or frames [g0*G, min(g1*G, T)) of
        // the single stream (whole GOPs from a key frame)
        size_t f0, f1, c0, c1;   // frame range (global [s][t] order) and CS-frame range of the group
        int sub_seq, sub_T;
        if (n_seq > 1) {
            f0 = (size_t)gr.s0 * T;
            f1 = (size_t)gr.s1 * T;
            c0 = (size_t)gr.s0 * cs_s;
            c1 = (size_t)gr.s1 * cs_s;
            sub_seq = gr.s1 - gr.s0;
            sub_T = T;
        } else {
            f0 = (size_t)gr.g0 * g.G;
            f1 = std::min((size_t)gr.g1 * g.G, (size_t)T);
            c0 = (size_t)cs_frames_in_gops(T, g.G, 0, gr.g0);
            c1 = (size_t)cs_frames_in_gops(T, g.G, 0, gr.g1);
            sub_seq = 1;
            sub_T = (int)(f1 - f0);
        }
        err = cudaMemcpyAsync(e->ws_frames + f0 * frame_bytes, frames_host + f0 * frame_bytes,
                              (f1 - f0) * frame_bytes, cudaMemcpyHostToDevice, s_in);
        if (err != cudaSuccess) {
            rc = cuda_fail(err, "H2D");
            break;
        }
        cudaEvent_t* ev = &e->hev[i * (size_t)(1 + n_enc)];
        cudaEventRecord(ev[0], s_in);
        cudaStreamWaitEvent(s_run, ev[0], 0);
        if (c1 == c0) continue;
        for (int k = 0; k < n_enc && rc == CS_OK; ++k) {
            cs_encoder* x = encs[k];
            const size_t per_cs = (size_t)x->geo.nblk * x->geo.M;   // measurements per CS frame
            uint8_t* const ws = reinterpret_cast<uint8_t*>(x->ws_out);
            uint8_t* const meas_dev = ws + c0 * per_cs * elem;
            float* const sc_dev = reinterpret_cast<float*>(ws + sc_off[k]) + c0 * sc_per_cs[k];
            const uint8_t* const fr = e->ws_frames + f0 * frame_bytes;
            rc = q16 ? cs_encode_batch_q16(x, fr, sub_seq, sub_T, granularity, reinterpret_cast<int16_t*>(meas_dev), sc_dev, s_run)
                     : cs_encode_batch(x, fr, sub_seq, sub_T, reinterpret_cast<float*>(meas_dev), s_run);
            if (rc != CS_OK) break;
            cudaEventRecord(ev[1 + k], s_run);
            cudaStreamWaitEvent(s_out, ev[1 + k], 0);
            err = cudaMemcpyAsync(reinterpret_cast<uint8_t*>(outs_host[k]) + c0 * per_cs * elem, meas_dev,
                                  (c1 - c0) * per_cs * elem, cudaMemcpyDeviceToHost, s_out);
            if (err == cudaSuccess && q16)
                err = cudaMemcpyAsync(scales_host[k] + c0 * sc_per_cs[k], sc_dev, (c1 - c0) * sc_per_cs[k] * sizeof(float),
                                      cudaMemcpyDeviceToHost, s_out);
            if (err != cudaSuccess) rc = cuda_fail(err, "D2H");
        }
    }
    cudaError_t e1 = cudaStreamSynchronize(s_in), e2 = cudaStreamSynchronize(s_run), e3 = cudaStreamSynchronize(s_out);
    if (rc != CS_OK) return rc;
    if (e1 != cudaSuccess) return cuda_fail(e1, "sync");
    if (e2 != cudaSuccess) return cuda_fail(e2, "encode");
    if (e3 != cudaSuccess) return cuda_fail(e3, "sync");
    return CS_OK;
}

}  // namespace

extern "C" {

int cs_encode_batch_host_multi(cs_encoder* const* encs, int n_enc, const uint8_t* frames_host, int n_seq, int T,
                               float* const* outs_host) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_batch_host_multi");
    std::vector<void*> outs(outs_host ? n_enc : 0);
    for (size_t k = 0; k < outs.size(); ++k) outs[k] = outs_host[k];
    return host_pipeline(encs, n_enc, frames_host, n_seq, T, -1, outs_host ? outs.data() : nullptr, nullptr);
}

int cs_encode_batch_host(cs_encoder* e, const uint8_t* frames_host, int n_seq, int T, float* out_host) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_batch_host");
    return cs_encode_batch_host_multi(&e, 1, frames_host, n_seq, T, &out_host);
}

int cs_encode_batch_host_multi_q16(cs_encoder* const* encs, int n_enc, const uint8_t* frames_host, int n_seq, int T,
                                   int granularity, int16_t* const* codes_host, float* const* scales_host) {
    csenc::host::NvtxScope nvtx_scope("cs_encode_batch_host_multi_q16");
    if (granularity < 0) return fail(CS_ERR_ARG, "bad granularity");
    std::vector<void*> outs(codes_host && n_enc > 0 ? n_enc : 0);
    for (size_t k = 0; k < outs.size(); ++k) outs[k] = codes_host[k];
    return host_pipeline(encs, n_enc, frames_host, n_seq, T, granularity, codes_host ? outs.data() : nullptr,
                         scales_host);
}

int cs_encode_batch_host_q16(cs_encoder* e, const uint8_t* frames_host, int n_seq, int T, int granularity,
                             int16_t* codes_host, float* scales_host) {
    return cs_encode_batch_host_multi_q16(&e, 1, frames_host, n_seq, T, granularity, &codes_host, &scales_host);
}

}  // extern "C"
