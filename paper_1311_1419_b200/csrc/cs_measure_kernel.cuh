// cs_measure_kernel.cuh -- K1: fused GOP residual formation + block CS measurement on sm_100a.
//
// One persistent, warp-specialised kernel per encode call.  Work unit =
// (stream s, GOP g, tile t of full-width block rows, range of CS frames of the GOP).  Item =
// one K-chunk (chunk_rows pixel rows of every block) of one CS frame of the unit's tile.
//
//   warp 12       TMA producer: Phi -> SMEM once (bulk copy).  Per item the tile strip of the
//                 CS frame -- contiguous in HBM, rows [y0, y0+rows) x all W columns -- arrives
//                 in ONE cp.async.bulk per piece into a ring slot; rows beyond H are filled from
//                 a zero buffer (partial blocks, reading R10), so every slot holds whole blocks.
//                 The unit's key strip: KM=2 once per unit through a ring slot into converter
//                 registers; KM=1 into a double-buffered SMEM region; KM=0 with every item.
//   warps 0..7    converters (a2 im2col + a3 residual), two warpgroups splitting each item's row
//                 groups; thread = TMEM lane = block of the tile.  Reads its block's row segments
//                 of the CS strip (and key) from SMEM, forms r = F - F_key exactly in fp16 (magic
//                 number 0x64XX = 1024 + XX), and writes it with tcgen05.st as the MMA A operand
//                 in TMEM (row = block, two fp16 per 32-bit column, K order of ptx::residual4).
//   warp 13       MMA issuer (a4) + TMEM allocator: D[tmem, fp32] += A[tmem, fp16] x
//                 Phi^T[smem, fp16], one tcgen05.mma.kind::f16 (M=128 lanes, N=Mpad, K=16) per
//                 16 pixels; commit -> mbarriers.  Warp-uniform loop, one elected issuing lane.
//   warp 14       (KEY_CHUNK kernels only) second MMA issuer: the two warps take alternate items.
//   warps 8..11   epilogue (a6): tcgen05.ld of the fp32 accumulators -> (swizzled SMEM tile) ->
//                 row-contiguous vector stores of y[s][g][c][by][bx][0..M) (block-major).
//
// The warp scheduler arbitrates highest-warp-id first, so the single-thread roles (MMA issue,
// TMA issue) have the highest ids and are never starved by the converter warps.  The kernel is
// templated on the block size B and the key mode KM so that each instantiation carries only the
// code its plan runs (instruction-cache footprint matters: 14 warps run 4 different loops).
//
// Pipelines (mbarrier parity rings): stage_full/empty (TMA <-> converters), key_full/empty
// (KM=1), a_full/empty (converters <-> MMA, TMEM A buffers), d_full/empty (MMA <-> epilogue,
// TMEM accumulators).  Paper passages: Eq.(1) P:83-85, P:87 and Eq.(2)-(3) P:89-91.
//
// Launch overlap: the kernel is launched with programmatic stream serialization; it releases the next
// kernel's launch in its prologue and waits for the previous kernel (griddepcontrol.wait) before it touches
// global memory -- the whole CTA by default, only the epilogue warps when the caller has promised stable
// inputs (KParams::pdl_early, cs_encoder_set_stable_inputs).
#pragma once
#include <cuda.h>
#include <type_traits>
#include <cstdint>

#include "ptx_sm100.cuh"

// The KEY_CHUNK branches of the role loops end in `continue`, so in those instantiations the other
// modes' loops that follow are unreachable by construction (warning 128).
#pragma nv_diagnostic push
#pragma nv_diag_suppress 128

#ifndef CSENC_DEBUG
#define CSENC_DEBUG 0  // 1: compile the ablation switches (KParams::dbg_*) into the kernel
#endif
// CS_CHECK (CSENC_CHECKS builds): see ptx_sm100.cuh

namespace csenc {

constexpr int kConvWarps = 8;                    // warps 0..7: two converter warpgroups
constexpr int kEpiWarp0 = 8;                     // warps 8..11: epilogue warpgroup
constexpr int kProducerWarp = 12;                // TMA producer
constexpr int kMmaWarp = 13;                     // MMA issuer + TMEM allocator
constexpr int kThreads = 14 * 32;
// KEY_CHUNK kernels run a second MMA-issuing warp (warp 14): one thread issues a small-N TS tcgen05.mma every
// ~49 cycles whatever N <= 64 is, two threads together one every ~30 (the tensor pipe's time for N = 64;
// tools/mma_microbench3.cu).  The two warps take alternate items, each item whole and in K order.
constexpr int kThreadsChunk = 15 * 32;
template <int KM>
constexpr int threads_for() { return KM == 3 ? kThreadsChunk : kThreads; }
constexpr int kMaxFolds = 8;
constexpr int kMaxStages = 8;
constexpr int kMaxTmemBufs = 8;                  // TMEM A buffers / accumulators (ring depth cap)
constexpr uint32_t kTmemCols = 512;

enum KeyMode : int { KEY_STREAMED = 0, KEY_RESIDENT = 1, KEY_REGS = 2, KEY_CHUNK = 3 };
// epilogue variants (template EPI): fp32 measurements (a6), or 16-bit codes (f1)
// One instantiation per variant keeps each kernel's code small: the four roles' loops share the SM's
// instruction cache (measured: a 64-value register path in the shared q16 kernel cost the other
// modes 7-10%; split out, the row mode gained 38% at M = 16/32).
enum Epilogue : int {
    EPI_F32 = 0,    // fp32 measurements
    EPI_Q16 = 1,    // Q_ABSMAX / Q_FRAME (the two passes of the per-frame scale)
    // (2: a single-pass per-frame look-back mode, measured slower than two passes and removed in round 2)
    EPI_Q16R = 3,   // Q_ROW, general (two TMEM passes, named barrier)
    EPI_Q16RR = 4,  // Q_ROW, register path: one fold, M = 16 or 32, <= kRowRegRows block rows
    EPI_Q16RR64 = 5,  // the same for M = 48 or 64
    EPI_F32A = 6,   // fp32 measurements + per-CS-frame |y| maximum (atomicMax into amax): the first
                    // pass of the per-frame scale when storing y and re-quantising it is cheaper than
                    // measuring twice (8 M < N)
};
// EPI_Q16 sub-modes (KParams::qmode)
enum QMode : int {
    Q_ABSMAX = 1,     // pass 1 of the per-frame scale: atomicMax of |y| bits into amax[cs], no stores
    Q_FRAME = 2,      // pass 2: codes with scale = amax[cs] / 32767 (1 if 0)
    Q_ROW = 3,        // single pass: one scale per (CS frame, block row), reduced in SMEM
    Q_STOREMAX = 5,   // EPI_F32A: fp32 y to a workspace + atomicMax of |y| bits into amax[cs]
};
constexpr int kRowSlots = 40;                    // Q_ROW: max block rows per tile (3 x 40 u32 slots)
constexpr uint32_t kRowSlotOff = 512;            // Q_ROW slots live in the barrier page (bytes 512..991)
static_assert(16 * kMaxStages + 32 + 32 * kMaxTmemBufs + 24 <= (int)kRowSlotOff, "barrier block overlaps row slots");
static_assert(kRowSlotOff + 3 * kRowSlots * 4 <= 1024, "row slots overflow the barrier page");
// Q_ROW register path (one fold, M = 16 or 32, <= 32 block rows): values stay in registers between the
// row reduction and the codes; each epilogue warp's row maxima go to its own slots in the upper half
// of its 4 KB staging tile (codes use <= 2 KB of it), kRowBufs items deep, behind row_full mbarriers.
constexpr int kRowBufs = 4;
constexpr int kRowRegRows = 32;
constexpr uint32_t kRowBarOff = 448;             // row_full[kRowBufs] (4 epilogue-warp arrivals each)
constexpr uint32_t kRowSlotTileOff = 2048;
static_assert(16 * kMaxStages + 32 + 32 * kMaxTmemBufs + 24 <= (int)kRowBarOff, "barrier block overlaps row barriers");
static_assert(kRowBarOff + 8 * kRowBufs <= kRowSlotOff, "row barriers overlap the row slots");
static_assert(kRowSlotTileOff + kRowBufs * kRowRegRows * 4 <= 4096, "row slots overflow the staging tile");

struct KParams {
    // tma_strips != 0 (KEY_STREAMED / KEY_CHUNK multi-piece plans, H % B == 0): the T_r pieces of a strip
    // arrive by ONE TMA box of KParamsTS::smap instead of T_r bulk copies.  2 (KEY_CHUNK, W % 128 == 0):
    // the box is written with the 128-B swizzle (16-byte chunk c of 128-B line L lands at chunk c ^ (L & 7)),
    // so the converters' 16-byte reads of blocks 32 bytes apart spread over all banks (unswizzled, lanes
    // l and l + 4 of a quarter-warp hit the same banks: every read took two wavefronts)
    int tma_strips;
    // pdl_early != 0 (cs_encoder_set_stable_inputs): the inputs do not depend on the stream's previous kernel,
    // so only the epilogue warps wait for it (before their first store / first read of the frame maxima)
    int pdl_early;
    // phi_stream != 0 (multi-chunk plans, KM 0/1): Phi is not resident; each stage carries the K-slice
    // of Phi its chunk needs (phi_slice_bytes at stage offset stage_phi_off, a contiguous range of the
    // canonical layout), and the stage is freed only when the converters AND the MMAs are done with it
    int phi_stream;
    uint32_t phi_slice_bytes, stage_phi_off;
    const uint8_t* frames;    // device [n_seq][T][H][W]
    const uint8_t* zeros;     // device, >= piece_rows * W zero bytes (rows beyond H)
    float* out;
    const uint16_t* phi;      // device, canonical UMMA layout, phi_bytes
    uint32_t phi_bytes;
    // f4 variant (per-GOP seeds): n_phis > 0 -> GOP g is measured with
    // phis[g % n_phis] (each phi_bytes, same layout), reloaded into SMEM when a unit's GOP changes
    const uint16_t* phis;
    int n_phis;
    uint32_t off_phi2;        // per-GOP Phi, resident: a second Phi slot (0 = one slot): the next GOP's matrix
                              // loads while the current one is in use
    int W, H, M, Mpad, N;
    int nbx, nby, nblk;
    // tiling
    int T_r, F, L, n_tiles;
    int Lq;                   // logical lanes per TMEM lane quarter: physical lane 32q + r holds logical
                              // lane q*Lq + r (r < Lq), so small tiles use all four SM sub-partitions
    int chunk_rows, n_chunks, chunk_k;
    int pieces;               // strips per stage: 1 (all T_r*B rows, n_chunks == 1) or T_r
    int piece_rows;           // rows per strip
    int single_piece;
    uint32_t piece_bytes, stage_cs_bytes, stage_bytes, key_bytes;
    uint32_t set_bytes;       // bytes one load_strips() call delivers: pieces * piece_rows * W
    int n_stages;
    uint32_t off_tab, off_epi, off_phi, off_key, off_stage;
    // work
    int G, T, gop_begin, n_gops_sel, cs_per_stream_sel, n_splits, cs_per_unit, n_units;
    // MMA
    uint32_t idesc, lbo, sbo;
    int a_cols, d_cols;
    int n_abuf, n_dbuf;       // TMEM ring depths (1..kMaxTmemBufs)
    // optional timeline trace (CTA 0 only): trace[event * trace_cap + i] = clock64 of the i-th
    // occurrence of the event; nullptr disables (the default)
    unsigned long long* trace;
    int trace_cap;
    int dbg_load_only;        // CSENC_DEBUG only: converters release stages, no MMA/epilogue
    int dbg_flags;            // CSENC_DEBUG only: 2 = converters write zeros, 8 = no output stores
    // CSENC_CHECKS only: bounds
    uint32_t smem_bytes;      // dynamic SMEM size (from the aligned base)
    long long out_floats;     // output buffer size in floats
    long long frames_bytes;   // input buffer size in bytes
    // f4 closed loop: decoded key frames [n_seq][n_gops_T][H][W] (nullptr = the raw key frames of
    // `frames`, the north star's pass-through); n_gops_T = ceil(T / G)
    const uint8_t* keys;
    int n_gops_T;
    long long keys_bytes;     // CSENC_CHECKS: size of `keys`
    // f4 variant (KM == KEY_STREAMED plans only): every CS frame's reference is the previous raw
    // frame (Eq. 3 read literally: D_N = F_N - F_{N-1}) instead of the GOP key
    int chained;
    // EPI_Q16 (f1)
    int qmode;                // QMode
    int16_t* codes;           // [n_cs][nblk][M] int16, same layout as out
    uint32_t* amax;           // Q_ABSMAX / Q_FRAME / Q_STOREMAX: [n_cs] fp32 |y| max bits (zeroed)
    float* scales;            // Q_ROW: [n_cs][nby] fp32 scales
};

// KEY_STREAMED kernels' parameters: + the strip tensor map (frames as u32 words [n_seq*T][nby][B][W/4],
// box [1][T_r][chunk_rows][W/4], block rows past nby zero-filled).  Only these kernels carry it:
// a CUtensorMap in the parameters of the other kernels measurably slowed them (C4 M = 64: -2%).
struct KParamsTS : KParams {
    alignas(64) CUtensorMap smap;
};
template <int KM>
using KParamsFor = typename std::conditional<KM == KEY_STREAMED || KM == KEY_CHUNK, KParamsTS, KParams>::type;

// trace events
enum : int {
    EV_P_EMPTY = 0,   // producer: stage slot free
    EV_P_ISSUED,      // producer: stage copies issued
    EV_C_FULL,        // converter: stage data landed
    EV_C_AEMPTY,      // converter: A buffer free
    EV_C_DONE,        // converter: A written (before a_full arrive)
    EV_M_AFULL,       // MMA: A ready
    EV_M_ISSUED,      // MMA: chunk MMAs issued + committed
    EV_E_DFULL,       // epilogue: accumulator ready
    EV_E_DONE,        // epilogue: stores issued, D released
    EV_C_CONV,        // converter: all tcgen05.st issued (before wait::st)
    EV_E_ARRIVED,     // epilogue (Q_ROW register path): row maxima published
    EV_E_ROWS,        // epilogue (Q_ROW register path): all 4 warps' row maxima present
    EV_K_START,       // CTA 0 thread 0: kernel entry (one occurrence)
    EV_K_END,         // CTA 0 thread 0: after the final barrier (one occurrence)
    EV_COUNT
};

__device__ __forceinline__ void trace_ev(const KParams& p, int ev, int i) {
    if (p.trace != nullptr && blockIdx.x == 0 && i < p.trace_cap)
        p.trace[(size_t)ev * p.trace_cap + i] = clock64();
}

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

__device__ __forceinline__ int key_frame(const KParams& p, const Unit& w) { return w.s * p.T + w.g * p.G; }

// Copy the strips of K-chunk k of tile t of `frame` into dst ([piece][piece_rows][W]); rows at or
// beyond H come from the zero buffer.  Always delivers pieces * piece_rows * W bytes, so the
// mbarrier transaction count of a slot is a constant.
template <int B>
__device__ __forceinline__ void load_strips(const KParams& p, uint32_t dst, const uint8_t* frame, int t, int k,
                                            uint32_t bar, uint64_t policy, int fidx = -1,
                                            const CUtensorMap* smap = nullptr) {
    if (smap != nullptr && fidx >= 0 && p.tma_strips) {   // all T_r pieces in one box (frame fidx of `frames`)
        if (p.tma_strips == 2)   // 128-B lines, swizzled (KEY_CHUNK, W % 128 == 0)
            ptx::tma_load_5d(dst, smap, bar, 0, 0, k * p.chunk_rows, t * p.T_r, fidx, policy);
        else
            ptx::tma_load_4d(dst, smap, bar, 0, k * p.chunk_rows, t * p.T_r, fidx, policy);
        return;
    }
    for (int pc = 0; pc < p.pieces; ++pc) {
        const int y0 = p.single_piece ? t * p.T_r * B : (t * p.T_r + pc) * B + k * p.chunk_rows;
        const int rows = max(0, min(p.piece_rows, p.H - y0));
        const uint32_t d = dst + (uint32_t)pc * p.piece_bytes;
        CS_CHECK(rows == 0 ||
                 (frame >= p.frames && (long long)(frame - p.frames) + (long long)(y0 + rows) * p.W <= p.frames_bytes) ||
                 (p.keys != nullptr && frame >= p.keys &&
                  (long long)(frame - p.keys) + (long long)(y0 + rows) * p.W <= p.keys_bytes));
        CS_CHECK(rows >= p.piece_rows || (uint32_t)(p.piece_rows - rows) * p.W <= p.smem_bytes);
        if (rows > 0) ptx::bulk_load_hint(d, frame + (size_t)y0 * p.W, (uint32_t)rows * p.W, bar, policy);
        if (rows < p.piece_rows)
            ptx::bulk_load(d + (uint32_t)rows * p.W, p.zeros, (uint32_t)(p.piece_rows - rows) * p.W, bar);
    }
}

// Converter: one block row segment of B pixels -> B/2 fp16x2 residual words.  `half2` (B=32 only)
// is false when the block's right 16 columns lie beyond W (they are then zero in both frames).
template <int B>
struct RowConv;
template <>
struct RowConv<8> {
    static constexpr int kWords = 4;
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w, bool) {
        uint2 c = ptx::lds64(cs), k = ptx::lds64(key);
        ptx::residual4(c.x, k.x, w[0], w[1]);
        ptx::residual4(c.y, k.y, w[2], w[3]);
    }
};
template <>
struct RowConv<16> {
    static constexpr int kWords = 8;
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w, bool) {
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
    __device__ __forceinline__ static void run(uint32_t cs, uint32_t key, uint32_t* w, bool half2) {
        RowConv<16>::run(cs, key, w, true);
        // a right half beyond W: zeros from both frames (predicated loads), 1024 - 1024 = 0 -- no per-lane
        // branch (its divergence / reconvergence stalls cost the converters ~20% in the KEY_CHUNK loop)
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        const uint4 c = half2 ? ptx::lds128(cs + 16) : z, k = half2 ? ptx::lds128(key + 16) : z;
        ptx::residual4(c.x, k.x, w[8], w[9]);
        ptx::residual4(c.y, k.y, w[10], w[11]);
        ptx::residual4(c.z, k.z, w[12], w[13]);
        ptx::residual4(c.w, k.w, w[14], w[15]);
    }
};

// Same as RowConv, with the key row's u8 words already in registers (kw: B/4 words).
template <int B>
struct RowConvK;
template <>
struct RowConvK<8> {
    __device__ __forceinline__ static void run(uint32_t cs, const uint32_t* kw, uint32_t* w, bool) {
        uint2 c = ptx::lds64(cs);
        ptx::residual4(c.x, kw[0], w[0], w[1]);
        ptx::residual4(c.y, kw[1], w[2], w[3]);
    }
};
template <>
struct RowConvK<16> {
    __device__ __forceinline__ static void run(uint32_t cs, const uint32_t* kw, uint32_t* w, bool) {
        uint4 c = ptx::lds128(cs);
        ptx::residual4(c.x, kw[0], w[0], w[1]);
        ptx::residual4(c.y, kw[1], w[2], w[3]);
        ptx::residual4(c.z, kw[2], w[4], w[5]);
        ptx::residual4(c.w, kw[3], w[6], w[7]);
    }
};
template <>
struct RowConvK<32> {
    __device__ __forceinline__ static void run(uint32_t cs, const uint32_t* kw, uint32_t* w, bool half2) {
        RowConvK<16>::run(cs, kw, w, true);
        const uint4 c = half2 ? ptx::lds128(cs + 16) : make_uint4(0u, 0u, 0u, 0u);
        ptx::residual4(c.x, half2 ? kw[4] : 0u, w[8], w[9]);
        ptx::residual4(c.y, half2 ? kw[5] : 0u, w[10], w[11]);
        ptx::residual4(c.z, half2 ? kw[6] : 0u, w[12], w[13]);
        ptx::residual4(c.w, half2 ? kw[7] : 0u, w[14], w[15]);
    }
};

// KEY_CHUNK, B = 32: the residual words of one row of 32 pixels (u8 words cw[0..7], loaded earlier)
// against the row's pre-expanded key (kx[2q], kx[2q+1] = magic2 of key word q).
// A right half beyond W needs no special case here: the caller loads zeros for it from BOTH frames, and
// 1024 - 1024 = 0 (a per-lane branch in this loop cost ~20% of the converters' time: divergence and
// reconvergence stalls around every row).
__device__ __forceinline__ void row32_vs_kexp(const uint32_t* cw, const uint32_t* kx, uint32_t (&w)[16]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) ptx::residual4x(cw[q], kx[2 * q], kx[2 * q + 1], w[2 * q], w[2 * q + 1]);
}

// u8 words of one row segment of B pixels (B/4 words) from SMEM
template <int B>
__device__ __forceinline__ void load_row_words(uint32_t addr, uint32_t* kw) {
    if constexpr (B == 8) {
        uint2 k = ptx::lds64(addr);
        kw[0] = k.x;
        kw[1] = k.y;
    } else {
#pragma unroll
        for (int h = 0; h < B / 16; ++h) {
            uint4 k = ptx::lds128(addr + 16 * h);
            kw[4 * h] = k.x;
            kw[4 * h + 1] = k.y;
            kw[4 * h + 2] = k.z;
            kw[4 * h + 3] = k.w;
        }
    }
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                 : "=r"(pred));
    return pred != 0;
}

// KS MMAs of one fold of one K-chunk, straight-line: A advances 8 TMEM columns (16 fp16) per
// K step, Phi's descriptor advances 2 core matrices.  Called by one elected thread.
template <int KS>
__device__ __forceinline__ void issue_chunk(uint32_t d, uint32_t a, uint64_t bdesc, uint64_t bstep, uint32_t idesc,
                                            uint32_t acc0) {
#pragma unroll
    for (int s = 0; s < KS; ++s)
        ptx::mma_f16_ts(d, a + (uint32_t)(s * 8), bdesc + (uint64_t)s * bstep, idesc, s == 0 ? acc0 : 1u);
}

// Epilogue helper: a warp's 32 accumulator rows x CW columns (CW = 16 or 32) -> global, through a
// 4 KB XOR-swizzled SMEM tile so every st.global.v4 writes whole 64/128-byte row segments.
// v = this lane's CW values (its row); rows r < rows_valid are stored at dst_row0 + r*M + col.
template <int CW>
__device__ __forceinline__ void stage_store(const uint32_t* v, uint32_t tile, uint32_t lane, float* dst_row0, int M,
                                            int j0, int rows_valid, bool skip) {
    constexpr int CPR = CW / 4;           // 16-byte chunks per row
    constexpr uint32_t PITCH = CW * 4;    // staged row pitch
    constexpr int RPI = 32 / CPR;         // rows per store instruction
#pragma unroll
    for (int q = 0; q < CPR; ++q) {
        const int slot = (CPR == 8) ? (q ^ (int)(lane & 7u)) : (q ^ (int)((lane >> 1) & 3u));
        ptx::sts128(tile + lane * PITCH + (uint32_t)slot * 16u, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncwarp();
    const int cc = (int)(lane % CPR);
    const int col = j0 + cc * 4;
    const int rsub = (int)(lane / CPR);
#pragma unroll
    for (int it = 0; it < CPR; ++it) {
        const int r = it * RPI + rsub;
        const int slot = (CPR == 8) ? (cc ^ (r & 7)) : (cc ^ ((r >> 1) & 3));
        uint4 t = ptx::lds128(tile + (uint32_t)r * PITCH + (uint32_t)slot * 16u);
        if (r < rows_valid && col < M && !skip) ptx::stg128(dst_row0 + (long long)r * M + col, t.x, t.y, t.z, t.w);
    }
    __syncwarp();
}

// f1 epilogue helper: a warp's 32 rows x (4*CPR) 32-bit words of packed int16 codes -> global through
// the same 4 KB swizzled SMEM tile (CPR 16-byte chunks per row, CPR = 2 or 4).  dst_row0 points at
// row 0's word col0w; rows are row_words apart; chunk cc is stored if col0w + 4*cc < valid_words.
template <int CPR>
__device__ __forceinline__ void stage_store_codes(const uint32_t* w, uint32_t tile, uint32_t lane, uint32_t* dst_row0,
                                                  int row_words, int col0w, int valid_words, int rows_valid) {
    constexpr uint32_t PITCH = CPR * 16;
    constexpr int RPI = 32 / CPR;
#pragma unroll
    for (int q = 0; q < CPR; ++q) {
        const int slot = (CPR == 4) ? (q ^ (int)((lane >> 1) & 3u)) : (q ^ (int)((lane >> 2) & 1u));
        ptx::sts128(tile + lane * PITCH + (uint32_t)slot * 16u, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
    __syncwarp();
    const int cc = (int)(lane % CPR);
    const int rsub = (int)(lane / CPR);
    const bool col_ok = col0w + 4 * cc < valid_words;
#pragma unroll
    for (int it = 0; it < CPR; ++it) {
        const int r = it * RPI + rsub;
        const int slot = (CPR == 4) ? (cc ^ ((r >> 1) & 3)) : (cc ^ ((r >> 2) & 1));
        uint4 t = ptx::lds128(tile + (uint32_t)r * PITCH + (uint32_t)slot * 16u);
        if (r < rows_valid && col_ok) ptx::stg128(dst_row0 + (long long)r * row_words + 4 * cc, t.x, t.y, t.z, t.w);
    }
    __syncwarp();
}

// y -> 16-bit code, SPEC.md:154-162 round(y / scale), evaluated as round-half-even of the exact
// product y * inv with inv = fl32(1 / scale) (R18): one FFMA against 1.5 * 2^23 puts
// the rounded integer in the low mantissa bits (|y * inv| <= 32767 * (1 + 2^-22) << 2^22), whose
// low 16 bits are the int16 two's-complement code.  No clamp is reachable: |y| <= amax, so
// |y * inv| < 32767.5.
__device__ __forceinline__ uint32_t q16_bits(uint32_t ybits, float inv) {
    return __float_as_uint(__fmaf_rn(__uint_as_float(ybits), inv, 12582912.0f));
}
__device__ __forceinline__ uint32_t q16_pack(uint32_t y0, uint32_t y1, float inv) {
    return ptx::prmt(q16_bits(y0, inv), q16_bits(y1, inv), 0x5410u);
}
__device__ __forceinline__ float q16_scale(uint32_t amax_bits) {
    return amax_bits == 0 ? 1.0f : __fdiv_rn(__uint_as_float(amax_bits), 32767.0f);
}
__device__ __forceinline__ float q16_inv(float scale) { return __frcp_rn(scale); }

template <int B, int KM, int EPI>
__global__ void __launch_bounds__(threads_for<KM>(), 1) cs_measure_kernel(const __grid_constant__ KParamsFor<KM> p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const uint8_t* const smem_ptr = smem_raw + (sbase - ptx::smem_addr(smem_raw));   // sbase as a C++ pointer
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (threadIdx.x == 0) trace_ev(p, EV_K_START, 0);
#if CSENC_DEBUG
    const int dbg_load_only = p.dbg_load_only, dbg_flags = p.dbg_flags;
#else
    constexpr int dbg_load_only = 0, dbg_flags = 0;
#endif

    // barrier block at sbase: [stage_full x8][stage_empty x8][key_full x2][key_empty x2]
    //                         [a_full x4][a_empty x4][d_full x4][d_empty x4][phi_full][tmem slot]
    const uint32_t bar_stage_full = sbase;
    const uint32_t bar_stage_empty = sbase + 8 * kMaxStages;
    const uint32_t bar_key_full = sbase + 16 * kMaxStages;
    const uint32_t bar_key_empty = bar_key_full + 16;
    const uint32_t bar_a_full = bar_key_full + 32;
    const uint32_t bar_a_empty = bar_a_full + 8 * kMaxTmemBufs;
    const uint32_t bar_d_full = bar_a_empty + 8 * kMaxTmemBufs;
    const uint32_t bar_d_empty = bar_d_full + 8 * kMaxTmemBufs;
    const uint32_t bar_phi = bar_d_empty + 8 * kMaxTmemBufs;
    const uint32_t tmem_slot = bar_phi + 8;
    const uint32_t bar_phi_empty = bar_phi + 16;   // per-GOP Phi: MMAs on the current Phi done
    // per-GOP Phi with two resident slots: slot 1's full / empty barriers (bytes 992..1007 of the barrier
    // page: past the Q_ROW slots)
    const uint32_t bar_phi2 = sbase + 992, bar_phi_empty2 = sbase + 1000;
    static_assert(kRowSlotOff + 3 * kRowSlots * 4 <= 992, "row slots overlap the second Phi slot's barriers");
    const uint32_t s_phi = sbase + p.off_phi;
    // Phi streaming and 4-D strip boxes only exist for multi-chunk plans, which never hold the key in
    // registers: compiled out of the KEY_REGS instantiations (their code stays as small as before).
    // KEY_STREAMED: the chunk's Phi K-slice rides in every stage (freed by the MMA's commit too);
    // KEY_CHUNK: it is loaded once per (unit, chunk) into a double-buffered region at off_key
    // (slice_full / slice_empty = the key_full / key_empty barriers, unused by this mode otherwise).
    const bool phi_stream = KM == KEY_STREAMED && p.phi_stream;
    const bool phi_slices = KM == KEY_CHUNK && p.phi_stream;
    const CUtensorMap* smap = nullptr;
    if constexpr (KM == KEY_STREAMED || KM == KEY_CHUNK) smap = &p.smap;
    const uint32_t s_key = sbase + p.off_key;
    const uint32_t s_stage = sbase + p.off_stage;
    CS_CHECK(p.off_stage + (uint32_t)p.n_stages * p.stage_bytes <= p.smem_bytes);
    CS_CHECK(p.set_bytes * (KM == KEY_STREAMED ? 2u : 1u) <= p.stage_bytes);
    CS_CHECK((KM != KEY_RESIDENT && !phi_slices) || p.off_key + 2u * p.key_bytes <= p.off_stage);
    CS_CHECK(!phi_slices || p.phi_slice_bytes <= p.key_bytes);
    CS_CHECK(KM != KEY_CHUNK || (p.cs_per_unit <= p.n_dbuf && p.n_stages >= 3));
    CS_CHECK(p.n_abuf * p.a_cols + p.n_dbuf * p.d_cols <= (int)kTmemCols);

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(bar_stage_full + 8 * i, 1);
            ptx::mbar_init(bar_stage_empty + 8 * i, kConvWarps + (phi_stream ? 1 : 0));
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar_key_full + 8 * i, 1);
            ptx::mbar_init(bar_key_empty + 8 * i, phi_slices ? 2 : kConvWarps);   // slice freed by both MMA warps' commits
        }
        for (int i = 0; i < kMaxTmemBufs; ++i) {
            ptx::mbar_init(bar_a_full + 8 * i, kConvWarps);
            ptx::mbar_init(bar_a_empty + 8 * i, 1);
            ptx::mbar_init(bar_d_full + 8 * i, 1);
            ptx::mbar_init(bar_d_empty + 8 * i, 4);
        }
        ptx::mbar_init(bar_phi, 1);
        ptx::mbar_init(bar_phi_empty, KM == KEY_CHUNK ? 2 : 1);   // (KEY_CHUNK: one commit per MMA warp)
        ptx::mbar_init(bar_phi2, 1);
        ptx::mbar_init(bar_phi_empty2, KM == KEY_CHUNK ? 2 : 1);
        if (EPI == EPI_Q16RR || EPI == EPI_Q16RR64)
            for (int i = 0; i < kRowBufs; ++i) ptx::mbar_init(sbase + kRowBarOff + 8 * i, 4);   // row_full
        ptx::fence_mbarrier_init();
        trace_ev(p, EV_K_START, 1);   // (prologue split: barriers initialised)
    }
    if (warp == kMmaWarp) {
        ptx::tmem_alloc(tmem_slot, kTmemCols);
        ptx::tmem_relinquish();
        if (lane == 0) trace_ev(p, EV_K_START, 2);   // TMEM allocated
    }
    if (warp < 4) {
        // Per (fold, lane) table: byte offset of the lane's block (its row 0 in the chunk) inside
        // a stage, and meta = row offset of the block within the tile | B=32 right-half-valid
        // (bit 16) | lane-valid (bit 17).
        const int lane_idx = threadIdx.x;                            // physical TMEM lane
        const int lq = (lane_idx >> 5) * p.Lq + (lane_idx & 31);     // logical lane
        for (int f = 0; f < p.F; ++f) {
            uint32_t off = 0, meta = 0;
            const int b = f * p.L + lq;
            if ((lane_idx & 31) < p.Lq && lq < p.L && b < p.T_r * p.nbx) {
                const int brow = b / p.nbx, bx = b - brow * p.nbx;
                const int pc = p.single_piece ? 0 : brow;
                const int row = p.single_piece ? brow * B : 0;
                off = (uint32_t)pc * p.piece_bytes + (uint32_t)(row * p.W + bx * B);
                meta = (uint32_t)(brow * B) | ((bx * B + B <= p.W) ? (1u << 16) : 0u) | (1u << 17);
            }
            const uint32_t e = sbase + p.off_tab + (uint32_t)(f * 128 + lane_idx) * 8u;
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(e), "r"(off), "r"(meta));
        }
        if (threadIdx.x == 0) trace_ev(p, EV_K_START, 4);   // converter offset table written
    }
    if (EPI == EPI_Q16R && threadIdx.x < 3 * kRowSlots) ptx::sts32(sbase + kRowSlotOff + threadIdx.x * 4u, 0u);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    // Programmatic dependent launch: the next kernel of the stream may be scheduled from here on (its CTAs
    // start as this kernel's CTAs leave their SMs and run their own prologue); this kernel touches global
    // memory (frames, keys, Phi in; measurements out; trace) only after the previous kernel has completed.
    ptx::grid_dep_launch();
    if (!p.pdl_early) ptx::grid_dep_wait();   // (pdl_early: the epilogue warps wait, before their first global access)
    if (threadIdx.x == 0) trace_ev(p, EV_K_START, 3);   // all warps through the prologue barrier
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));

    const uint32_t a_col0 = 0;
    const uint32_t d_col0 = (uint32_t)(p.n_abuf * p.a_cols);

    if (warp == kProducerWarp) {
        // ================================================================ TMA producer
        // Warp-uniform schedule walk (keeps addresses in uniform registers); one elected lane
        // issues the copies.
        const uint64_t pol_stream = ptx::policy_evict_first();
        const uint64_t pol_key = ptx::policy_evict_last();
        const size_t frame_bytes = (size_t)p.W * (size_t)p.H;
        if (p.n_phis == 0 && !phi_stream && !phi_slices) {
            if (elect_one()) {
                ptx::mbar_arrive_expect_tx(bar_phi, p.phi_bytes);
                ptx::bulk_load(s_phi, p.phi, p.phi_bytes, bar_phi);
            }
            __syncwarp();
        }
        if (lane == 0) trace_ev(p, EV_K_START, 5);   // producer: Phi issued, schedule walk starts
        int pb = 0;          // KEY_CHUNK phi_slices: slice buffer and its phase
        uint32_t pbph = 0;
        int phi_cur = -1;
        uint32_t phi_loads = 0;
        int st = 0;
        uint32_t ph = 0;
        int kb = 0;
        uint32_t kph = 0;
        int n_items = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            const uint8_t* const phi_src = reinterpret_cast<const uint8_t*>(p.n_phis > 0 ? p.phis + (size_t)(w.g % p.n_phis) * (p.phi_bytes / 2) : p.phi);
            if (p.n_phis > 0 && !phi_stream && !phi_slices) {   // per-GOP Phi: reload when the GOP's matrix differs from the resident one
                const int gsel = w.g % p.n_phis;
                if (gsel != phi_cur) {
                    // load k = phi_loads goes to slot k & 1 (two slots) or slot 0; it waits until the MMAs
                    // on the slot's previous matrix (load k - 2, or k - 1 with one slot) have completed
                    const uint32_t k = phi_loads;
                    const bool two = p.off_phi2 != 0;
                    const uint32_t slot = two ? (k & 1u) : 0u;
                    const uint32_t full = slot ? bar_phi2 : bar_phi, empty = slot ? bar_phi_empty2 : bar_phi_empty;
                    if (two ? k >= 2 : k > 0) ptx::mbar_wait(empty, (two ? (k - 2u) >> 1 : k - 1u) & 1u);
                    if (elect_one()) {
                        ptx::mbar_arrive_expect_tx(full, p.phi_bytes);
                        ptx::bulk_load(slot ? sbase + p.off_phi2 : s_phi,
                                       reinterpret_cast<const uint8_t*>(p.phis) + (size_t)gsel * p.phi_bytes,
                                       p.phi_bytes, full);
                    }
                    __syncwarp();
                    phi_cur = gsel;
                    ++phi_loads;
                }
            }
            const int key_idx = key_frame(p, w);
            const uint8_t* const raw_key = p.frames + (size_t)key_idx * frame_bytes;
            const int keyf_idx = p.keys ? -1 : key_idx;   // decoded keys live in another buffer: bulk copies
            const uint8_t* const key_f =
                p.keys ? p.keys + ((size_t)w.s * p.n_gops_T + (size_t)w.g) * frame_bytes : raw_key;
            if constexpr (KM == KEY_REGS) {  // the key strip is the unit's first ring item
                ptx::mbar_wait(bar_stage_empty + 8 * st, ph ^ 1u);
                if (elect_one()) {
                    ptx::mbar_arrive_expect_tx(bar_stage_full + 8 * st, p.set_bytes);
                    load_strips<B>(p, s_stage + (uint32_t)st * p.stage_bytes, key_f, w.t, 0, bar_stage_full + 8 * st,
                                   pol_key);   // (KEY_REGS plans are single-piece: plain bulk copy)
                }
                __syncwarp();
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
            } else if constexpr (KM == KEY_RESIDENT) {
                ptx::mbar_wait(bar_key_empty + 8 * kb, kph ^ 1u);
                if (elect_one()) {
                    ptx::mbar_arrive_expect_tx(bar_key_full + 8 * kb, (uint32_t)p.n_chunks * p.set_bytes);
                    for (int k = 0; k < p.n_chunks; ++k)
                        load_strips<B>(p, s_key + (uint32_t)kb * p.key_bytes + (uint32_t)k * p.stage_cs_bytes, key_f,
                                       w.t, k, bar_key_full + 8 * kb, pol_key);
                }
                __syncwarp();
                kb ^= 1;
                if (kb == 0) kph ^= 1u;
            }
            if constexpr (KM == KEY_CHUNK) {
                // chunk-outer order: per chunk k, (Phi slice k), key chunk k, then chunk k of every
                // CS frame of the unit -- the key chunk and the slice cross L2 -> SMEM once per unit
                if (lane == 0 && n_items == 0) trace_ev(p, EV_K_START, 6);   // first unit decoded
                for (int k = 0; k < p.n_chunks; ++k) {
                    if (phi_slices && !dbg_load_only) {   // (load-only ablation: no MMA frees the slices)
                        ptx::mbar_wait(bar_key_empty + 8 * pb, pbph ^ 1u);
                        if (elect_one()) {
                            ptx::mbar_arrive_expect_tx(bar_key_full + 8 * pb, p.phi_slice_bytes);
                            ptx::bulk_load(s_key + (uint32_t)pb * p.key_bytes, phi_src + (size_t)k * p.phi_slice_bytes,
                                           p.phi_slice_bytes, bar_key_full + 8 * pb);
                        }
                        __syncwarp();
                        if (lane == 0 && n_items == 0 && k == 0) trace_ev(p, EV_K_START, 7);   // first Phi slice issued
                        pb ^= 1;
                        if (pb == 0) pbph ^= 1u;
                    }
                    for (int c = w.c0 - 1; c < w.c1; ++c) {   // c = c0 - 1: the key chunk
                        ptx::mbar_wait(bar_stage_empty + 8 * st, ph ^ 1u);
                        if (lane == 0 && c >= w.c0) trace_ev(p, EV_P_EMPTY, n_items);
                        const uint32_t dst = s_stage + (uint32_t)st * p.stage_bytes;
                        if (elect_one()) {
                            ptx::mbar_arrive_expect_tx(bar_stage_full + 8 * st, p.set_bytes);
                            if (c < w.c0)
                                load_strips<B>(p, dst, key_f, w.t, k, bar_stage_full + 8 * st, pol_key, keyf_idx, smap);
                            else
                                load_strips<B>(p, dst, raw_key + (size_t)(1 + c) * frame_bytes, w.t, k,
                                               bar_stage_full + 8 * st, pol_stream, key_idx + 1 + c, smap);
                        }
                        __syncwarp();
                        if (lane == 0 && c >= w.c0) trace_ev(p, EV_P_ISSUED, n_items);
                        if (c >= w.c0) ++n_items;
                        if (++st == p.n_stages) {
                            st = 0;
                            ph ^= 1u;
                        }
                    }
                }
                continue;
            }
            for (int c = w.c0; c < w.c1; ++c) {
                const uint8_t* cs_f = raw_key + (size_t)(1 + c) * frame_bytes;
                for (int k = 0; k < p.n_chunks; ++k) {
                    ptx::mbar_wait(bar_stage_empty + 8 * st, ph ^ 1u);
                    if (lane == 0) trace_ev(p, EV_P_EMPTY, n_items);
                    const uint32_t dst = s_stage + (uint32_t)st * p.stage_bytes;
                    if (elect_one()) {
                        ptx::mbar_arrive_expect_tx(bar_stage_full + 8 * st,
                                                   (KM == KEY_STREAMED ? 2u : 1u) * p.set_bytes + (phi_stream ? p.phi_slice_bytes : 0u));
                        if (phi_stream)   // this chunk's K-slice of Phi (L2-resident)
                            ptx::bulk_load(dst + p.stage_phi_off, phi_src + (size_t)k * p.phi_slice_bytes, p.phi_slice_bytes,
                                           bar_stage_full + 8 * st);
                        load_strips<B>(p, dst, cs_f, w.t, k, bar_stage_full + 8 * st, pol_stream, key_idx + 1 + c, smap);
                        if constexpr (KM == KEY_STREAMED)   // chained (Eq. 3 literal): reference = previous frame
                            load_strips<B>(p, dst + p.stage_cs_bytes, p.chained ? cs_f - frame_bytes : key_f, w.t, k,
                                           bar_stage_full + 8 * st, pol_key, p.chained ? key_idx + c : keyf_idx, smap);
                    }
                    __syncwarp();
                    if (lane == 0) trace_ev(p, EV_P_ISSUED, n_items);
                    ++n_items;
                    if (++st == p.n_stages) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if ((warp == kMmaWarp || (KM == KEY_CHUNK && warp == kMmaWarp + 1)) && !dbg_load_only) {
        // ================================================================ MMA issuer
        // The whole warp walks the schedule (warp-uniform control flow keeps every operand in
        // uniform registers); one elected lane issues the tcgen05 instructions.
        // KEY_CHUNK: two issuing warps (mw = 0 / 1) walk the same schedule and take alternate items.  An
        // accumulator's chunks stay in K order without any handshake between the warps: a frame's next
        // chunk is the unit's item i + U, converted after item i + 2 was started, which needed item i's
        // A buffer back, i.e. item i's MMAs completed (n_abuf = 2) -- so it holds whenever U >= n_abuf,
        // and for even U both chunks belong to the same warp anyway; other units (U = 1 ...) are issued
        // by warp 0 alone.  The results are bitwise those of one issuing warp.
        const int mw = warp - kMmaWarp;
        if (p.n_phis == 0 && !phi_stream && !phi_slices) {
            ptx::mbar_wait(bar_phi, 0);
            ptx::tc_fence_after();
        }
        int pb = 0;    // KEY_CHUNK phi_slices: slice buffer and its phase
        uint32_t pbph = 0;
        uint32_t d_use = 0;   // KEY_CHUNK: per accumulator slot, parity of its uses so far (bit db)
        int pst = 0;   // phi_stream: stage of the current chunk (one stage per chunk: KM 0/1)
        uint32_t pph = 0;
        int phi_cur = -1;
        uint32_t phi_waits = 0;
        int ab = 0, db = 0;
        uint32_t aph = 0, dph = 0;
        const int ksteps = p.chunk_k / 16;
        // descriptor of Phi's first K step; K step kg starts 2*kg core matrices (2*kg*lbo bytes)
        // further, i.e. +2*lbo>>4 in the 14-bit start-address field (no carry: smem < 256 KB)
        uint64_t desc0 = ptx::smem_desc_noswizzle(s_phi, p.lbo, p.sbo);   // (per-GOP Phi: the current slot's)
        const uint64_t desc_step = (uint64_t)((2u * p.lbo) >> 4);
        const uint64_t desc_chunk = desc_step * (uint64_t)ksteps;
        const uint32_t a_fold = (uint32_t)(p.chunk_k / 2);
        int n_items = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            if (p.n_phis > 0 && !phi_stream && !phi_slices) {
                const int gsel = w.g % p.n_phis;
                if (gsel != phi_cur) {
                    // release the slot of the previous matrix once every MMA issued so far has completed,
                    // then wait for the next one (load k = phi_waits, in slot k & 1 with two slots)
                    const uint32_t k = phi_waits;
                    const bool two = p.off_phi2 != 0;
                    const uint32_t slot = two ? (k & 1u) : 0u;
                    if (k > 0) {
                        const uint32_t prev = two ? ((k - 1u) & 1u) : 0u;
                        if (elect_one()) ptx::tc_commit(prev ? bar_phi_empty2 : bar_phi_empty);
                        __syncwarp();
                    }
                    ptx::mbar_wait(slot ? bar_phi2 : bar_phi, (two ? k >> 1 : k) & 1u);
                    ptx::tc_fence_after();
                    desc0 = ptx::smem_desc_noswizzle(slot ? sbase + p.off_phi2 : s_phi, p.lbo, p.sbo);
                    phi_cur = gsel;
                    ++phi_waits;
                }
            }
            if constexpr (KM == KEY_CHUNK) {
                // chunk-outer: frame j of the unit accumulates into slot (db + j) % n_dbuf over all
                // chunks; its d_full is committed with its last chunk (the epilogue takes the
                // frames in the same order as every other mode)
                const int U = w.c1 - w.c0;
                const bool two = U >= p.n_abuf || (U & 1) == 0;   // alternate items between the two warps
                for (int k = 0; k < p.n_chunks; ++k) {
                    uint64_t dk = desc0 + (uint64_t)k * desc_chunk;
                    if (phi_slices) {
                        ptx::mbar_wait(bar_key_full + 8 * pb, pbph);
                        dk = ptx::smem_desc_noswizzle(s_key + (uint32_t)pb * p.key_bytes, p.lbo, p.sbo);
                    }
                    int dj = db;
                    for (int j = 0; j < U; ++j) {
                        const bool mine = two ? ((n_items & 1) == mw) : (mw == 0);
                        if (mine && k == 0) {
                            ptx::mbar_wait(bar_d_empty + 8 * dj, ((d_use >> dj) & 1u) ^ 1u);
                        }
                        if (mine) {
                        ptx::mbar_wait(bar_a_full + 8 * ab, aph);
                        ptx::tc_fence_after();
                        if (lane == 0) trace_ev(p, EV_M_AFULL, n_items);
                        const uint32_t d_tm = tmem_base + d_col0 + (uint32_t)dj * (uint32_t)p.d_cols;
                        const uint32_t a_tm = tmem_base + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                        const uint32_t acc0 = k > 0 ? 1u : 0u;
                        if (elect_one()) {
                            for (int f = 0; f < p.F; ++f) {
                                const uint32_t d_f = d_tm + (uint32_t)(f * p.Mpad);
                                const uint32_t a_f = a_tm + (uint32_t)f * a_fold;
                                switch (ksteps) {
                                    case 4: issue_chunk<4>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                    case 8: issue_chunk<8>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                    case 16: issue_chunk<16>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                    default:
                                        for (int s2 = 0; s2 < ksteps; ++s2)
                                            ptx::mma_f16_ts(d_f, a_f + (uint32_t)(s2 * 8), dk + (uint64_t)s2 * desc_step,
                                                            p.idesc, (k > 0 || s2 > 0) ? 1u : 0u);
                                }
                            }
                            ptx::tc_commit(bar_a_empty + 8 * ab);
                            if (k == p.n_chunks - 1) ptx::tc_commit(bar_d_full + 8 * dj);
                        }
                        __syncwarp();
                        if (lane == 0) trace_ev(p, EV_M_ISSUED, n_items);
                        }
                        if (k == p.n_chunks - 1) d_use ^= 1u << dj;
                        ++n_items;
                        if (++ab == p.n_abuf) {
                            ab = 0;
                            aph ^= 1u;
                        }
                        if (++dj == p.n_dbuf) dj = 0;
                    }
                    if (phi_slices) {   // every MMA of this chunk issued: the slice buffer may be refilled
                        if (elect_one()) ptx::tc_commit(bar_key_empty + 8 * pb);
                        __syncwarp();
                        pb ^= 1;
                        if (pb == 0) pbph ^= 1u;
                    }
                }
                db = (db + U) % p.n_dbuf;
                continue;
            }
            for (int c = w.c0; c < w.c1; ++c) {
                ptx::mbar_wait(bar_d_empty + 8 * db, dph ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d_tm = tmem_base + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                uint64_t dk = desc0;
                for (int k = 0; k < p.n_chunks; ++k, dk += desc_chunk) {
                    ptx::mbar_wait(bar_a_full + 8 * ab, aph);
                    if (phi_stream) {   // the chunk's Phi slice rides in its stage (landed: the converters saw it)
                        ptx::mbar_wait(bar_stage_full + 8 * pst, pph);
                        dk = ptx::smem_desc_noswizzle(s_stage + (uint32_t)pst * p.stage_bytes + p.stage_phi_off, p.lbo, p.sbo);
                    }
                    ptx::tc_fence_after();
                    if (lane == 0) trace_ev(p, EV_M_AFULL, n_items);
                    const uint32_t a_tm = tmem_base + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                    const uint32_t acc0 = k > 0 ? 1u : 0u;
                    if (elect_one()) {
                        for (int f = 0; f < p.F; ++f) {
                            const uint32_t d_f = d_tm + (uint32_t)(f * p.Mpad);
                            const uint32_t a_f = a_tm + (uint32_t)f * a_fold;
                            switch (ksteps) {
                                case 4: issue_chunk<4>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                case 8: issue_chunk<8>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                case 16: issue_chunk<16>(d_f, a_f, dk, desc_step, p.idesc, acc0); break;
                                default:
                                    for (int s2 = 0; s2 < ksteps; ++s2)
                                        ptx::mma_f16_ts(d_f, a_f + (uint32_t)(s2 * 8), dk + (uint64_t)s2 * desc_step,
                                                        p.idesc, (k > 0 || s2 > 0) ? 1u : 0u);
                            }
                        }
                        ptx::tc_commit(bar_a_empty + 8 * ab);
                        if (phi_stream) ptx::tc_commit(bar_stage_empty + 8 * pst);   // slice read: stage may go
                    }
                    __syncwarp();
                    if (phi_stream && ++pst == p.n_stages) {
                        pst = 0;
                        pph ^= 1u;
                    }
                    if (lane == 0) trace_ev(p, EV_M_ISSUED, n_items);
                    ++n_items;
                    if (++ab == p.n_abuf) {
                        ab = 0;
                        aph ^= 1u;
                    }
                }
                if (elect_one()) ptx::tc_commit(bar_d_full + 8 * db);
                __syncwarp();
                if (++db == p.n_dbuf) {
                    db = 0;
                    dph ^= 1u;
                }
            }
        }
    } else if (warp < kConvWarps) {
        // ================================================================ converters (a2 + a3)
        const int wg = warp >> 2;                                // converter warpgroup 0/1
        const int lane_idx = (warp & 3) * 32 + (int)lane;       // TMEM lane = block slot
        const uint32_t lane_bits = (uint32_t)((warp & 3) * 32) << 16;
        constexpr int kWords = RowConv<B>::kWords;      // fp16x2 words per pixel row
        constexpr int kRowsPerSt = 32 / kWords;         // rows per 32-column TMEM store
        const int groups = p.chunk_rows / kRowsPerSt;   // row groups per fold per chunk
        const int n_groups = p.F * groups;
        int st = 0, ab = 0, kb = 0;
        uint32_t ph = 0, aph = 0, kph = 0;
        int n_items = 0;
        const bool tr = (warp == 0 && lane == 0);
        const uint32_t tab_lane = sbase + p.off_tab + (uint32_t)lane_idx * 8u;
        // KEY_REGS: this thread's key rows for its (<= 2) row groups, u8 words; the groups'
        // geometry is constant for the whole kernel
        uint32_t kreg[2][16];
        uint32_t g_off[2] = {0, 0}, g_acol[2] = {0, 0};
        bool g_half2[2] = {true, true};
        // KEY_CHUNK with swizzled strips: byte offset of the left 16 bytes of row rr of group j inside a stage
        // (the right 16 bytes are at offset ^ 16); stages are 1024-B aligned, so the swizzle is a function
        // of the offset alone
        uint32_t g_swz[2][2] = {{0, 0}, {0, 0}}, g_swr[2][2] = {{0, 0}, {0, 0}};   // left / right 16 bytes
        if constexpr (KM == KEY_REGS || KM == KEY_CHUNK) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int g = wg + 2 * j;
                if (g < n_groups) {
                    const int f = g / groups, r0 = (g - f * groups) * kRowsPerSt;
                    uint32_t meta;
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                                 : "=r"(g_off[j]), "=r"(meta)
                                 : "r"(tab_lane + (uint32_t)(f * 1024)));
                    g_off[j] += (uint32_t)(r0 * p.W);
                    g_half2[j] = (meta >> 16) & 1u;
                    g_acol[j] = (uint32_t)(f * (p.chunk_k / 2) + r0 * kWords);
                    if constexpr (KM == KEY_CHUNK) {
#pragma unroll
                        for (int rr = 0; rr < 2; ++rr) {
                            const uint32_t lin = g_off[j] + (uint32_t)(rr * p.W);
                            const uint32_t sw = p.tma_strips == 2 ? ((lin >> 7) & 7u) << 4 : 0u;
                            g_swz[j][rr] = lin ^ sw;
                            g_swr[j][rr] = (lin + 16u) ^ sw;
                        }
                    }
                }
            }
        }
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            if constexpr (KM == KEY_CHUNK) {
                // per chunk: the key chunk's rows of this thread's (<= 2) row groups into registers,
                // already expanded to the fp16 "magic" operand form (the expansion is paid once per
                // unit and chunk, not once per CS frame), then chunk k of every CS frame of the unit
                static_assert(KM != KEY_CHUNK || B == 32, "KEY_CHUNK is instantiated for B = 32");
                for (int k = 0; k < p.n_chunks; ++k) {
                    uint32_t kx[2][32];
                    ptx::mbar_wait(bar_stage_full + 8 * st, ph);
                    {
                        const uint32_t kbase = s_stage + (uint32_t)st * p.stage_bytes;
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            if (wg + 2 * j < n_groups) {
#pragma unroll
                                for (int rr = 0; rr < kRowsPerSt; ++rr) {
                                    uint32_t kw[8];
                                    {
                                        const uint4 a = ptx::lds128(kbase + g_swz[j][rr]);
                                        const uint4 b = g_half2[j] ? ptx::lds128(kbase + g_swr[j][rr]) : make_uint4(0u, 0u, 0u, 0u);
                                        kw[0] = a.x, kw[1] = a.y, kw[2] = a.z, kw[3] = a.w;
                                        kw[4] = b.x, kw[5] = b.y, kw[6] = b.z, kw[7] = b.w;
                                    }
#pragma unroll
                                    for (int q = 0; q < 8; ++q) ptx::magic2(kw[q], kx[j][rr * 16 + 2 * q], kx[j][rr * 16 + 2 * q + 1]);
                                }
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(bar_stage_empty + 8 * st);
                    if (++st == p.n_stages) {
                        st = 0;
                        ph ^= 1u;
                    }
                    for (int c = w.c0; c < w.c1; ++c) {
                        if (dbg_load_only) {
                            ptx::mbar_wait(bar_stage_full + 8 * st, ph);
                            if (tr) trace_ev(p, EV_C_FULL, n_items);
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(bar_stage_empty + 8 * st);
                            if (++st == p.n_stages) {
                                st = 0;
                                ph ^= 1u;
                            }
                            ++n_items;
                            continue;
                        }
                        // the strip has usually landed and the A buffer is usually free: probe both at once
#if defined(CSENC_INJECT_RACE)
                        ptx::mbar_wait(bar_stage_full + 8 * st, ph);
#else
                        ptx::mbar_wait2(bar_stage_full + 8 * st, ph, bar_a_empty + 8 * ab, aph ^ 1u);
#endif
                        if (tr) trace_ev(p, EV_C_FULL, n_items);
                        ptx::tc_fence_after();
                        if (tr) trace_ev(p, EV_C_AEMPTY, n_items);
                        const uint32_t cs_base = s_stage + (uint32_t)st * p.stage_bytes;
                        const uint32_t a_tm = tmem_base + lane_bits + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                        // per row group: both rows loaded (plain C++ shared loads after the stage-full
                        // wait, so the compiler can issue them together), then the residual words and
                        // the TMEM stores
                        const uint8_t* const cs_ptr = smem_ptr + (cs_base - sbase);
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            if (wg + 2 * j < n_groups) {
                                // the CS part of the slot (pieces 128-B aligned); a right half beyond W is not read
                                CS_CHECK(g_off[j] + (uint32_t)((kRowsPerSt - 1) * p.W + (g_half2[j] ? B : B / 2)) <= p.stage_cs_bytes);
                                CS_CHECK(g_acol[j] + 32u <= (uint32_t)p.a_cols);
                                uint32_t cw[kRowsPerSt][8];
#pragma unroll
                                for (int rr = 0; rr < kRowsPerSt; ++rr) {
                                    const uint4 a = *reinterpret_cast<const uint4*>(cs_ptr + g_swz[j][rr]);
                                    const uint4 b = g_half2[j] ? *reinterpret_cast<const uint4*>(cs_ptr + g_swr[j][rr])
                                                               : make_uint4(0u, 0u, 0u, 0u);
                                    cw[rr][0] = a.x, cw[rr][1] = a.y, cw[rr][2] = a.z, cw[rr][3] = a.w;
                                    cw[rr][4] = b.x, cw[rr][5] = b.y, cw[rr][6] = b.z, cw[rr][7] = b.w;
                                }
#pragma unroll
                                for (int rr = 0; rr < kRowsPerSt; ++rr) {
                                    uint32_t v[16];
                                    if (dbg_flags & 2) {   // ablation: no residual ALU
#pragma unroll
                                        for (int i = 0; i < 16; ++i) v[i] = 0u;
                                    } else {
                                        row32_vs_kexp(cw[rr], &kx[j][rr * 16], v);
                                    }
                                    ptx::tmem_st_32x32b_x16(a_tm + g_acol[j] + (uint32_t)(rr * 16), v);
                                }
                            }
                        }
                        if (tr) trace_ev(p, EV_C_CONV, n_items);
                        ptx::tc_wait_st();
                        ptx::tc_fence_before();
                        if (tr) trace_ev(p, EV_C_DONE, n_items);
                        ++n_items;
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
                continue;
            }
            if constexpr (KM == KEY_RESIDENT) ptx::mbar_wait(bar_key_full + 8 * kb, kph);
            if constexpr (KM == KEY_REGS) {
                ptx::mbar_wait(bar_stage_full + 8 * st, ph);
                const uint32_t kbase = s_stage + (uint32_t)st * p.stage_bytes;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (wg + 2 * j < n_groups) {
#pragma unroll
                        for (int rr = 0; rr < kRowsPerSt; ++rr)
                            load_row_words<B>(kbase + g_off[j] + (uint32_t)(rr * p.W), &kreg[j][rr * (B / 4)]);
                    }
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_stage_empty + 8 * st);
                if (++st == p.n_stages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
            for (int c = w.c0; c < w.c1; ++c) {
                for (int k = 0; k < p.n_chunks; ++k) {
                    ptx::mbar_wait(bar_stage_full + 8 * st, ph);
                    if (tr) trace_ev(p, EV_C_FULL, n_items);
                    if (dbg_load_only) {
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(bar_stage_empty + 8 * st);
                        if (++st == p.n_stages) {
                            st = 0;
                            ph ^= 1u;
                        }
                        ++n_items;
                        continue;
                    }
                    ptx::mbar_wait(bar_a_empty + 8 * ab, aph ^ 1u);
                    ptx::tc_fence_after();
                    if (tr) trace_ev(p, EV_C_AEMPTY, n_items);
                    const uint32_t cs_base = s_stage + (uint32_t)st * p.stage_bytes;
                    const uint32_t a_tm = tmem_base + lane_bits + a_col0 + (uint32_t)ab * (uint32_t)p.a_cols;
                    if (dbg_flags & 2) {
                        uint32_t v[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0u;
                        for (int g = wg; g < n_groups; g += 2)
                            ptx::tmem_st_32x32b_x32(a_tm + (uint32_t)((g / groups) * (p.chunk_k / 2) +
                                                                       (g % groups) * kRowsPerSt * kWords),
                                                    v);
                    } else if constexpr (KM == KEY_REGS) {
                        // <= 2 row groups per warpgroup (planner guarantee); key words in kreg[j]
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            if (wg + 2 * j < n_groups) {
                                CS_CHECK(g_off[j] + (uint32_t)((kRowsPerSt - 1) * p.W + B) <= p.set_bytes);
                                CS_CHECK(g_acol[j] + 32u <= (uint32_t)p.a_cols);
                                uint32_t v[32];
#pragma unroll
                                for (int rr = 0; rr < kRowsPerSt; ++rr)
                                    RowConvK<B>::run(cs_base + g_off[j] + (uint32_t)(rr * p.W), &kreg[j][rr * (B / 4)],
                                                     v + rr * kWords, g_half2[j]);
                                ptx::tmem_st_32x32b_x32(a_tm + g_acol[j], v);
                            }
                        }
                    } else {
                        const uint32_t key_base = (KM == KEY_RESIDENT)
                                                      ? s_key + (uint32_t)kb * p.key_bytes + (uint32_t)k * p.stage_cs_bytes
                                                      : cs_base + p.stage_cs_bytes;
                        // row groups g = f*groups + gi, round-robin over the two warpgroups
                        int f = 0, gi = wg;
                        while (gi >= groups && f < p.F) {
                            gi -= groups;
                            ++f;
                        }
                        for (int g = wg; g < n_groups; g += 2) {
                            const int r0 = gi * kRowsPerSt;
                            uint32_t off, meta;
                            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                                         : "=r"(off), "=r"(meta)
                                         : "r"(tab_lane + (uint32_t)(f * 1024)));
                            off += (uint32_t)(r0 * p.W);
                            const bool half2 = (meta >> 16) & 1u;
                            CS_CHECK(off + (uint32_t)((kRowsPerSt - 1) * p.W + (half2 ? B : B / 2)) <= p.stage_cs_bytes);
                            CS_CHECK((uint32_t)(f * (p.chunk_k / 2) + r0 * kWords + 32) <= (uint32_t)p.a_cols);
                            uint32_t v[32];
#pragma unroll
                            for (int rr = 0; rr < kRowsPerSt; ++rr) {
                                const uint32_t ro = off + (uint32_t)(rr * p.W);
                                RowConv<B>::run(cs_base + ro, key_base + ro, v + rr * kWords, half2);
                            }
                            ptx::tmem_st_32x32b_x32(a_tm + (uint32_t)(f * (p.chunk_k / 2) + r0 * kWords), v);
                            gi += 2;
                            while (gi >= groups) {
                                gi -= groups;
                                ++f;
                            }
                        }
                    }
                    if (tr) trace_ev(p, EV_C_CONV, n_items);
                    ptx::tc_wait_st();
                    ptx::tc_fence_before();
                    if (tr) trace_ev(p, EV_C_DONE, n_items);
                    ++n_items;
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
            if constexpr (KM == KEY_RESIDENT) {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_key_empty + 8 * kb);
                kb ^= 1;
                if (kb == 0) kph ^= 1u;
            }
        }
    } else if (EPI != EPI_F32 && EPI != EPI_F32A && warp >= kEpiWarp0 && warp < kEpiWarp0 + 4 && !dbg_load_only) {
        // ================================================================ epilogue, 16-bit codes (f1)
        // Per item: (Q_ABSMAX) warp max of |y| -> one atomicMax per warp into amax[cs];
        // (Q_FRAME) codes with the frame's scale; (Q_ROW) pass A: per-block-row max reduced across
        // the 4 epilogue warps in SMEM slots (triple-buffered, one named barrier per item), pass B:
        // re-read the accumulators from TMEM and store codes with the row's scale.
        if (p.pdl_early) ptx::grid_dep_wait();
        const int ew = warp - kEpiWarp0;
        const int lane_idx = ew * 32 + (int)lane;
        const uint32_t lane_bits = (uint32_t)(ew * 32) << 16;
        const uint32_t stage_tile = sbase + p.off_epi + (uint32_t)ew * 4096u;
        // the mode is fixed by the instantiation where it can be (dead modes compile away)
        const int qmode = (EPI == EPI_Q16R || EPI == EPI_Q16RR || EPI == EPI_Q16RR64) ? (int)Q_ROW
                        : (p.qmode == Q_ABSMAX ? (int)Q_ABSMAX : (int)Q_FRAME);
        const int smode = (p.M == 4) ? 0 : ((p.M & 7) == 0 ? 1 : 2);   // store mode
        // Q_ROW: block row (within the tile) of this lane's block in fold f, and the warp's lowest /
        // highest row in fold f, 6 bits per fold (rows < kRowSlots <= 63; fixed for the kernel)
        uint64_t rowpack = 0, lopack = 0, hipack = 0;
        if (qmode == Q_ROW) {
            for (int f = 0; f < p.F; ++f) {
                const int b = f * p.L + ew * p.Lq + (int)lane;
                const bool ok = (int)lane < p.Lq && ew * p.Lq + (int)lane < p.L && b < p.T_r * p.nbx;
                const uint32_t r = ok ? (uint32_t)(b / p.nbx) : 63u;
                const uint32_t lo = __reduce_min_sync(0xFFFFFFFFu, r);
                const uint32_t hi = __reduce_max_sync(0xFFFFFFFFu, ok ? r : 0u);
                rowpack |= (uint64_t)r << (6 * f);
                lopack |= (uint64_t)lo << (6 * f);
                hipack |= (uint64_t)hi << (6 * f);
            }
        }
        int db = 0;
        uint32_t dph = 0;
        int n_items = 0;
        const bool tr = (warp == kEpiWarp0 && lane == 0);
        if constexpr (EPI == EPI_Q16RR || EPI == EPI_Q16RR64) {
            constexpr int NV = EPI == EPI_Q16RR ? 32 : 64;   // accumulator columns held in registers
            CS_CHECK(p.F == 1 && p.Mpad <= NV && p.Mpad == p.M && p.T_r <= kRowRegRows);
            // Q_ROW, register path (M = 16..64, one fold): the accumulator is read from TMEM once and
            // released at once; the row maxima of the 4 warps meet in SMEM behind a row_full mbarrier;
            // the codes are made from the registers.  Slot reuse: a warp writes buffer j % 4 at item j after waiting for
            // every warp's item j-1 arrival, which each warp makes after reading item j-2's slots.
            const uint32_t my_slots = stage_tile + kRowSlotTileOff;
            const uint32_t slots0 = sbase + p.off_epi + kRowSlotTileOff;   // warp k's slots: + k * 4096
            const int r_lane = (int)(rowpack & 63u);
            const int rlo = (int)(lopack & 63u), rhi = (int)(hipack & 63u);
            const int row0 = ew * p.Lq;
            const bool valid_l = (int)lane < p.Lq && row0 + (int)lane < p.L;
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                Unit w;
                if (!decode_unit(p, u, w)) continue;
                const int rows_here = min(p.T_r, p.nby - w.t * p.T_r);
                const int blocks_here = rows_here * p.nbx;
                const int blk0 = w.t * p.T_r * p.nbx;
                const bool valid = valid_l && row0 + (int)lane < blocks_here;
                for (int c = w.c0; c < w.c1; ++c) {
                    ptx::mbar_wait(bar_d_full + 8 * db, dph);
                    ptx::tc_fence_after();
                    if (tr) trace_ev(p, EV_E_DFULL, n_items);
                    const long long cs_global = (long long)w.s * p.cs_per_stream_sel +
                                                (long long)(w.g - p.gop_begin) * (p.G - 1) + c;
                    CS_CHECK((cs_global + 1) * p.nblk * (long long)p.M <= p.out_floats);
                    const uint32_t d_tm = tmem_base + lane_bits + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                    uint32_t v[NV];
                    if (NV == 32 && p.Mpad == 32) ptx::tmem_ld_32x32b_x32(d_tm, *reinterpret_cast<uint32_t(*)[32]>(v));
                    if (NV == 32 && p.Mpad == 16) ptx::tmem_ld_32x32b_x16(d_tm, *reinterpret_cast<uint32_t(*)[16]>(v));
                    if (NV == 64) {
                        ptx::tmem_ld_32x32b_x32(d_tm, *reinterpret_cast<uint32_t(*)[32]>(v));
                        if (p.Mpad == 64) ptx::tmem_ld_32x32b_x32(d_tm + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                        else ptx::tmem_ld_32x32b_x16(d_tm + 32u, *reinterpret_cast<uint32_t(*)[16]>(v + 32));
                    }
                    ptx::tc_wait_ld();
                    ptx::tc_fence_before();   // accumulator in registers: hand it back to the MMA now
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(bar_d_empty + 8 * db);
                    float mff = 0.0f;
#pragma unroll
                    for (int q = 0; q < NV; ++q)
                        if (q < p.Mpad) mff = fmaxf(mff, fabsf(__uint_as_float(v[q])));
                    const uint32_t mf = valid ? __float_as_uint(mff) : 0u;
                    // lane rr <- maximum of block row rr over this warp's lanes (0 for rows it lacks)
                    uint32_t acc = 0;
                    for (int rr = rlo; rr <= rhi; ++rr) {
                        const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, r_lane == rr ? mf : 0u);
                        if ((int)lane == rr) acc = m;
                    }
                    const uint32_t buf = (uint32_t)(n_items % kRowBufs);
                    if ((int)lane < p.T_r) ptx::sts32(my_slots + (buf * kRowRegRows + lane) * 4u, acc);
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(sbase + kRowBarOff + 8 * buf);
                    if (tr) trace_ev(p, EV_E_ARRIVED, n_items);
                    ptx::mbar_wait(sbase + kRowBarOff + 8 * buf, (uint32_t)(n_items / kRowBufs) & 1u);
                    if (tr) trace_ev(p, EV_E_ROWS, n_items);
                    // both row maxima (the scale this lane writes, the row of its block) in one round of
                    // SMEM loads: the epilogue's shared-memory traffic queues behind the converters'
                    const uint32_t a_s = slots0 + (buf * kRowRegRows + (uint32_t)min(lane_idx, p.T_r - 1)) * 4u;
                    const uint32_t a_r = slots0 + (buf * kRowRegRows + (uint32_t)(valid ? r_lane : 0)) * 4u;
                    const uint32_t s0 = ptx::lds32(a_s), s1 = ptx::lds32(a_s + 4096u), s2 = ptx::lds32(a_s + 8192u),
                                   s3 = ptx::lds32(a_s + 12288u);
                    const uint32_t q0 = ptx::lds32(a_r), q1 = ptx::lds32(a_r + 4096u), q2 = ptx::lds32(a_r + 8192u),
                                   q3 = ptx::lds32(a_r + 12288u);
                    const uint32_t m_s = max(max(s0, s1), max(s2, s3)), m_r = max(max(q0, q1), max(q2, q3));
                    if (lane_idx < rows_here) p.scales[cs_global * p.nby + w.t * p.T_r + lane_idx] = q16_scale(m_s);
                    const float inv = q16_inv(q16_scale(valid ? m_r : 0u));
                    int16_t* const codes_cs = p.codes + (cs_global * p.nblk + blk0) * (long long)p.M;
                    if constexpr (NV == 32) {
                        if (valid) {   // codes straight from registers: the lane's row is 2M <= 64 contiguous bytes
                            uint32_t* dst = reinterpret_cast<uint32_t*>(codes_cs + (long long)(row0 + (int)lane) * p.M);
#pragma unroll
                            for (int q = 0; q < NV; q += 8)
                                if (q < p.Mpad)
                                    ptx::stg128(dst + q / 2, q16_pack(v[q], v[q + 1], inv), q16_pack(v[q + 2], v[q + 3], inv),
                                                q16_pack(v[q + 4], v[q + 5], inv), q16_pack(v[q + 6], v[q + 7], inv));
                        }
                    } else {   // 96-128 B rows: through the swizzled staging tile, whole 64-B row segments per store
                        const int rows_valid = min(p.Lq, min(p.L - row0, blocks_here - row0));
#pragma unroll
                        for (int j0 = 0; j0 < NV; j0 += 32) {
                            uint32_t wd[16];
#pragma unroll
                            for (int q = 0; q < 16; ++q) wd[q] = q16_pack(v[j0 + 2 * q], v[j0 + 2 * q + 1], inv);
                            uint32_t* dst_row0 = reinterpret_cast<uint32_t*>(codes_cs + (long long)row0 * p.M + j0);
                            if (p.Mpad - j0 >= 32)
                                stage_store_codes<4>(wd, stage_tile, lane, dst_row0, p.M / 2, j0 / 2, p.M / 2, rows_valid);
                            else
                                stage_store_codes<2>(wd, stage_tile, lane, dst_row0, p.M / 2, j0 / 2, p.M / 2, rows_valid);
                        }
                    }
                    if (tr) trace_ev(p, EV_E_DONE, n_items);
                    ++n_items;
                    if (++db == p.n_dbuf) {
                        db = 0;
                        dph ^= 1u;
                    }
                }
            }
        } else
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            const int rows_here = min(p.T_r, p.nby - w.t * p.T_r);
            const int blocks_here = rows_here * p.nbx;
            const int blk0 = w.t * p.T_r * p.nbx;
            for (int c = w.c0; c < w.c1; ++c) {
                ptx::mbar_wait(bar_d_full + 8 * db, dph);
                ptx::tc_fence_after();
                if (tr) trace_ev(p, EV_E_DFULL, n_items);
                const long long cs_global = (long long)w.s * p.cs_per_stream_sel +
                                            (long long)(w.g - p.gop_begin) * (p.G - 1) + c;
                const uint32_t d_tm = tmem_base + lane_bits + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                CS_CHECK((cs_global + 1) * p.nblk * (long long)p.M <= p.out_floats);
                CS_CHECK(qmode != Q_ROW || p.T_r <= kRowSlots);
                if (qmode == Q_ABSMAX || qmode == Q_ROW) {
                    const uint32_t slots = sbase + kRowSlotOff + (uint32_t)(n_items % 3) * (kRowSlots * 4);
                    if (qmode == Q_ROW && lane_idx < kRowSlots)   // next item's slots: last read 2 items ago
                        ptx::sts32(sbase + kRowSlotOff + (uint32_t)((n_items + 1) % 3) * (kRowSlots * 4) +
                                       (uint32_t)lane_idx * 4u, 0u);
                    uint32_t mx = 0;
                    for (int f = 0; f < p.F; ++f) {
                        const int b = f * p.L + ew * p.Lq + (int)lane;
                        const bool valid = (int)lane < p.Lq && ew * p.Lq + (int)lane < p.L && b < blocks_here;
                        float mff = 0.0f;
                        for (int j0 = 0; j0 < p.Mpad; j0 += 32) {
                            uint32_t v[32];
                            if (p.Mpad - j0 >= 32) {
                                ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)(f * p.Mpad + j0), v);
                            } else {
                                ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad + j0),
                                                        *reinterpret_cast<uint32_t(*)[16]>(v));
#pragma unroll
                                for (int q = 16; q < 32; ++q) v[q] = 0;
                            }
                            ptx::tc_wait_ld();
#pragma unroll
                            for (int q = 0; q < 32; ++q) mff = fmaxf(mff, fabsf(__uint_as_float(v[q])));
                        }
                        const uint32_t mf = valid ? __float_as_uint(mff) : 0u;
                        if (qmode == Q_ABSMAX) {
                            mx = max(mx, mf);
                        } else {
                            // segmented warp max over the (few) block rows this warp's 32 blocks touch
                            const int r = (int)((rowpack >> (6 * f)) & 63u);
                            const int rlo = (int)((lopack >> (6 * f)) & 63u);
                            const int rhi = (int)((hipack >> (6 * f)) & 63u);
                            CS_CHECK(rhi < kRowSlots);
                            for (int rr = rlo; rr <= rhi; ++rr) {
                                const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, r == rr ? mf : 0u);
                                if (lane == 0 && m != 0) ptx::atom_smem_max(slots + (uint32_t)rr * 4u, m);
                            }
                        }
                    }
                    if (qmode == Q_ABSMAX) {
                        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
                        if (lane == 0 && mx != 0) atomicMax(p.amax + cs_global, mx);
                    } else {
                        ptx::named_bar(1, 128);
                    }
                }
                if (qmode == Q_FRAME || qmode == Q_ROW) {
                    const uint32_t slots = sbase + kRowSlotOff + (uint32_t)(n_items % 3) * (kRowSlots * 4);
                    float inv = 1.0f;
                    int inv_row = -1;
                    if (qmode == Q_FRAME) {
                        inv = q16_inv(q16_scale(__ldcg(p.amax + cs_global)));
                    } else if (lane_idx < rows_here) {
                        p.scales[cs_global * p.nby + w.t * p.T_r + lane_idx] =
                            q16_scale(ptx::lds32(slots + (uint32_t)lane_idx * 4u));
                    }
                    int16_t* const codes_cs = p.codes + (cs_global * p.nblk + blk0) * (long long)p.M;
                    for (int f = 0; f < p.F; ++f) {
                        const int row0 = f * p.L + ew * p.Lq;
                        const int b = row0 + (int)lane;
                        const bool valid = (int)lane < p.Lq && ew * p.Lq + (int)lane < p.L && b < blocks_here;
                        const int rows_valid = min(p.Lq, min(p.L - ew * p.Lq, blocks_here - row0));
                        if (qmode == Q_ROW) {
                            const int r = (int)((rowpack >> (6 * f)) & 63u);
                            if (r != inv_row) {   // rows only grow with f: at most rows-per-tile updates
                                inv_row = r;
                                inv = q16_inv(q16_scale(valid ? ptx::lds32(slots + (uint32_t)r * 4u) : 0u));
                            }
                        }
                        if (smode == 0) {
                            uint32_t v[16];
                            ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad), v);
                            ptx::tc_wait_ld();
                            if (valid) ptx::stg64(codes_cs + (long long)b * 4, q16_pack(v[0], v[1], inv),
                                                  q16_pack(v[2], v[3], inv));
                            continue;
                        }
                        for (int j0 = 0; j0 < p.Mpad; j0 += 32) {
                            const int cw = min(32, p.Mpad - j0);
                            uint32_t v[32];
                            if (cw == 32) {
                                ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)(f * p.Mpad + j0), v);
                            } else {
                                ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad + j0),
                                                        *reinterpret_cast<uint32_t(*)[16]>(v));
                            }
                            ptx::tc_wait_ld();
                            if (smode == 2) {
                                if (valid) {
                                    int16_t* dst = codes_cs + (long long)b * p.M + j0;
#pragma unroll
                                    for (int q = 0; q < 32; ++q)
                                        if (q < cw && j0 + q < p.M) dst[q] = (int16_t)(q16_bits(v[q], inv) & 0xFFFFu);
                                }
                                continue;
                            }
                            uint32_t wd[16];
#pragma unroll
                            for (int q = 0; q < 16; ++q) wd[q] = q16_pack(v[2 * q], v[2 * q + 1], inv);
                            uint32_t* dst_row0 = reinterpret_cast<uint32_t*>(codes_cs + (long long)row0 * p.M + j0);
                            if (cw == 32)
                                stage_store_codes<4>(wd, stage_tile, lane, dst_row0, p.M / 2, j0 / 2, p.M / 2,
                                                     rows_valid);
                            else
                                stage_store_codes<2>(wd, stage_tile, lane, dst_row0, p.M / 2, j0 / 2, p.M / 2,
                                                     rows_valid);
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_d_empty + 8 * db);
                if (tr) trace_ev(p, EV_E_DONE, n_items);
                ++n_items;
                if (++db == p.n_dbuf) {
                    db = 0;
                    dph ^= 1u;
                }
            }
        }
    } else if ((EPI == EPI_F32 || EPI == EPI_F32A) && warp >= kEpiWarp0 && warp < kEpiWarp0 + 4 && !dbg_load_only) {
        // ================================================================ epilogue (a6)
        // Output rows (blocks) are M*4 bytes apart.  For M == 4 a thread's row is one 16-byte
        // vector and the warp's 32 rows are contiguous: store straight from registers.  For other
        // M % 4 == 0 each 32-row x (16|32)-column accumulator chunk goes through a 4 KB
        // XOR-swizzled SMEM tile so that every st.global.v4 instruction writes whole 64/128-byte
        // row segments (bank-conflict-free on both sides).  Other M: scalar stores.
        if (p.pdl_early) ptx::grid_dep_wait();
        const int ew = warp - kEpiWarp0;
        const uint32_t lane_bits = (uint32_t)(ew * 32) << 16;
        const uint32_t stage_tile = sbase + p.off_epi + (uint32_t)ew * 4096u;
        const int mode = (p.M == 4) ? 0 : ((p.M & 3) == 0 ? 1 : 2);
        const bool skip = (dbg_flags & 8) != 0;
        int db = 0;
        uint32_t dph = 0;
        int n_items = 0;
        const bool tr = (warp == kEpiWarp0 && lane == 0);
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            Unit w;
            if (!decode_unit(p, u, w)) continue;
            const int rows_here = min(p.T_r, p.nby - w.t * p.T_r);
            const int blocks_here = rows_here * p.nbx;
            const int blk0 = w.t * p.T_r * p.nbx;
            for (int c = w.c0; c < w.c1; ++c) {
                ptx::mbar_wait(bar_d_full + 8 * db, dph);
                ptx::tc_fence_after();
                if (tr) trace_ev(p, EV_E_DFULL, n_items);
                const long long cs_global = (long long)w.s * p.cs_per_stream_sel +
                                            (long long)(w.g - p.gop_begin) * (p.G - 1) + c;
                float* const out_cs = p.out + (cs_global * p.nblk + blk0) * (long long)p.M;
                const uint32_t d_tm = tmem_base + lane_bits + d_col0 + (uint32_t)db * (uint32_t)p.d_cols;
                CS_CHECK(d_col0 + (uint32_t)(db + 1) * (uint32_t)p.d_cols <= kTmemCols);
                CS_CHECK((cs_global + 1) * p.nblk * (long long)p.M <= p.out_floats);
                float amx = 0.0f;   // EPI_F32A: |y| maximum of this lane's blocks
                for (int f = 0; f < p.F; ++f) {
                    const int row0 = f * p.L + ew * p.Lq;            // tile block of this warp's lane 0
                    const int b = row0 + (int)lane;
                    const bool valid = (int)lane < p.Lq && ew * p.Lq + (int)lane < p.L && b < blocks_here;
                    const int rows_valid = min(p.Lq, min(p.L - ew * p.Lq, blocks_here - row0));
                    if (mode == 0) {
                        uint32_t v[16];
                        ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad), v);
                        ptx::tc_wait_ld();
                        if (valid && !skip) ptx::stg128(out_cs + (long long)b * 4, v[0], v[1], v[2], v[3]);
                        if constexpr (EPI == EPI_F32A)
                            if (valid)
#pragma unroll
                                for (int q = 0; q < 4; ++q) amx = fmaxf(amx, fabsf(__uint_as_float(v[q])));
                        continue;
                    }
                    for (int j0 = 0; j0 < p.Mpad; j0 += 32) {
                        const int cw = min(32, p.Mpad - j0);     // 16 or 32 columns
                        uint32_t v[32];
                        if (cw == 32) {
                            ptx::tmem_ld_32x32b_x32(d_tm + (uint32_t)(f * p.Mpad + j0), v);
                        } else {
                            ptx::tmem_ld_32x32b_x16(d_tm + (uint32_t)(f * p.Mpad + j0),
                                                    *reinterpret_cast<uint32_t(*)[16]>(v));
                        }
                        ptx::tc_wait_ld();
                        if constexpr (EPI == EPI_F32A)   // padded columns (j0 + q >= M) hold 0: Phi's pad rows are 0
                            if (valid)
#pragma unroll
                                for (int q = 0; q < 32; ++q)
                                    if (q < cw) amx = fmaxf(amx, fabsf(__uint_as_float(v[q])));
                        if (mode == 2) {
                            if (valid) {
                                float* dst = out_cs + (long long)b * p.M + j0;
#pragma unroll
                                for (int q = 0; q < 32; ++q)
                                    if (q < cw && j0 + q < p.M) dst[q] = __uint_as_float(v[q]);
                            }
                            continue;
                        }
                        float* dst_row0 = out_cs + (long long)row0 * p.M;
                        if (cw == 32)
                            stage_store<32>(v, stage_tile, lane, dst_row0, p.M, j0, rows_valid, skip);
                        else
                            stage_store<16>(v, stage_tile, lane, dst_row0, p.M, j0, rows_valid, skip);
                    }
                }
                if constexpr (EPI == EPI_F32A) {
                    const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(amx));
                    if (lane == 0 && mx != 0) atomicMax(p.amax + cs_global, mx);
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar_d_empty + 8 * db);
                if (tr) trace_ev(p, EV_E_DONE, n_items);
                ++n_items;
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
    if (threadIdx.x == 0) trace_ev(p, EV_K_END, 0);
    if (warp == kMmaWarp) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace csenc

#pragma nv_diagnostic pop
