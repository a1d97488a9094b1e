/*
 * cs_encoder.h -- C ABI of libcsenc.so, the B200 (sm_100a) encoder hot path of
 * "Increasing Compression Ratio of Low Complexity Compressive Sensing Video
 * Encoder with Application-Aware Configurable Mechanism" (arXiv 1311.1419).
 *
 * What one encode computes (PAPER.md line numbers, "P:n"):
 *   For every stream s and GOP g of G frames (sec.3.1 "we divide the source
 *   video into a key frame and several residual frames"; last GOP may be short),
 *   every CS frame F_t of the GOP minus the GOP's key frame F_key (sec.3.2
 *   "The CS frames all subtract the same key frame in a GOP"; Eq.(3) P:91 with
 *   the key passed through raw, i.e. Eq.(2) with e_coding = e_decoding = 0),
 *   cut into B x B blocks (block (by,bx) in raster order, pixel j = yy*B + xx
 *   inside the block; pixels outside the frame count as 0), each block measured
 *   with the same M x N matrix Phi, N = B*B (Eq.(1): y = A x):
 *
 *     y[s][g][c][by][bx][m] = sum_{j<N} Phi[m][j] * (F_{gG+1+c} - F_{gG})[by*B + j/B][bx*B + j%B]
 *
 *   Phi is IEEE fp16 (the caller's rounding of N(0,1/M) samples, "A
 *   Gaussian random matrix is used to make the measurements"); residuals are
 *   exact integers in [-255,255]; products are exact; accumulation is fp32 on
 *   the tensor cores.  Output is fp32, block-major, concatenated per stream,
 *   per GOP, per CS frame:
 *     meas[((s*CS_s + g*(G-1) + c) * nblk + by*nbx + bx) * M + m],
 *     CS_s = number of CS frames per stream, nbx = ceil(W/B), nby = ceil(H/B),
 *     nblk = nby*nbx.
 *   Accuracy contract: |y_gpu - y_exact| <= 1e-5 * sum_j |Phi[m][j] * r_j| per
 *   entry (entries whose scale is 0 are exactly 0).
 *
 * Conventions: every function returns a status (CS_OK = 0) unless noted; on
 * failure cs_last_error() returns a thread-local message.  No C++ exception
 * crosses the ABI.  Device pointers are caller-owned CUDA device memory; host
 * pointers are caller-owned host memory.  Encodes are asynchronous on the given
 * stream (cudaStream_t; NULL = legacy default stream); kernel faults surface at
 * the caller's next synchronisation.  The encoder is immutable after create
 * (except its internal caches, guarded by a mutex), so concurrent encodes on
 * different streams are safe.
 * Devices: an encoder lives on the device that was current at create.  Every
 * device-buffer call (encode, q16, adjoint, key codec, set_gop_phis, autotune)
 * must be made with that device current, else it returns CS_ERR_ARG without
 * launching; the host-buffer calls switch to it for their duration and restore
 * the caller's current device.
 */
#ifndef CS_ENCODER_H
#define CS_ENCODER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cs_encoder cs_encoder;      /* opaque */
typedef struct CUstream_st* cs_stream_t;   /* == cudaStream_t */

enum {
    CS_OK = 0,
    CS_ERR_ARG = 1,          /* bad argument (NULL, out of range, misaligned) */
    CS_ERR_UNSUPPORTED = 2,  /* valid but unsupported shape (B not in {8,16,32}, W % 16 != 0, M > 256 ...) */
    CS_ERR_PHI = 3,          /* Phi has a non-finite entry or |entry| > 2048 */
    CS_ERR_CUDA = 4,         /* CUDA runtime/driver error (message has the CUDA error string) */
    CS_ERR_OOM = 5           /* device allocation failed */
};

/* Planner output (read-only diagnostics of how the kernel tiles the work). */
typedef struct cs_plan_info {
    int tile_block_rows;   /* block rows per tile (tiles are full-width) */
    int folds;             /* tile blocks folded onto the 128 TMEM lanes */
    int lanes;             /* lanes used per fold */
    int chunk_rows;        /* pixel rows of a block per K-chunk (K-chunk = chunk_rows*B) */
    int stages;            /* shared-memory ring depth */
    int key_resident;      /* key strip: 2 = converter registers, 1 = resident in SMEM, 0 = streamed per chunk */
    int box_w;             /* bytes per strip row (= W: strips are full-width frame rows) */
    int smem_bytes;        /* dynamic shared memory per CTA */
    int tmem_cols;         /* TMEM columns used */
    int m_pad;             /* MMA N dimension (M rounded up to 16) */
    int chains;            /* independent TMEM accumulation chains per block (summed in the epilogue) */
    int prefetch_items;    /* items the producer prefetches into L2 ahead of the SMEM loads */
    int a_bufs;            /* TMEM A-operand ring depth (converters -> MMA) */
    int d_bufs;            /* TMEM accumulator ring depth (MMA -> epilogue) */
    int sms;               /* SMs of the device at create time */
    int phi_stream;        /* 1: Phi's K-slices ride in the stages (multi-chunk plans), 0: Phi resident in SMEM */
} cs_plan_info;

/* ---- lifecycle ------------------------------------------------------------------------- */

/* Create an encoder for W x H uint8 frames, GOP size gop (>= 1), B x B blocks and M
 * measurements per block ("the GOP size and the measurement matrix size can be
 * configured").
 *   phi_fp16: HOST pointer, M*B*B IEEE fp16 bit patterns, row-major [M][B*B]; copied.
 *   *out    : receives the encoder; left NULL on failure.
 * Validation: W,H >= 1; gop >= 1; B in {8,16,32} (else CS_ERR_UNSUPPORTED);
 * 1 <= M <= min(B*B, 256); W % 16 == 0 (TMA row pitch) else CS_ERR_UNSUPPORTED; Phi entries finite with |Phi| <= 2048 else CS_ERR_PHI.  Argument validation
 * happens before any CUDA call.  Allocates the device copy of Phi on the current
 * device.  Phi stays resident in shared memory when it fits beside the ring (Mpad*B*B*2 bytes,
 * Mpad = M rounded up to 16); otherwise (B = 32 with large M) the planner streams its K-slices with
 * the frame strips; CS_ERR_UNSUPPORTED only if no tiling fits at all. */
int cs_encoder_create(int W, int H, int gop, int B, int M, const uint16_t* phi_fp16, cs_encoder** out);

/* Free the encoder and its device memory.  NULL-safe.  The caller must have
 * synchronised every stream that used it. */
int cs_encoder_destroy(cs_encoder* enc);

/* Autotune: time the planner's best `max_candidates` plans (ranked by its cost model) on the
 * caller's buffers -- `reps` timed cs_encode_batch calls each on `stream`, after one warm-up --
 * and keep the fastest for all later encodes.  Every plan produces bit-identical measurements
 * (the per-block K order of the MMA chain does not depend on the plan), so tuning is invisible
 * in the output.  Synchronises `stream`.  Not safe concurrently with other encodes of `enc`. */
int cs_encoder_autotune(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, float* meas_dev,
                        int max_candidates, int reps, cs_stream_t stream);

/* Number of feasible plans the planner ranked (-1 for NULL), and explicit selection of one
 * (tests / tools).  Host only; not safe concurrently with encodes of `enc`. */
int cs_encoder_num_candidates(const cs_encoder* enc);
int cs_encoder_set_candidate(cs_encoder* enc, int index);
int cs_encoder_candidate_index(const cs_encoder* enc);  /* plan in use (0 = model's best) */

/* Fill *info with the tiling plan.  Host only. */
int cs_encoder_plan(const cs_encoder* enc, cs_plan_info* info);

/* Debug timeline (tracing subsystem): when cap > 0, every subsequent encode launch records, for
 * CTA 0 only, the SM clock (clock64) of each pipeline event into trace_dev (DEVICE, caller-owned,
 * CS_TRACE_EVENTS * cap uint64): trace_dev[event * cap + i] = i-th occurrence of the event.
 * Events: 0 producer slot free, 1 producer TMA issued, 2 converter data landed, 3 converter A
 * buffer free, 4 converter A written, 5 MMA A ready, 6 MMA issued+committed, 7 epilogue
 * accumulator ready, 8 epilogue done, 9 converter tcgen05.st issued, 10 / 11 (q16 row-scale register
 * path) epilogue row maxima published / all four warps' maxima present, 12 kernel entry and 13 CTA
 * exit (one occurrence each; occurrences 1..7 of event 12 are start-up marks: barriers initialised,
 * TMEM allocated, prologue barrier passed, offset table written, producer started, producer's first
 * unit decoded, first Phi slice issued).  cap = 0 disables (default).  While a trace buffer is set the
 * kernels do not overlap their predecessors (cs_encoder_set_stable_inputs is ignored).
 * Not thread-safe with concurrent encodes of the same encoder. */
#define CS_TRACE_EVENTS 14
/* Profiling ranges: with CSENC_NVTX=1 in the environment (read once per process), every encode /
 * adjoint / key-codec / frame-encode entry point opens an NVTX range named after itself (ncu --nvtx,
 * nsys); header-only nvtx3, a no-op when no tool is attached. */
int cs_encoder_set_trace(cs_encoder* enc, unsigned long long* trace_dev, int cap);

/* Launch overlap (programmatic dependent launch).  Every encode / adjoint kernel is launched so that its
 * CTAs may start while the stream's previous KERNEL is still draining (they take an SM as soon as that
 * kernel's CTA there has exited).  By default the kernel then waits for the previous kernel to complete
 * before it touches global memory at all, so only its prologue overlaps.  `flags` is the caller's promise
 * about INPUTS (bit mask, default 0):
 *   CS_STABLE_FRAMES (1): the frames (and Phi) of this encoder's ENCODE calls are never written by the
 *     kernel that precedes the call in the stream -- e.g. they arrive by cudaMemcpyAsync, which is ordered
 *     as usual, or were finished earlier;
 *   CS_STABLE_MEASUREMENTS (2): the same for the measurements given to cs_adjoint (NOT true for
 *     cs_adjoint right after the encode that produced them).
 * With the promise, loads, conversion and MMAs start at once and only the output stores (and the reads of
 * the per-frame maxima of a two-pass quantisation) wait for the previous kernel, which keeps
 * write-after-write order on a reused output buffer.  Calls whose inputs come from the preceding kernel by
 * construction (cs_encode_batch_keys: the decoded keys) ignore the setting.  Worth ~3 us per launch back
 * to back (C4 step -4%; short launches, C2 / C3, more). */
#define CS_STABLE_FRAMES 1
#define CS_STABLE_MEASUREMENTS 2
int cs_encoder_set_stable_inputs(cs_encoder* enc, int flags);

/* ---- encode (device buffers; asynchronous) ---------------------------------------------- */

/* Encode one GOP (SPEC.md:355-358 encode_gop): frames_dev = DEVICE [n_frames][H][W] uint8,
 * 16-byte aligned, frame 0 is the key; 1 <= n_frames <= gop (a short final GOP is allowed).
 * meas_dev = DEVICE fp32 [n_frames-1][nby][nbx][M], 16-byte aligned.  n_frames == 1 writes
 * nothing.  One kernel launch on `stream`; no allocation. */
int cs_encode_gop(cs_encoder* enc, const uint8_t* frames_dev, int n_frames, float* meas_dev, cs_stream_t stream);

/* Encode n_seq independent streams of T frames each: frames_dev = DEVICE [n_seq][T][H][W]
 * uint8; meas_dev = DEVICE fp32, cs_measurement_count(enc, n_seq, T) floats, layout above.
 * ONE kernel launch covers every GOP of every stream (persistent grid of one CTA per SM).
 * No allocation and no host synchronisation: capturable in a CUDA graph (tests/test_gpu_graph.py). */
int cs_encode_batch(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, float* meas_dev,
                    cs_stream_t stream);

/* Same, restricted to GOPs [gop_begin, gop_end) of every stream (GOP index within a stream);
 * meas_dev receives only those GOPs' measurements, in the same order.  Used to shard a batch
 * across devices or to pipeline host copies. */
int cs_encode_batch_gops(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, int gop_begin,
                         int gop_end, float* meas_dev, cs_stream_t stream);

/* ---- 16-bit measurement quantisation ---------------------------- */

/* SPEC.md:154-162 quantize: scale = max|y_i| / 32767 (1 if all y_i == 0), codes = round(y_i /
 * scale), round half to even, clamped to +-32767; dequantize = codes * scale.  The kernel takes
 * the decision in fp32 on its own fp32 y: scale = fl32(amax / 32767), inv = fl32(1 / scale), code =
 * round-half-even of the fp32 FFMA y * inv (R18), so a code can differ by one from the
 * exact round(y / scale) only where y / scale lies within ~32767 * 2^-23 of a half-integer.  Container payload per CS frame: f32 scale + M*nblk int16 codes.
 *   CS_Q16_FRAME: one scale per CS frame, exactly as SPEC states.  The frame maximum is a
 *     grid-wide dependency.  When 8*M <= B*B (storing fp32 y and reading it back moves no more
 *     bytes than reading the frames again) one measurement pass writes y to a stream-ordered workspace
 *     (stream-ordered, from the encoder's own memory pool, n_cs*nblk*M floats;
 *     the pool keeps its memory for later calls until cs_encoder_destroy) together with the frame
 *     maxima and a re-quantisation kernel makes the codes; otherwise the measurement runs twice: an
 *     absmax pass (no stores, one atomicMax per warp and frame) and a codes pass.  Then a tiny
 *     finalize kernel (memset + 3 launches either way).  Both give the same codes, bit for bit.
 *   CS_Q16_ROW: one scale per (CS frame, block row of B pixel rows): a single fused pass (the
 *     maximum is reduced on chip).  A documented deviation (R19).  Needs tiles of
 *     <= 40 block rows: when the encoder's current plan has taller tiles the call runs the best
 *     candidate plan that qualifies (CS_ERR_UNSUPPORTED only if none does). */
#define CS_Q16_FRAME 0
#define CS_Q16_ROW 1

/* Number of fp32 scales cs_encode_batch_q16 writes: n_cs (FRAME) or n_cs * nby (ROW), where
 * n_cs = n_seq * CS frames per stream; -1 on bad arguments. */
int64_t cs_q16_scale_count(const cs_encoder* enc, int n_seq, int T, int granularity);

/* frames_dev as cs_encode_batch; codes_dev = DEVICE int16 [n_cs][nby][nbx][M] (the measurement
 * layout), 16-byte aligned; scales_dev = DEVICE fp32, cs_q16_scale_count entries, 4-byte
 * aligned, [n_cs] or [n_cs][nby].  Asynchronous on `stream`; no allocation.  Errors: CS_ERR_ARG
 * (NULL / misaligned / bad granularity), CS_ERR_UNSUPPORTED (see CS_Q16_ROW), CS_ERR_CUDA. */
int cs_encode_batch_q16(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, int granularity,
                        int16_t* codes_dev, float* scales_dev, cs_stream_t stream);

/* ---- paper-faithful frame-level measurement ---------------------- */

/* Eq. (1), as the paper states it: ONE dense measurement matrix A in R^{m x n}, n = W*H
 * (SPEC.md:133-134), applied to the whole vectorised residual of every CS frame:
 *     y[cs][i] = sum_{j < n} A[i][j] * (F_cs - F_key)[j / W][j % W]     (row-major vec)
 * with the GOP structure and key reference of the block path (a1, a3).  A is fp16 (e.g. seeded
 * N(0, 1/m), m = round(n / CR); QCIF at CR 50: m = 507); products are exact, accumulation is
 * fp32 on the tensor cores (kind::f16 GEMM, 2 x 128 measurements x up to 256 CS frames per tile; the
 * (tile, K chunk) sequence is split into equal per-SM ranges (stream-K), and tiles cut by a range
 * boundary are summed from their pieces' partial tiles in a fixed order by a second kernel).
 * Accuracy contract: |y_gpu - y| <= (n/16 + 16) * 2^-23 * sum_j |A[i][j] r_j| (fp32 accumulation
 * of n/16 tensor-core partial sums; R24). */
typedef struct cs_frame_encoder cs_frame_encoder;

/* A_fp16: HOST [m][W*H] fp16 bits, copied to the device (m*n*2 bytes).  W % 16 == 0; |A| <= 2048
 * and finite (CS_ERR_PHI).  gop >= 1. */
int cs_frame_encoder_create(int W, int H, int gop, int m, const uint16_t* A_fp16, cs_frame_encoder** out);
int cs_frame_encoder_destroy(cs_frame_encoder* enc);

/* Debug timeline of CTA 0 (as cs_encoder_set_trace): trace_dev[event * cap + i] = clock64 of the i-th
 * K chunk's event: 0 producer issued the TMA loads, 1 converters saw the data, 2 residual operand
 * written, 3 MMAs issued.  cap = 0 disables. */
int cs_frame_encoder_set_trace(cs_frame_encoder* enc, unsigned long long* trace_dev, int cap);

/* n_seq * (CS frames per stream) * m; -1 on bad arguments. */
int64_t cs_frame_measurement_count(const cs_frame_encoder* enc, int n_seq, int T);

/* frames_dev = DEVICE uint8 [n_seq][T][H][W]; y_dev = DEVICE fp32 [n_seq * CS_s][m] (CS frames in
 * the block path's order), both 16-byte aligned.  Asynchronous on `stream` (1 launch, or 2 when a
 * tile is cut by a stream-K range boundary; the partial tiles are stream-ordered allocations from the
 * encoder's own pool, freed on the stream). */
int cs_frame_encode_batch(cs_frame_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, float* y_dev,
                          cs_stream_t stream);

/* ---- adjoint / back-projection ---------------------------------- */

/* SPEC.md:145-153 adjoint(A, v) = A^T v, the decoder's start point x = A^T y, for the
 * block-based Phi: every block b of every frame gets x_b = Phi^T y_b (B*B values from M), laid back
 * into the frame (block (by, bx), in-block index j = yy*B + xx -> pixel (by*B + yy, bx*B + xx);
 * pixels of padded blocks outside the frame are dropped).
 *   meas_dev = DEVICE fp32 [n_frames][nby][nbx][M] (the layout cs_encode_batch writes; any fp32
 *              values), 16-byte aligned;  x_dev = DEVICE fp32 [n_frames][H][W], 16-byte aligned.
 * Tensor cores (kind::tf32) with y split into two tf32 terms: |error| <~ 1e-6 * sum_m |Phi_mj y_m|.
 * One asynchronous launch on `stream`; no allocation.  Errors: CS_ERR_ARG (NULL / misaligned /
 * n_frames < 0), CS_ERR_UNSUPPORTED (M % 4 != 0: measurement rows must be 16-byte multiples;
 * more than 2^31 blocks in one call; per-GOP matrices set by cs_encoder_set_gop_phis -- the
 * adjoint uses the Phi given at create, restore it with cs_encoder_set_gop_phis(enc, 0, NULL)),
 * CS_ERR_CUDA. */
int cs_adjoint(cs_encoder* enc, const float* meas_dev, int64_t n_frames, float* x_dev, cs_stream_t stream);

/* ---- closed-loop key frame --------------------------------------- */

/* Eq. (2)-(3): the CS frames subtract the reconstructed key F-hat = decode(encode(F_key)),
 * which cancels the key codec's error at the decoder (Eq. 4).  The key codec is SPEC's stand-in for
 * H.264 intra: per 8x8 block (frame padded to multiples of 8 by edge
 * replication) s = pixel - 128; fixed-point DCT with Ci = rint(4096 * C) (C the orthonormal DCT-II):
 *   forward  t1 = floor((s Ci^T + 2^4) / 2^5), t2 = Ci t1,
 *            q = sign(t2) * floor((|t2| + qstep * 2^18) / (qstep * 2^19))
 *   inverse  t1 = floor((q*qstep Ci + 2^11) / 2^12), t2 = Ci^T t1,
 *            pixel = clamp(floor((t2 + 2^11) / 2^12) + 128, 0, 255)
 * (R21).  Entropy coding and the CR-23 rate search are not part of this library. */

/* Quantiser steps [v][u] = clamp(round_half_even(quant_scale * T.81 Table K.1), 1, 4096).  Host. */
int cs_key_qsteps(double quant_scale, int32_t qsteps_out[64]);

/* The fixed-point DCT basis Ci[u][x] the kernels use (diagnostics / tests).  Host. */
void cs_key_dct_basis(int32_t basis_out[64]);

/* Number of int16 coefficients cs_key_codec writes: n_seq * ceil(T/gop) * ceil(H/8) * ceil(W/8) * 64. */
int64_t cs_key_coef_count(const cs_encoder* enc, int n_seq, int T);

/* Code and decode every GOP key frame (frame g*gop of every stream) of frames_dev [n_seq][T][H][W]:
 *   qsteps_host : HOST int32 [64], each in [1, 4096] (else CS_ERR_ARG);
 *   coef_dev    : DEVICE int16 [n_seq][ceil(T/gop)][ceil(H/8)][ceil(W/8)][8 v][8 u] or NULL;
 *   keys_dev    : DEVICE uint8 [n_seq][ceil(T/gop)][H][W], the decoded key frames F-hat.
 * 16-byte aligned device buffers.  One asynchronous launch on `stream`. */
int cs_key_codec(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, const int32_t* qsteps_host,
                 int16_t* coef_dev, uint8_t* keys_dev, cs_stream_t stream);

/* cs_encode_batch with every CS frame's residual taken against keys_dev[s][g] (e.g. the decoded keys
 * from cs_key_codec) instead of the raw key frame; same output layout and accuracy contract. */
int cs_encode_batch_keys(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, const uint8_t* keys_dev,
                         float* meas_dev, cs_stream_t stream);

/* Variant (Eq. (3) P:91 read literally): every CS frame's residual is taken
 * against the PREVIOUS raw frame, D_t = F_t - F_{t-1} (open loop; the GOP structure still decides
 * which frames are keys and are not measured).  Same output layout and accuracy contract as
 * cs_encode_batch; runs the planner's best streamed-key plan (CS_ERR_UNSUPPORTED if none fits). */
int cs_encode_batch_chained(cs_encoder* enc, const uint8_t* frames_dev, int n_seq, int T, float* meas_dev,
                            cs_stream_t stream);

/* Variant ("per-GOP seeds are derivable (seed xor GOP index)"):
 * after this call every encode of `enc` measures GOP g of each stream (g = GOP index within the
 * stream) with phis[g % n_phi] instead of the create-time Phi.  phis: HOST, n_phi matrices of
 * [M][B*B] fp16 bits (each validated like cs_encoder_create's Phi; copied).  n_phi = 0 restores the
 * single Phi.  The resident Phi is reloaded into shared memory whenever a CTA's next unit belongs
 * to a GOP with a different matrix.  Host; not safe concurrently with encodes of `enc`. */
int cs_encoder_set_gop_phis(cs_encoder* enc, int n_phi, const uint16_t* phis);

/* ---- encode (HOST buffers; synchronous) ------------------------------------------------- */

/* End-to-end call: frames_host = HOST [n_seq][T][H][W] uint8, meas_host = HOST fp32 output
 * (cs_measurement_count floats).  Copies in, encodes, copies out, and returns after the
 * result is in meas_host.  Pinned host memory gives full PCIe bandwidth; pageable works.
 * Work is split into GOP groups and the host<->device copies of one group overlap the
 * encode of another (internal streams and device workspace, allocated on first use and
 * kept until destroy). */
int cs_encode_batch_host(cs_encoder* enc, const uint8_t* frames_host, int n_seq, int T, float* meas_host);

/* The same for several encoders over the SAME frames (e.g. several measurement matrices / rates,
 * the M sweep): encs[0..n_enc-1] must share W, H, gop and device (B and M may differ; no encoder
 * twice); meas_host[k] receives encoder k's output.  Each frame group crosses PCIe once, all
 * encoders run on it, and every output is copied back as soon as its encode finishes.  Uses the
 * first encoder's frame workspace and streams; locks every encoder's workspace. */
int cs_encode_batch_host_multi(cs_encoder* const* encs, int n_enc, const uint8_t* frames_host, int n_seq, int T,
                               float* const* meas_host);

/* 16-bit form of the host calls (f1; SPEC.md:154-162 and the container's "f32 scale + m x i16 codes",
 * SPEC.md:410): the same pipeline with cs_encode_batch_q16 per group, codes_host = HOST int16 (the
 * measurement layout, cs_measurement_count entries) and scales_host = HOST fp32 (cs_q16_scale_count
 * entries), so the device->host copy moves 2 bytes per measurement instead of 4.  Groups are whole
 * streams (n_seq > 1) or whole GOPs, and every scale (per CS frame or per CS-frame block row) lies
 * inside one group, so the result equals cs_encode_batch_q16 on the whole batch, bit for bit.
 * Errors as cs_encode_batch_q16 and cs_encode_batch_host_multi. */
int cs_encode_batch_host_q16(cs_encoder* enc, const uint8_t* frames_host, int n_seq, int T, int granularity,
                             int16_t* codes_host, float* scales_host);
int cs_encode_batch_host_multi_q16(cs_encoder* const* encs, int n_enc, const uint8_t* frames_host, int n_seq, int T,
                                   int granularity, int16_t* const* codes_host, float* const* scales_host);

/* ---- accounting (host only) ------------------------------------------------------------- */

/* Number of fp32 measurements cs_encode_batch writes for n_seq streams of T frames
 * (-1 on bad arguments). */
int64_t cs_measurement_count(const cs_encoder* enc, int n_seq, int T);

/* CR = original bits / (key-frame bits + measurement bits) (BASELINE.json north_star;
 * Table I).  T = 0 means one full GOP; key_cr = 1.0 means raw key frames;
 * bits_per_measurement = 8 is the paper's sample-count convention (CR_cs = n/m),
 * 32 gives the realised fp32 payload ratio.  Uses the real GOP composition and counts
 * padded blocks.  Returns a negative value on bad arguments. */
double cs_compression_ratio(const cs_encoder* enc, int T, double key_cr, int bits_per_measurement);

/* Same accounting without an encoder (pure host arithmetic). */
double cs_compression_ratio_cfg(int W, int H, int gop, int B, int M, int T, double key_cr,
                                int bits_per_measurement);
int64_t cs_measurement_count_cfg(int W, int H, int gop, int B, int M, int n_seq, int T);

/* Table I closed form: G / (1/key_cr + (G-1)/cs_cr). Negative on bad arguments. */
double cs_total_cr(int G, double key_cr, double cs_cr);

/* Validate a configuration exactly as cs_encoder_create does, without touching CUDA.
 * phi_fp16 may be NULL (then Phi is not checked). */
int cs_validate_config(int W, int H, int gop, int B, int M, const uint16_t* phi_fp16);

/* Planner without an encoder (pure host): the plan cs_encoder_create would pick on a device
 * with `smem_limit` bytes of opt-in shared memory per block and `sms` SMs (B200: 232448, 148). */
int cs_plan_cfg(int W, int H, int gop, int B, int M, int smem_limit, int sms, cs_plan_info* info);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* cs_last_error(void);

/* Library version string. */
const char* cs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CS_ENCODER_H */
