"""oracle -- plain, slow, obviously-correct CPU reference of the encoder hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1311_1419_b200``) never imports it, and
this package never imports the product path; the two share no code.  The
only shared module is ``synth`` (seeded input generators, no method
arithmetic).

Everything is fp64 numpy.  Why fp64 is EXACT here (SURVEY.md sec.8(c),
DESIGN.md "Exactness"): every fp16 value of Phi is an integer multiple of
2^-24 and every residual r_j is an integer with |r_j| <= 255, so every product
Phi_mj * r_j and every partial sum is a multiple of 2^-24; with |Phi| <= 2048
and N <= 1024 every partial sum is below 2^29 in magnitude, so 29 + 24 = 53
bits hold it exactly.  The fp64 result is therefore the exact real value in
any summation order, and a library matmul (BLAS dgemm) may serve as the
summation step without any rounding caveat.

Paper passages followed (PAPER.md line numbers, section):
  a1 GOP partition   -- P:25, sec.3.1 ("divided into key frame and several
                        residual frames"), sec.3.2; short final GOP SPEC.md:385-390
  a2 block vector    -- P:85 sec.3.2 (x is the vectorised signal); row-major
                        vectorisation SPEC.md:89; B x B blocks with a shared Phi
                        is BASELINE.json:5's adaptation (reading R1)
  a3 residual        -- P:87 ("The CS frames all subtract the same key frame in
                        a GOP"), Eq.(2)-(3) P:89-91 with the raw key pass-through
                        (e_coding = e_decoding = 0, BASELINE.json:5)
  a4 measurement     -- Eq.(1): y = A x, A in R^{m x n}
  a5 Phi             -- fp16 bit patterns supplied by the caller (synth.phi_from_seed)
  a6 output layout   -- y[s][g][c][by][bx][m], block-major (BASELINE.json:5 item 4)
  a7 CR accounting   -- "original bits / (key bits + measurement bits)"
                        (BASELINE.json:5); Table I closed form P:113-126
  f1 quantisation    -- SPEC.md:154-162 (scale = max|y|/32767, codes = round(y/scale)) on the
                        exact y, f32 scale SPEC.md:410, ties to even (R17-R18)
  f2 frame-level A   -- Eq.(1) P:83-85 with one dense A in R^{m x n}, n = W*H
  f3 adjoint         -- SPEC.md:145-153 (A^T v), TVAL3 start point x = A^T y SPEC.md:235;
                        per block x_b = Phi^T y_b reassembled into the frame (inverse of a2)
  f4 closed-loop key -- Eq.(2)-(3) P:87-91 with SPEC's 8x8 DCT intra codec as the
                        stand-in for H.264 intra; fixed-point transform DESIGN.md R21
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "measure_frame", "block_matrix_as_frame", "quantize", "dequantize", "quantize_frames", "frame_unblocks", "adjoint_blocks", "adjoint",
    "adjoint_tolerance_scale", "JPEG_LUMA", "dct_basis", "dct_basis_int", "key_qsteps", "pad8",
    "intra_forward", "intra_inverse", "decode_key", "encode_stream_closed_loop", "encode_stream_chained", "encode_stream_gop_phis", "measure_entries", "gop_partition", "cs_frame_count", "block_grid", "frame_blocks", "residual", "measure",
    "tolerance_scale", "encode", "encode_stream", "phi_values", "compression_ratio", "total_cr",
    "check_tolerance",
]


# -- a1 ------------------------------------------------------------------------------------------
def gop_partition(T: int, G: int):
    """GOPs of a T-frame sequence: list of (key frame index, [CS frame indices]).

    P:71 sec.3.1 "we divide the source video into a key frame and several
    residual frames"; sec.3.2 one key per GOP.  The final GOP may be short
    (10 frames, G=4 -> lengths 4,4,2)."""
    if T < 0 or G < 1:
        raise ValueError("T >= 0 and G >= 1 required")
    gops = []
    for t0 in range(0, T, G):
        gops.append((t0, list(range(t0 + 1, min(t0 + G, T)))))
    return gops


def cs_frame_count(T: int, G: int) -> int:
    return sum(len(cs) for _, cs in gop_partition(T, G))


# -- a2 ------------------------------------------------------------------------------------------
def block_grid(W: int, H: int, B: int):
    """(nby, nbx): B x B blocks covering the frame, partial blocks zero padded (reading R10)."""
    return (H + B - 1) // B, (W + B - 1) // B


def frame_blocks(frame: np.ndarray, B: int) -> np.ndarray:
    """int64 [nby*nbx][B*B]: block (by,bx) in raster order, pixel j = yy*B + xx
    (row-major inside the block).  Pixels outside the frame are 0."""
    H, W = frame.shape
    nby, nbx = block_grid(W, H, B)
    pad = np.zeros((nby * B, nbx * B), dtype=np.int64)
    pad[:H, :W] = frame
    return pad.reshape(nby, B, nbx, B).transpose(0, 2, 1, 3).reshape(nby * nbx, B * B)


# -- a3 ------------------------------------------------------------------------------------------
def residual(cs_frame: np.ndarray, key_frame: np.ndarray) -> np.ndarray:
    """D = F_cs - F_key as signed integers, no clamping (Eq.(3)).
    With the raw key pass-through F_hat_key = F_key (Eq.(2) with zero codec error)."""
    if cs_frame.shape != key_frame.shape:
        raise ValueError("frame shapes differ")
    return cs_frame.astype(np.int64) - key_frame.astype(np.int64)


# -- a4 / a5 -------------------------------------------------------------------------------------
def phi_values(phi_bits: np.ndarray) -> np.ndarray:
    """fp64 values of the fp16 bit patterns (exact widening)."""
    return np.asarray(phi_bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def measure(R: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """y_b = Phi r_b for every block row r_b of R (Eq.(1) constraint Ax = y).
    R: integer [nblk][N]; phi: fp64 [M][N]; returns fp64 [nblk][M] (exact, see module doc)."""
    return np.asarray(R, dtype=np.float64) @ np.asarray(phi, dtype=np.float64).T


def tolerance_scale(R: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """S[b][m] = sum_j |Phi_mj * r_bj| -- the per-entry scale of BASELINE.json:5's
    acceptance bound |dy| <= 1e-5 * S (exact in fp64 for the same reason)."""
    return np.abs(np.asarray(R, dtype=np.float64)) @ np.abs(np.asarray(phi, dtype=np.float64)).T


# -- a1..a6 --------------------------------------------------------------------------------------
def encode_stream(frames: np.ndarray, phi_bits: np.ndarray, G: int, B: int, with_scale: bool = True):
    """One stream, frames uint8 [T][H][W] -> (y, S) fp64 [n_cs][nblk][M].

    For every GOP (a1), every CS frame minus the GOP's key frame (a3), cut into
    blocks (a2), measured with the shared Phi (a4); output concatenated per GOP,
    per CS frame, block-major (a6)."""
    T, H, W = frames.shape
    phi = phi_values(phi_bits)
    M, N = phi.shape
    if N != B * B:
        raise ValueError("Phi must have B*B columns")
    nby, nbx = block_grid(W, H, B)
    n_cs = cs_frame_count(T, G)
    y = np.empty((n_cs, nby * nbx, M), dtype=np.float64)
    S = np.empty_like(y) if with_scale else None
    i = 0
    for key_t, cs_ts in gop_partition(T, G):
        for t in cs_ts:
            R = frame_blocks(residual(frames[t], frames[key_t]), B)
            y[i] = measure(R, phi)
            if with_scale:
                S[i] = tolerance_scale(R, phi)
            i += 1
    return y, S


def encode(frames: np.ndarray, phi_bits: np.ndarray, G: int, B: int, with_scale: bool = True):
    """frames uint8 [S][T][H][W] -> (y, S) fp64 [S * n_cs][nblk][M] (streams concatenated)."""
    ys, Ss = [], []
    for s in range(frames.shape[0]):
        y, S = encode_stream(frames[s], phi_bits, G, B, with_scale)
        ys.append(y)
        Ss.append(S)
    y = np.concatenate(ys, axis=0)
    return y, (np.concatenate(Ss, axis=0) if with_scale else None)


def measure_entries(frames: np.ndarray, phi_bits: np.ndarray, G: int, B: int, cs_index: np.ndarray,
                    blocks: np.ndarray):
    """y and S for selected (CS frame, block) pairs of one stream, one by one from the
    definition (for full-size parity where encoding everything on the CPU is too slow).
    cs_index: indices into the stream's CS-frame order (a1); blocks: raster block indices.
    Returns fp64 arrays [len][M]."""
    T, H, W = frames.shape
    phi = phi_values(phi_bits)
    nby, nbx = block_grid(W, H, B)
    order = [(k, t) for k, cs in gop_partition(T, G) for t in cs]
    ys, Ss = [], []
    for i, b in zip(np.asarray(cs_index).ravel(), np.asarray(blocks).ravel()):
        key_t, t = order[int(i)]
        by, bx = divmod(int(b), nbx)
        blk = np.zeros((B, B), dtype=np.int64)
        y0, x0 = by * B, bx * B
        h, w = min(B, H - y0), min(B, W - x0)
        blk[:h, :w] = residual(frames[t, y0:y0 + h, x0:x0 + w], frames[key_t, y0:y0 + h, x0:x0 + w])
        r = blk.reshape(1, B * B)
        ys.append(measure(r, phi)[0])
        Ss.append(tolerance_scale(r, phi)[0])
    return np.asarray(ys), np.asarray(Ss)


# -- f1: 16-bit measurement quantisation ---------------------------------------------------------
def quantize(y, bits: int = 16):
    """SPEC.md:154-162 quantize: scale = max|y_i| / 32767 (scale = 1 if y is all zero),
    codes = round(y_i / scale), dequantize = codes * scale.  The container stores the scale as f32
    (SPEC.md:410), so scale is rounded to fp32 (R17); round = round half to even (SPEC
    leaves the tie rule open, R17).  y is the exact measurement (fp64, as encode() returns it) and
    the rounding of y / scale is decided EXACTLY (R18): q0 = rint of the fp64 quotient, then the
    exact remainder d = y - q0 * scale (q0 * scale has <= 16 + 24 significant bits and d is a
    multiple of min(ulp(y), ulp(scale)) below scale in magnitude, so both are exact in fp64) moves q0
    by one where the quotient's rounding crossed a half-integer, and an exact tie (|d| = scale/2)
    goes to the even neighbour.  Returns (int16 codes, float32 scale)."""
    if bits != 16:
        raise ValueError("16-bit quantisation only")
    y = np.asarray(y, dtype=np.float64)
    if not np.all(np.isfinite(y)):
        raise ValueError("non-finite measurement")
    qmax = (1 << (bits - 1)) - 1
    amax = float(np.max(np.abs(y))) if y.size else 0.0
    scale = np.float32(amax / qmax) if amax > 0 else np.float32(1.0)
    s = float(scale)
    q = np.rint(y / s)
    d = y - q * s                                        # exact remainder of y / scale at q
    q = np.where(d > 0.5 * s, q + 1, np.where(d < -0.5 * s, q - 1, q))
    d = y - q * s
    tie = np.abs(d) == 0.5 * s
    q = np.where(tie & (np.mod(q, 2) != 0), q + np.sign(d), q)   # half to even
    codes = np.clip(q, -qmax, qmax).astype(np.int16)
    return codes, scale


def dequantize(codes, scale):
    return np.asarray(codes, dtype=np.float64) * float(scale)


def quantize_frames(y, group_blocks=None):
    """Quantise every CS frame of y [n_cs][nblk][M]: one scale per frame (SPEC), or -- with
    group_blocks = list of (b0, b1) block ranges -- one scale per (frame, range) (per-tile
    variant).  Returns (codes int16 like y, scales float32 [n_cs] or [n_cs][n_groups])."""
    y = np.asarray(y, dtype=np.float64)
    codes = np.empty(y.shape, dtype=np.int16)
    if group_blocks is None:
        scales = np.empty(y.shape[0], dtype=np.float32)
        for i in range(y.shape[0]):
            codes[i], scales[i] = quantize(y[i])
    else:
        scales = np.empty((y.shape[0], len(group_blocks)), dtype=np.float32)
        for i in range(y.shape[0]):
            for gi, (b0, b1) in enumerate(group_blocks):
                codes[i, b0:b1], scales[i, gi] = quantize(y[i, b0:b1])
    return codes, scales


# -- f2: paper-faithful frame-level measurement ---------------------------------------------------
def measure_frame(frames: np.ndarray, A_bits: np.ndarray, G: int, with_scale: bool = True):
    """Eq. (1) P:83-85 as the paper states it: one dense A (m x n, n = W*H) measures
    the whole vectorised residual of every CS frame: y = A r, r = vec(F_cs - F_key) row-major
    (SPEC.md:89).  frames uint8 [T][H][W] of one stream -> (y, S) fp64 [n_cs][m], CS frames in
    GOP order (a1).  Exact in fp64 while max|A| * 255 * n < 2^29 (all terms multiples of 2^-24),
    which the function checks."""
    T, H, W = frames.shape
    A = phi_values(A_bits)
    m, n = A.shape
    if n != W * H:
        raise ValueError("A must have W*H columns")
    if A.size and float(np.max(np.abs(A))) * 255.0 * n >= 2.0 ** 29:
        raise ValueError("entries too large for the exact fp64 sum")
    n_cs = cs_frame_count(T, G)
    y = np.empty((n_cs, m))
    S = np.empty((n_cs, m)) if with_scale else None
    i = 0
    for key_t, cs_ts in gop_partition(T, G):
        for t in cs_ts:
            r = residual(frames[t], frames[key_t]).reshape(-1).astype(np.float64)
            y[i] = A @ r
            if with_scale:
                S[i] = np.abs(A) @ np.abs(r)
            i += 1
    return y, S


def block_matrix_as_frame(phi_bits: np.ndarray, W: int, H: int, B: int) -> np.ndarray:
    """The frame-level A (fp16 bits, [nblk*M][W*H]) that computes the block-based measurement: row
    (b, i) holds Phi[i] at block b's pixels (inside the frame).  Used to tie f2 to a4."""
    phi = np.asarray(phi_bits, dtype=np.uint16)
    M = phi.shape[0]
    nby, nbx = block_grid(W, H, B)
    A = np.zeros((nby * nbx * M, H * W), dtype=np.uint16)
    for b in range(nby * nbx):
        by, bx = divmod(b, nbx)
        for j in range(B * B):
            Y, X = by * B + j // B, bx * B + j % B
            if Y < H and X < W:
                A[b * M:(b + 1) * M, Y * W + X] = phi[:, j]
    return A


# -- f3: adjoint / back-projection ---------------------------------------------------------------
def frame_unblocks(X: np.ndarray, W: int, H: int, B: int) -> np.ndarray:
    """Inverse of frame_blocks: [nby*nbx][B*B] (block raster order, row-major inside the block)
    -> [H][W], dropping the zero padding outside the frame."""
    nby, nbx = block_grid(W, H, B)
    X = np.asarray(X)
    full = X.reshape(nby, nbx, B, B).transpose(0, 2, 1, 3).reshape(nby * B, nbx * B)
    return full[:H, :W]


def adjoint_blocks(v: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """SPEC.md:145-153 adjoint: A^T v for every block row v_b of v [nblk][M] -> [nblk][N],
    x_b = Phi^T v_b (fp64)."""
    return np.asarray(v, dtype=np.float64) @ np.asarray(phi, dtype=np.float64)


def adjoint(meas: np.ndarray, phi_bits: np.ndarray, W: int, H: int, B: int) -> np.ndarray:
    """Back-projection x0 = Phi^T y of every block of every frame (the TVAL3
    initial point x = A^T y), reassembled into frames: meas [n][nblk][M] (the
    measurement layout, a6) -> fp64 [n][H][W]."""
    phi = phi_values(phi_bits)
    meas = np.asarray(meas, dtype=np.float64)
    return np.stack([frame_unblocks(adjoint_blocks(meas[i], phi), W, H, B) for i in range(meas.shape[0])]) \
        if meas.shape[0] else np.zeros((0, H, W))


def adjoint_tolerance_scale(meas: np.ndarray, phi_bits: np.ndarray, W: int, H: int, B: int) -> np.ndarray:
    """S[n][y][x] = sum_m |Phi_mj| |v_m| for the pixel's block and in-block index j (the per-entry
    scale of the acceptance bound, in the form BASELINE.json:5 states for y)."""
    return adjoint(np.abs(np.asarray(meas, dtype=np.float64)),
                   np.abs(phi_values(phi_bits)).astype(np.float16).view(np.uint16), W, H, B)


# -- f4: closed-loop key frame through the stand-in intra codec -----------------------------------
# 8x8 block DCT, uniform quantisation by quant_scale * the standard luminance
# perceptual matrix, dequantise, inverse DCT, clamp to [0, 255]; edge-replication padding to
# multiples of 8.  The transform is defined in fixed point (R21) so that every integer
# decision (coefficient rounding, pixel rounding) is exact and identical on every platform
# ("bit-exact deterministic").  Entropy coding and the CR-23 rate search
# are host-side and out of scope.
JPEG_LUMA = np.array([
    [16, 11, 10, 16, 24, 40, 51, 61],
    [12, 12, 14, 19, 26, 58, 60, 55],
    [14, 13, 16, 24, 40, 57, 69, 56],
    [14, 17, 22, 29, 51, 87, 80, 62],
    [18, 22, 37, 56, 68, 109, 103, 77],
    [24, 35, 55, 64, 81, 104, 113, 92],
    [49, 64, 78, 87, 103, 121, 120, 101],
    [72, 92, 95, 98, 112, 100, 103, 99]], dtype=np.int64)   # ITU-T T.81 Annex K, Table K.1
DCT_BITS = 12


def dct_basis() -> np.ndarray:
    """Orthonormal 8-point DCT-II: C[u][x] = a(u) cos((2x+1) u pi / 16), a(0) = sqrt(1/8),
    a(u>0) = sqrt(2/8); the 2-D transform of a block s is C s C^T."""
    u = np.arange(8)[:, None]
    x = np.arange(8)[None, :]
    a = np.where(u == 0, np.sqrt(1.0 / 8.0), np.sqrt(2.0 / 8.0))
    return a * np.cos((2 * x + 1) * u * np.pi / 16.0)


def dct_basis_int() -> np.ndarray:
    """C scaled by 2^12 and rounded to integers (the fixed-point basis of R21)."""
    return np.rint(dct_basis() * (1 << DCT_BITS)).astype(np.int64)


def key_qsteps(quant_scale: float) -> np.ndarray:
    """Integer quantiser steps [v][u] = clip(round(quant_scale * JPEG_LUMA), 1, 4096) (R21)."""
    return np.clip(np.rint(quant_scale * JPEG_LUMA), 1, 4096).astype(np.int64)


def pad8(frame: np.ndarray) -> np.ndarray:
    """Edge replication to multiples of 8."""
    H, W = frame.shape
    return np.pad(frame, ((0, (-H) % 8), (0, (-W) % 8)), mode="edge")


def intra_forward(frame: np.ndarray, qsteps: np.ndarray) -> np.ndarray:
    """Quantised DCT coefficients int16 [nby8][nbx8][8 (v)][8 (u)] of a uint8 frame (R21).
    Per 8x8 block s (level-shifted by -128): t1 = s Ci^T (exact, |t1| < 2^21);
    t1 = floor((t1 + 2^4) / 2^5); t2 = Ci t1 (exact, |t2| < 2^30; scale 2^19);
    q = sign(t2) * floor((|t2| + qstep * 2^18) / (qstep * 2^19))  (round half away from zero)."""
    Ci = dct_basis_int()
    P = pad8(np.asarray(frame)).astype(np.int64) - 128
    nby, nbx = P.shape[0] // 8, P.shape[1] // 8
    out = np.empty((nby, nbx, 8, 8), dtype=np.int16)
    d = np.asarray(qsteps, dtype=np.int64) << 19
    for by in range(nby):
        for bx in range(nbx):
            s = P[by * 8:(by + 1) * 8, bx * 8:(bx + 1) * 8]
            t1 = (s @ Ci.T + 16) >> 5
            t2 = Ci @ t1
            q = np.sign(t2) * ((np.abs(t2) + d // 2) // d)
            out[by, bx] = np.clip(q, -32768, 32767)
    return out


def intra_inverse(coef: np.ndarray, qsteps: np.ndarray, W: int, H: int) -> np.ndarray:
    """Decoded uint8 frame [H][W] (Eq. 2's F-hat): dq = q * qstep; t1 = dq Ci (scale 2^12),
    t1 = floor((t1 + 2^11) / 2^12); t2 = Ci^T t1; pixel = floor((t2 + 2^11) / 2^12) + 128, clamped to
    [0, 255]; the padding is cropped."""
    Ci = dct_basis_int()
    coef = np.asarray(coef, dtype=np.int64)
    nby, nbx = coef.shape[:2]
    out = np.empty((nby * 8, nbx * 8), dtype=np.int64)
    half = 1 << (DCT_BITS - 1)
    for by in range(nby):
        for bx in range(nbx):
            dq = coef[by, bx] * np.asarray(qsteps, dtype=np.int64)
            t1 = (dq @ Ci + half) >> DCT_BITS
            t2 = Ci.T @ t1
            out[by * 8:(by + 1) * 8, bx * 8:(bx + 1) * 8] = ((t2 + half) >> DCT_BITS) + 128
    return np.clip(out, 0, 255)[:H, :W].astype(np.uint8)


def decode_key(frame: np.ndarray, qsteps: np.ndarray) -> np.ndarray:
    """F-hat_key = decode(encode(F_key)) (Eq. 2), computed at the encoder (closed loop)."""
    H, W = frame.shape
    return intra_inverse(intra_forward(frame, qsteps), qsteps, W, H)


def encode_stream_closed_loop(frames: np.ndarray, phi_bits: np.ndarray, G: int, B: int, qsteps: np.ndarray,
                              with_scale: bool = True):
    """As encode_stream, with every CS frame's residual taken against its GOP's DECODED key frame
    (Eq. 3: D = F_N - F-hat_key; "we reconstruct key frame, which is subtracted from CS
    frames")."""
    frames = np.array(frames, copy=True)
    for key_t, _ in gop_partition(frames.shape[0], G):
        frames[key_t] = decode_key(frames[key_t], qsteps)
    return encode_stream(frames, phi_bits, G, B, with_scale)


def encode_stream_gop_phis(frames: np.ndarray, phis_bits, G: int, B: int, with_scale: bool = True):
    """f4 variant, per-GOP matrices (seed xor GOP index): GOP g of the stream is
    measured with phis_bits[g % len(phis_bits)]; otherwise encode_stream."""
    T, H, W = frames.shape
    phis = [phi_values(p) for p in phis_bits]
    nby, nbx = block_grid(W, H, B)
    n_cs = cs_frame_count(T, G)
    y = np.empty((n_cs, nby * nbx, phis[0].shape[0]))
    S = np.empty_like(y) if with_scale else None
    i = 0
    for g, (key_t, cs_ts) in enumerate(gop_partition(T, G)):
        phi = phis[g % len(phis)]
        for t in cs_ts:
            R = frame_blocks(residual(frames[t], frames[key_t]), B)
            y[i] = measure(R, phi)
            if with_scale:
                S[i] = tolerance_scale(R, phi)
            i += 1
    return y, S


def encode_stream_chained(frames: np.ndarray, phi_bits: np.ndarray, G: int, B: int, with_scale: bool = True):
    """f4 variant, Eq. (3) P:91 read literally: D_N = F_N - F_{N-1}, every CS frame against the
    PREVIOUS raw frame (open loop); keys still come from the GOP partition (a1) and are not measured."""
    T, H, W = frames.shape
    phi = phi_values(phi_bits)
    nby, nbx = block_grid(W, H, B)
    n_cs = cs_frame_count(T, G)
    y = np.empty((n_cs, nby * nbx, phi.shape[0]))
    S = np.empty_like(y) if with_scale else None
    i = 0
    for _, cs_ts in gop_partition(T, G):
        for t in cs_ts:
            R = frame_blocks(residual(frames[t], frames[t - 1]), B)
            y[i] = measure(R, phi)
            if with_scale:
                S[i] = tolerance_scale(R, phi)
            i += 1
    return y, S


# -- a7 ------------------------------------------------------------------------------------------
def compression_ratio(W: int, H: int, G: int, B: int, M: int, T: int = 0, key_cr: float = 1.0,
                      bits_per_measurement: int = 8) -> float:
    """CR = original bits / (key-frame bits + measurement bits) (BASELINE.json:5).

    Original: T frames of W*H 8-bit pixels.  Key frames: W*H*8/key_cr bits each
    (key_cr = 1: raw pass-through).  CS frames: nblk*M measurements of
    `bits_per_measurement` bits (8 = the paper's sample-count convention, under
    which CR_cs = n/m as in P:99 "The compression ratio of all CS frames is 50").
    T = 0 means one full GOP.  Real GOP composition and padded blocks counted."""
    T = G if T == 0 else T
    gops = gop_partition(T, G)
    n_key = len(gops)
    n_cs = sum(len(cs) for _, cs in gops)
    nby, nbx = block_grid(W, H, B)
    orig = T * W * H * 8.0
    key_bits = n_key * W * H * 8.0 / key_cr
    meas_bits = n_cs * nby * nbx * M * float(bits_per_measurement)
    return orig / (key_bits + meas_bits)


def total_cr(G: int, key_cr: float, cs_cr: float) -> float:
    """Total CR of one GOP from the per-frame ratios: G frames cost 1/key_cr + (G-1)/cs_cr
    frame-equivalents (Table I: reproduces all nine rows)."""
    return G / (1.0 / key_cr + (G - 1) / cs_cr)


# -- acceptance ----------------------------------------------------------------------------------
def check_tolerance(y_gpu: np.ndarray, y: np.ndarray, S: np.ndarray, rel: float = 1e-5):
    """BASELINE.json:5 acceptance: |y_gpu - y| <= rel * S per entry; S == 0 => y_gpu == 0.
    Returns (ok, stats dict)."""
    y_gpu = np.asarray(y_gpu, dtype=np.float64)
    d = np.abs(y_gpu - y)
    bound = rel * S
    bad = d > bound
    zero = S == 0
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(zero, 0.0, d / np.where(zero, 1.0, S))
    stats = {
        "n": int(y.size),
        "n_bad": int(bad.sum()),
        "max_rel": float(ratio.max()) if ratio.size else 0.0,
        "n_zero_scale": int(zero.sum()),
        "max_abs_at_zero_scale": float(np.abs(y_gpu[zero]).max()) if zero.any() else 0.0,
        "frac_bit_equal_rn32": float(np.mean(y_gpu.astype(np.float32) == y.astype(np.float32))) if y.size else 1.0,
    }
    return stats["n_bad"] == 0 and not np.isnan(y_gpu).any(), stats
