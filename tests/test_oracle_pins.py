"""Pins of the fp64 oracle against what the paper and the mathematics fix (not against itself).

Each test names the plausible oracle mistake it would catch.  No GPU needed.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from conftest import load_golden


def fp16_bits(values):
    return np.asarray(values, dtype=np.float64).astype(np.float16).view(np.uint16)


def two_frame(key, cs):
    return np.stack([np.asarray(key, np.uint8), np.asarray(cs, np.uint8)])


# ---------------------------------------------------------------- worked examples (golden)
@pytest.mark.parametrize("name", ["worked_e1.json", "worked_e2.json"])
def test_worked_examples(name):
    """Hand-worked examples: catch wrong block order, wrong in-block vectorisation,
    a transposed Phi, a sign flip of the residual, wrong zero padding."""
    g = load_golden(name)
    frames = two_frame(g["key"], g["cs"])
    phi = fp16_bits(g["phi"])
    R = oracle.frame_blocks(oracle.residual(frames[1], frames[0]), g["B"])
    assert R.tolist() == g["residual_blocks"]
    y, S = oracle.encode_stream(frames, phi, g["G"], g["B"])
    assert y.shape == (1, len(g["y"]), 2)
    assert y[0].tolist() == g["y"]  # exact


# ---------------------------------------------------------------- Table I (paper values)
def test_table1_total_cr_closed_form():
    """All nine Total-CR values printed in Table I."""
    t = load_golden("table1_cr.json")
    for r in t["rows"]:
        v = oracle.total_cr(r["gop"], r["key_cr"], r["cs_cr"])
        assert abs(v - r["total_cr"]) <= t["tolerance"], r


def test_table1_via_bit_accounting():
    """The bit-accounting CR (original bits / (key + measurement bits)) must reproduce
    Table I when the frame has exactly n/m = cs_cr per CS frame and key CR 23 --
    catches a wrong key count, wrong CS count, or counting the key as a CS frame."""
    t = load_golden("table1_cr.json")
    for r in t["rows"]:
        cs = r["cs_cr"]
        B = cs        # N = cs^2 pixels per block, M = cs measurements per block -> N/M = cs
        W = H = 2 * B
        v = oracle.compression_ratio(W, H, r["gop"], B, cs, T=0, key_cr=r["key_cr"], bits_per_measurement=8)
        assert abs(v - r["total_cr"]) <= t["tolerance"], (r, v)


def test_cr_special_cases():
    # key-only GOP: total CR = key CR
    assert oracle.total_cr(1, 23.0, 60.0) == 23.0
    assert oracle.compression_ratio(32, 32, 1, 16, 4, T=0, key_cr=23.0) == pytest.approx(23.0, rel=1e-15)
    # raw key, one full GOP: G*WH / (WH + (G-1)*nblk*M)   (SURVEY.md D2 "CR nominal")
    assert oracle.compression_ratio(1920, 1080, 8, 16, 16) == pytest.approx(8 * 1920 * 1080 / (1920 * 1080 + 7 * 8160 * 16))
    # C5: 10.894 nominal, not 60
    assert round(oracle.compression_ratio(1280, 720, 32, 8, 4), 3) == 10.894


def test_gop_partition():
    """10 frames, G=4 -> GOP lengths 4,4,2; key = first frame of each."""
    gops = oracle.gop_partition(10, 4)
    assert [1 + len(cs) for _, cs in gops] == [4, 4, 2]
    assert [k for k, _ in gops] == [0, 4, 8]
    assert gops[0][1] == [1, 2, 3]
    assert oracle.gop_partition(5, 1) == [(i, []) for i in range(5)]
    assert oracle.cs_frame_count(300, 8) == 262 and oracle.cs_frame_count(600, 16) == 562
    assert oracle.cs_frame_count(240, 8) == 210 and oracle.cs_frame_count(128, 32) == 124


# ---------------------------------------------------------------- special cases / closed forms
def rand_frames(rng, T, H, W):
    return rng.integers(0, 256, size=(T, H, W), dtype=np.uint8)


def test_zero_residual():
    """key == CS frame -> y == 0 exactly and S == 0."""
    rng = np.random.default_rng(1)
    f = rand_frames(rng, 1, 40, 48)
    frames = np.repeat(f, 5, axis=0)
    phi = synth.phi_from_seed(7, 16, 256)
    y, S = oracle.encode_stream(frames, phi, 5, 16)
    assert np.all(y == 0) and np.all(S == 0)


@pytest.mark.parametrize("B", [2, 8, 16])
def test_identity_rows(B):
    """Phi rows = unit vectors e_{j_m}: y_m = r_{j_m} exactly -- catches a wrong
    in-block index map (row-major j = yy*B + xx) and transposition."""
    N = B * B
    rng = np.random.default_rng(B)
    js = rng.choice(N, size=min(N, 5), replace=False)
    phi = np.zeros((len(js), N))
    phi[np.arange(len(js)), js] = 1.0
    frames = rand_frames(rng, 2, 3 * B + 1, 2 * B + 3)  # ragged
    y, _ = oracle.encode_stream(frames, fp16_bits(phi), 2, B)
    H, W = frames.shape[1:]
    nby, nbx = -(-H // B), -(-W // B)
    r = frames[1].astype(int) - frames[0].astype(int)
    for b in range(nby * nbx):
        by, bx = divmod(b, nbx)
        for m, j in enumerate(js):
            yy, xx = divmod(int(j), B)
            Y, X = by * B + yy, bx * B + xx
            want = r[Y, X] if (Y < H and X < W) else 0
            assert y[0, b, m] == want


def test_full_identity_M_equals_N():
    """M = N identity (lossless diagnostic): y is the residual block itself."""
    B = 4
    rng = np.random.default_rng(3)
    frames = rand_frames(rng, 3, 8, 12)
    y, _ = oracle.encode_stream(frames, fp16_bits(np.eye(B * B)), 3, B)
    for i, t in enumerate([1, 2]):
        r = frames[t].astype(int) - frames[0].astype(int)
        blocks = r.reshape(2, B, 3, B).transpose(0, 2, 1, 3).reshape(6, B * B)
        assert np.array_equal(y[i], blocks)


def test_unit_residual_every_position():
    """One pixel differs by v -> y = v * Phi[:, j] for the block holding it, 0 elsewhere
    (SPEC.md:143 x = e_j -> column j).  Sweeps every in-block position."""
    B, M = 8, 6
    phi = synth.phi_from_seed(11, M, B * B)
    phiv = oracle.phi_values(phi)
    key = np.full((2 * B, 3 * B), 77, np.uint8)
    for yy in range(B):
        for xx in range(B):
            cs = key.copy()
            Y, X = B + yy, 2 * B + xx           # block (1, 2)
            cs[Y, X] = 77 - 50
            y, _ = oracle.encode_stream(two_frame(key, cs), phi, 2, B)
            want = np.zeros((6, M))
            want[1 * 3 + 2] = -50 * phiv[:, yy * B + xx]
            assert np.array_equal(y[0], want), (yy, xx)


def test_linearity():
    """y(R1 + R2) = y(R1) + y(R2) exactly (all values exact in fp64)."""
    rng = np.random.default_rng(5)
    H, W, B = 33, 48, 16
    K = rng.integers(60, 190, size=(H, W)).astype(np.int64)
    d1 = rng.integers(-30, 31, size=(H, W))
    d2 = rng.integers(-30, 31, size=(H, W))
    F1, F2, F3 = K + d1, K + d2, K + d1 + d2
    phi = synth.phi_from_seed(9, 32, 256)
    mk = lambda F: two_frame(K, F)
    y1, _ = oracle.encode_stream(mk(F1), phi, 2, B)
    y2, _ = oracle.encode_stream(mk(F2), phi, 2, B)
    y3, _ = oracle.encode_stream(mk(F3), phi, 2, B)
    assert np.array_equal(y3, y1 + y2)


def test_antisymmetry_and_pow2_scaling():
    rng = np.random.default_rng(6)
    f = rand_frames(rng, 2, 32, 32)
    phi = synth.phi_from_seed(3, 16, 256)
    y, _ = oracle.encode_stream(f, phi, 2, 16)
    ys, _ = oracle.encode_stream(f[::-1].copy(), phi, 2, 16)
    assert np.array_equal(ys, -y)            # swapping key and CS frame negates y
    phi4 = (oracle.phi_values(phi) * 4.0).astype(np.float16).view(np.uint16)
    y4, _ = oracle.encode_stream(f, phi4, 2, 16)
    assert np.array_equal(y4, 4.0 * y)       # Phi * 2^k -> y * 2^k


def test_block_translation():
    """Shifting the whole scene by exactly B pixels permutes the blocks."""
    rng = np.random.default_rng(8)
    B = 8
    big = rand_frames(rng, 2, 4 * B, 6 * B)
    a = big[:, :, : 5 * B].copy()
    b = big[:, :, B:].copy()
    phi = synth.phi_from_seed(4, 5, 64)
    ya, _ = oracle.encode_stream(a, phi, 2, B)
    yb, _ = oracle.encode_stream(b, phi, 2, B)
    ya = ya[0].reshape(4, 5, 5)
    yb = yb[0].reshape(4, 5, 5)
    assert np.array_equal(ya[:, 1:], yb[:, :4])


def test_subnormal_and_saturation():
    # smallest fp16 subnormal 2^-24 times r = 255 -> 255 * 2^-24 exactly (no flush to zero)
    phi = np.zeros((1, 4), np.uint16)
    phi[0, 2] = 0x0001
    key = np.zeros((2, 2), np.uint8)
    cs = key.copy()
    cs[1, 0] = 255                           # j = 1*2 + 0 = 2
    y, S = oracle.encode_stream(two_frame(key, cs), phi, 2, 2)
    assert y[0, 0, 0] == 255 * 2.0 ** -24 and S[0, 0, 0] == 255 * 2.0 ** -24
    # key = 0, CS = 255, Phi = 1 -> 255 * N
    for B in (16, 32):
        f = np.stack([np.zeros((B, B), np.uint8), np.full((B, B), 255, np.uint8)])
        y, _ = oracle.encode_stream(f, fp16_bits(np.ones((3, B * B))), 2, B)
        assert np.all(y == 255 * B * B)
    assert 255 * 256 == 65280 and 255 * 1024 == 261120


def test_exact_against_rational_brute_force():
    """Pure-Python exact rational arithmetic on tiny random inputs, looping over the
    definition y[c][b][m] = sum_{yy,xx} Phi[m][yy*B+xx] * (F_t - F_key)[..] -- independent
    of numpy's matmul; the fp64 oracle must agree bit for bit (exactness claim)."""
    rng = np.random.default_rng(12)
    for trial in range(6):
        B = int(rng.choice([2, 4, 8]))
        H, W = int(rng.integers(1, 3 * B)), int(rng.integers(1, 3 * B))
        T, G, M = int(rng.integers(1, 6)), int(rng.integers(1, 4)), int(rng.integers(1, B * B + 1))
        frames = rand_frames(rng, T, H, W)
        phi = synth.phi_from_seed(100 + trial, M, B * B)
        phif = [[Fraction(float(v)) for v in row] for row in oracle.phi_values(phi)]
        y, _ = oracle.encode_stream(frames, phi, G, B)
        nby, nbx = -(-H // B), -(-W // B)
        i = 0
        for g0 in range(0, T, G):
            for t in range(g0 + 1, min(g0 + G, T)):
                for by in range(nby):
                    for bx in range(nbx):
                        for m in range(M):
                            acc = Fraction(0)
                            for yy in range(B):
                                for xx in range(B):
                                    Y, X = by * B + yy, bx * B + xx
                                    if Y < H and X < W:
                                        r = int(frames[t, Y, X]) - int(frames[g0, Y, X])
                                        acc += phif[m][yy * B + xx] * r
                            assert Fraction(float(y[i, by * nbx + bx, m])) == acc
                i += 1
        assert i == y.shape[0]


def test_exact_against_int64_path():
    """Phi * 2^24 is an integer matrix; integer matmul with the integer residual gives
    y * 2^24 exactly -- a second exact path."""
    cfg = synth.CONFIGS["C1"]
    frames = synth.gen_video(cfg)[0]
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    y, _ = oracle.encode_stream(frames, phi, cfg.G, cfg.B)
    phi_int = (oracle.phi_values(phi) * 2.0 ** 24).astype(np.int64)
    assert np.array_equal(phi_int.astype(np.float64), oracle.phi_values(phi) * 2.0 ** 24)
    for i, t in enumerate([1, 2, 3]):
        r = frames[t].astype(np.int64) - frames[0].astype(np.int64)
        R = r.reshape(9, 16, 11, 16).transpose(0, 2, 1, 3).reshape(99, 256)
        yint = R @ phi_int.T
        assert np.array_equal(yint.astype(np.float64) / 2.0 ** 24, y[i])


def test_output_order_streams_gops():
    """Concatenation order: per stream, per GOP, per CS frame (a6).  Each CS frame t
    differs from its key by exactly t at every pixel, Phi = one row e_0 -> y = t."""
    T, G = 10, 4
    frames = np.zeros((2, T, 4, 4), np.uint8)
    for s in range(2):
        for t in range(T):
            frames[s, t] = 10 * s + t
    phi = np.zeros((1, 4))
    phi[0, 0] = 1.0
    y, _ = oracle.encode(frames, fp16_bits(phi), G, 2)
    # CS frames of T=10, G=4: GOP0 -> 1,2,3 (key 0); GOP1 -> 5,6,7 (key 4); GOP2 -> 9 (key 8)
    want = [1, 2, 3, 1, 2, 3, 1] * 2
    assert y[:, :, 0].tolist() == [[w] * 4 for w in want]


def test_tolerance_scale_properties():
    rng = np.random.default_rng(13)
    f = rand_frames(rng, 3, 24, 40)
    phi = synth.phi_from_seed(21, 8, 64)
    y, S = oracle.encode_stream(f, phi, 3, 8)
    assert np.all(S >= np.abs(y))
    # all-positive Phi and non-negative residual: S == y
    f2 = np.stack([np.zeros((8, 8), np.uint8), rng.integers(0, 256, (8, 8), dtype=np.uint8)])
    y2, S2 = oracle.encode_stream(f2, fp16_bits(np.abs(oracle.phi_values(phi))), 2, 8)
    assert np.array_equal(y2, S2)


def test_check_tolerance_semantics():
    y = np.array([1.0, 0.0, -2.0])
    S = np.array([1.0, 0.0, 4.0])
    ok, st = oracle.check_tolerance(np.array([1.0 + 5e-6, 0.0, -2.0]), y, S)
    assert ok and st["n_zero_scale"] == 1
    ok, _ = oracle.check_tolerance(np.array([1.0, 1e-30, -2.0]), y, S)   # S = 0 demands exact 0
    assert not ok
    ok, _ = oracle.check_tolerance(np.array([1.0 + 2e-5, 0.0, -2.0]), y, S)
    assert not ok


# ---------------------------------------------------------------- f1: 16-bit quantisation
def test_quantize_zero_vector():
    """y = 0 -> codes all zero, scale 1, round-trip exact."""
    codes, scale = oracle.quantize(np.zeros(37))
    assert scale == np.float32(1.0) and np.all(codes == 0)
    assert np.all(oracle.dequantize(codes, scale) == 0)


def test_quantize_bounds_and_extremes():
    """max|y| = 32767*s -> round-trip error <= s/2 (as printed: the oracle decides
    on the exact y); the max element maps to +-32767; antisymmetry.  Catches a decision taken on a
    rounded y or a rounded reciprocal (error above s/2) and a wrong clamp."""
    rng = np.random.default_rng(21)
    for trial in range(200):
        y = rng.normal(size=rng.integers(1, 400)) * 10.0 ** rng.uniform(-6, 6)
        codes, scale = oracle.quantize(y)
        err = np.abs(oracle.dequantize(codes, scale) - y)
        # s/2 wherever |y| <= 32767 s; the clamp at 32767 (s = fl32(max/32767) may sit
        # just below max/32767) adds |y| - 32767 s, at most 2^-24 * max|y|
        over = np.maximum(np.abs(y) - 32767 * float(scale), 0.0)
        assert np.all(err <= float(scale) * 0.5 + over), (trial, err.max() / scale)
        k = np.argmax(np.abs(y))
        assert abs(int(codes[k])) == 32767
        assert np.all(np.abs(codes.astype(int)) <= 32767)
        c2, s2 = oracle.quantize(-y)
        assert s2 == scale and np.array_equal(c2, -codes)
    s = np.float32(0.25)
    y = np.array([32767 * 0.25, -0.125, 0.375, 1.0])      # ties: -0.5 -> -0 (even), 1.5 -> 2 (even)
    codes, scale = oracle.quantize(y)
    assert scale == s and codes.tolist() == [32767, 0, 2, 4]


def _round_half_even(fr: Fraction) -> int:
    f = fr.numerator // fr.denominator
    rem = fr - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2 == 1):
        return f + 1
    return f


def test_quantize_against_rational_brute_force():
    """codes = round(y / scale) in exact rational arithmetic (ties to even, R17), on
    measurement-like values (multiples of 2^-24) placed ON and within a few 2^-24 of every kind of
    tie -- the cases where an fp64 quotient, an fp32 y or an fp32 reciprocal decide wrongly."""
    rng = np.random.default_rng(23)
    checked = 0
    for trial in range(60):
        amax = float(rng.integers(1, 2 ** 20)) * 2.0 ** -int(rng.integers(0, 24))
        scale = float(np.float32(amax / 32767))
        k = rng.integers(-32767, 32767, size=40).astype(np.float64)
        eps = rng.integers(-3, 4, size=40) * 2.0 ** -24
        y = np.concatenate([[amax], (k + 0.5) * scale + eps, rng.uniform(-amax, amax, 40)])
        y = np.clip(np.rint(y * 2.0 ** 24) * 2.0 ** -24, -amax, amax)     # exact measurement grid
        codes, sc = oracle.quantize(y)
        assert float(sc) == scale
        for yi, ci in zip(y, codes):
            want = _round_half_even(Fraction(float(yi)) / Fraction(scale))
            assert int(ci) == max(-32767, min(32767, want)), (yi, scale)
            checked += 1
    assert checked == 60 * 81


def test_quantize_frames_per_group():
    rng = np.random.default_rng(22)
    y = rng.normal(size=(3, 10, 4))
    c, s = oracle.quantize_frames(y)
    assert s.shape == (3,) and c.shape == y.shape
    for i in range(3):
        ci, si = oracle.quantize(y[i])
        assert si == s[i] and np.array_equal(ci, c[i])
    c2, s2 = oracle.quantize_frames(y, [(0, 4), (4, 10)])
    assert s2.shape == (3, 2)
    assert np.array_equal(c2[1, 4:], oracle.quantize(y[1, 4:])[0])


# ---------------------------------------------------------------- f3: adjoint
def test_frame_unblocks_inverts_frame_blocks():
    rng = np.random.default_rng(31)
    for (H, W, B) in [(16, 16, 8), (33, 48, 16), (40, 96, 32), (7, 5, 2)]:
        F = rng.integers(0, 256, (H, W))
        assert np.array_equal(oracle.frame_unblocks(oracle.frame_blocks(F, B), W, H, B), F)


def test_adjoint_identity():
    """SPEC.md:144/153/556: <Phi r, v> == <r, Phi^T v> (per frame, summed over blocks), 1e-9 relative,
    on 100 random instances including ragged frames -- catches a transposed Phi, a wrong block
    placement or in-block order in the reassembly, or a dropped/duplicated block."""
    rng = np.random.default_rng(32)
    for trial in range(100):
        B = int(rng.choice([2, 4, 8]))
        M = int(rng.integers(1, B * B + 1))
        H, W = int(rng.integers(1, 3 * B + 2)), int(rng.integers(1, 3 * B + 2))
        phi = synth.phi_from_seed(int(rng.integers(1 << 30)), M, B * B)
        F = rng.integers(-255, 256, (H, W))
        nby, nbx = oracle.block_grid(W, H, B)
        v = rng.normal(size=(1, nby * nbx, M))
        y = oracle.measure(oracle.frame_blocks(F, B), oracle.phi_values(phi))
        x = oracle.adjoint(v, phi, W, H, B)[0]
        lhs, rhs = float(np.sum(y * v[0])), float(np.sum(F * x))
        assert abs(lhs - rhs) <= 1e-9 * max(1.0, np.sum(np.abs(y * v[0]))), (trial, lhs, rhs)


def test_adjoint_special_cases():
    """v = 0 -> 0; v = e_(b,i) -> row i of Phi laid into block b (cropped at the frame edge);
    Phi = I (M = N) -> the unblocked v; orthonormal rows (a row subset of a permutation) ->
    Phi Phi^T v = v."""
    B, M = 4, 5
    H, W = 6, 10                                    # nby = 2, nbx = 3, ragged both ways
    phi = synth.phi_from_seed(4, M, B * B)
    phiv = oracle.phi_values(phi)
    assert np.all(oracle.adjoint(np.zeros((2, 6, M)), phi, W, H, B) == 0)
    for b in range(6):
        for i in range(M):
            v = np.zeros((1, 6, M))
            v[0, b, i] = 1.0
            x = oracle.adjoint(v, phi, W, H, B)[0]
            want = np.zeros((2 * B, 3 * B))
            by, bx = divmod(b, 3)
            want[by * B:(by + 1) * B, bx * B:(bx + 1) * B] = phiv[i].reshape(B, B)
            assert np.array_equal(x, want[:H, :W]), (b, i)
    eye = np.eye(B * B).astype(np.float16).view(np.uint16)
    v = np.random.default_rng(5).normal(size=(2, 6, B * B))
    x = oracle.adjoint(v, eye, W, H, B)
    for k in range(2):
        assert np.array_equal(x[k], oracle.frame_unblocks(v[k], W, H, B))
    perm = np.random.default_rng(6).permutation(B * B)[:M]
    P = np.zeros((M, B * B))
    P[np.arange(M), perm] = 1.0
    v = np.random.default_rng(7).integers(-100, 100, size=(1, 6, M)).astype(np.float64)  # frame_blocks is integer
    Wf, Hf = 3 * B, 2 * B                           # no cropping: Phi (Phi^T v) == v exactly
    xb = oracle.frame_blocks(oracle.adjoint(v, P.astype(np.float16).view(np.uint16), Wf, Hf, B)[0], B)
    assert np.array_equal(oracle.measure(xb, P), v[0])


def test_adjoint_brute_force():
    """Exact rational loops over the definition x[Y][X] = sum_m Phi[m][j] v[b][m] on a tiny case."""
    B, M, H, W = 2, 3, 3, 5
    phi = synth.phi_from_seed(9, M, B * B)
    phiv = oracle.phi_values(phi)
    rng = np.random.default_rng(8)
    v = rng.integers(-50, 50, size=(1, 6, M)) / 8.0
    x = oracle.adjoint(v, phi, W, H, B)[0]
    for Y in range(H):
        for X in range(W):
            b = (Y // B) * 3 + X // B
            j = (Y % B) * B + X % B
            want = sum(Fraction(float(phiv[m, j])) * Fraction(float(v[0, b, m])) for m in range(M))
            assert Fraction(float(x[Y, X])) == want


def test_adjoint_tolerance_scale_brute_force():
    """S[n][Y][X] = sum_m |Phi[m][j]| |v[n][b][m]| by explicit loops over the definition (b, j the
    pixel's block and in-block index; pixels outside the frame dropped), and S >= |x| everywhere.
    Catches a missing absolute value, a transposed Phi or a block/pixel index mix-up."""
    B, M, H, W = 4, 5, 7, 10
    phi = synth.phi_from_seed(19, M, B * B)
    phiv = oracle.phi_values(phi)
    rng = np.random.default_rng(17)
    nby, nbx = oracle.block_grid(W, H, B)
    v = rng.normal(size=(2, nby * nbx, M)) * 3.0
    S = oracle.adjoint_tolerance_scale(v, phi, W, H, B)
    x = oracle.adjoint(v, phi, W, H, B)
    assert S.shape == (2, H, W)
    for n in range(2):
        for Y in range(H):
            for X in range(W):
                b = (Y // B) * nbx + X // B
                j = (Y % B) * B + X % B
                want = 0.0
                for m in range(M):
                    want += abs(float(phiv[m, j])) * abs(float(v[n, b, m]))
                assert abs(S[n, Y, X] - want) <= 1e-12 * want
    assert np.all(S >= np.abs(x) * (1 - 1e-12))


def test_measure_entries_equals_encode_stream():
    """measure_entries (the sampled checker of the full-size parity tests) = encode_stream at every
    (CS frame, block) of a ragged, multi-GOP, short-last-GOP stream, for 2 streams; y and S bitwise
    (both are exact).  Catches a wrong GOP/CS-frame order, a wrong key or a wrong block crop."""
    for s, (W, H, T, G, B, M) in enumerate([(40, 27, 11, 4, 8, 5), (48, 35, 9, 3, 16, 7)]):
        cfg = synth.CONFIGS["C1"].with_(W=W, H=H, T=T, G=G, B=B, Ms=(M,), S=2)
        frames = synth.gen_video(cfg)
        phi = synth.phi_from_seed(100 + s, M, B * B)
        for st in range(2):
            y, S = oracle.encode_stream(frames[st], phi, G, B)
            n_cs, nblk = y.shape[:2]
            ci, bi = np.meshgrid(np.arange(n_cs), np.arange(nblk), indexing="ij")
            ye, Se = oracle.measure_entries(frames[st], phi, G, B, ci.ravel(), bi.ravel())
            assert np.array_equal(ye, y.reshape(-1, M)) and np.array_equal(Se, S.reshape(-1, M))


# ---------------------------------------------------------------- f4: closed-loop key (Eq. 2-4)
def _psnr(a, b):
    mse = np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2)
    return np.inf if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)


def test_dct_basis_is_the_textbook_dct():
    """C is orthonormal, row 0 constant 1/sqrt(8), and C s C^T of a cosine image has one nonzero
    coefficient at (v, u) -- catches a transposed basis or a wrong normalisation; the integer basis
    is within 1/2 of 2^12 C and keeps the antisymmetry that makes flat blocks DC-only."""
    C = oracle.dct_basis()
    assert np.allclose(C @ C.T, np.eye(8), atol=1e-14)
    assert np.allclose(C[0], np.sqrt(1 / 8))
    x = np.arange(8)
    img = np.outer(np.cos((2 * x + 1) * 2 * np.pi / 16), np.cos((2 * x + 1) * 5 * np.pi / 16))  # v=2, u=5
    D = C @ img @ C.T
    assert abs(D[2, 5]) > 1 and np.sum(np.abs(D) > 1e-12) == 1
    Ci = oracle.dct_basis_int()
    assert np.all(np.abs(Ci - C * 4096) <= 0.5)
    assert np.all(Ci[1:].sum(axis=1) == 0)


def test_key_codec_flat_frame_dc_only():
    """SPEC.md:293 flat gray frame -> DC coefficients only; decoded within 1 grey level."""
    for c in (0, 37, 128, 200, 255):
        f = np.full((16, 24), c, np.uint8)
        for qs in (0.01, 1.0, 4.0):
            q = oracle.intra_forward(f, oracle.key_qsteps(qs))
            assert np.all(q[:, :, 0, 1:] == 0) and np.all(q[:, :, 1:, :] == 0)
    f = np.full((16, 24), 77, np.uint8)
    assert np.all(np.abs(oracle.decode_key(f, oracle.key_qsteps(0.01)).astype(int) - 77) <= 1)


def test_key_codec_near_lossless_and_monotone():
    """SPEC.md:301 minimum scale -> PSNR >= 45 dB; S:318 PSNR non-increasing in quant_scale over a
    ladder; S:295 decoded dimensions == original (ragged frame, edge-replication padding)."""
    cfg = synth.CONFIGS["C1"]
    f = synth.gen_video(cfg)[0, 0]
    ps = [_psnr(oracle.decode_key(f, oracle.key_qsteps(s)), f) for s in (0.01, 0.25, 0.5, 1, 2, 4, 8)]
    assert ps[0] >= 45, ps
    assert all(ps[i] >= ps[i + 1] - 1e-9 for i in range(len(ps) - 1)), ps
    rag = f[:13, :21]
    d = oracle.decode_key(rag, oracle.key_qsteps(1.0))
    assert d.shape == rag.shape and _psnr(d, rag) > 25


def test_key_codec_against_real_dct():
    """The fixed-point forward transform rounds to the same code as the exact real DCT except
    within the basis-rounding band (|t - k - 1/2| small), never by more than 1; the inverse of a
    single coefficient is the textbook basis image (horizontal frequency u along x)."""
    rng = np.random.default_rng(41)
    C = oracle.dct_basis()
    qs = oracle.key_qsteps(1.0)
    n_diff = 0
    for _ in range(200):
        blk = rng.integers(0, 256, (8, 8)).astype(np.uint8)
        q = oracle.intra_forward(blk, qs)[0, 0].astype(np.int64)
        t = (C @ (blk.astype(np.float64) - 128) @ C.T) / qs
        assert np.all(np.abs(q - np.sign(t) * np.floor(np.abs(t) + 0.5)) <= 1)
        n_diff += int(np.sum(q != np.sign(t) * np.floor(np.abs(t) + 0.5)))
    assert n_diff <= 200 * 64 * 0.01
    coef = np.zeros((1, 1, 8, 8), np.int16)
    coef[0, 0, 0, 1] = 40                       # v = 0, u = 1: varies along x only
    img = oracle.intra_inverse(coef, np.ones((8, 8), np.int64) * 4, 8, 8).astype(np.int64)
    assert np.all(img == img[0:1, :])           # every row identical
    want = 128 + 160 * C[1][None, :] * C[0][:, None]
    assert np.all(np.abs(img - want) <= 1)
    assert img[0, 0] > img[0, 7]                # cos decreasing along x


@pytest.mark.parametrize("qs", [0.3, 1.0, 5.0])
def test_closed_loop_cancellation_eq4(qs):
    """Eq. 4 / SPEC.md:371, 554: with M = N (Phi = I) the measurement IS the residual
    against the decoded key, so y + F-hat_key reproduces every CS frame exactly, whatever the key
    codec's error; and the closed-loop residual differs from the open-loop one by exactly the key's
    coding error (Eq. 3)."""
    B = 8
    cfg = synth.CONFIGS["C1"].with_(T=5, G=5)
    frames = synth.gen_video(cfg)[0]
    qst = oracle.key_qsteps(qs)
    eye = np.eye(B * B).astype(np.float16).view(np.uint16)
    y, _ = oracle.encode_stream_closed_loop(frames, eye, 5, B, qst)
    key_hat = oracle.decode_key(frames[0], qst)
    for i in range(4):
        rec = oracle.frame_unblocks(y[i], cfg.W, cfg.H, B) + key_hat.astype(np.float64)
        assert np.array_equal(rec, frames[1 + i].astype(np.float64))
    y_open, _ = oracle.encode_stream(frames, eye, 5, B)
    err = key_hat.astype(np.int64) - frames[0].astype(np.int64)          # e_coding + e_decoding
    diff = oracle.frame_unblocks(y_open[0] - y[0], cfg.W, cfg.H, B)
    assert np.array_equal(diff, err.astype(np.float64))


# ---------------------------------------------------------------- f2: frame-level A (Eq. 1)
def test_frame_level_reduces_to_block_path():
    """A built from Phi block by block reproduces the block path's y exactly (reordered) -- ties
    the frame-level measurement to a4 and catches a wrong vectorisation order (row-major
    r = vec(F)) or a transposed A."""
    B, M = 4, 3
    H, W = 9, 14                                   # ragged: padded blocks outside the frame
    phi = synth.phi_from_seed(12, M, B * B)
    rng = np.random.default_rng(13)
    frames = rng.integers(0, 256, (5, H, W), dtype=np.uint8)
    A = oracle.block_matrix_as_frame(phi, W, H, B)
    yf, Sf = oracle.measure_frame(frames, A, 5)
    yb, Sb = oracle.encode_stream(frames, phi, 5, B)
    assert np.array_equal(yf, yb.reshape(yb.shape[0], -1))
    assert np.array_equal(Sf, Sb.reshape(Sb.shape[0], -1))


def test_frame_level_special_cases():
    """A = I (m = n): y is the residual itself; unit residual at pixel j -> v * A[:, j];
    zero residual -> 0; the paper's QCIF CR-50 shape m = round(25344 / 50) = 507."""
    H, W = 6, 8
    n = H * W
    eye = np.eye(n).astype(np.float16).view(np.uint16)
    rng = np.random.default_rng(14)
    fr = rng.integers(0, 256, (3, H, W), dtype=np.uint8)
    y, _ = oracle.measure_frame(fr, eye, 3)
    for i in range(2):
        assert np.array_equal(y[i], (fr[1 + i].astype(float) - fr[0]).ravel())
    A = synth.phi_from_seed(15, 10, n)
    Av = oracle.phi_values(A)
    for j in (0, 17, n - 1):
        f = np.full((2, H, W), 100, np.uint8)
        f[1].flat[j] = 37
        y, _ = oracle.measure_frame(f, A, 2)
        assert np.array_equal(y[0], -63 * Av[:, j])
    y, S = oracle.measure_frame(np.repeat(fr[:1], 3, axis=0), A, 3)
    assert np.all(y == 0) and np.all(S == 0)
    assert round(176 * 144 / 50) == 507


def test_chained_reference_variant():
    """Eq. 3 literal (D_N = F_N - F_{N-1}): the first CS frame of a GOP equals the key-referenced
    residual; with Phi = I the chained measurements telescope -- their running sum over a GOP is
    the key-referenced measurement (exact)."""
    B = 4
    rng = np.random.default_rng(51)
    frames = rng.integers(0, 256, (9, 8, 12), dtype=np.uint8)
    eye = np.eye(B * B).astype(np.float16).view(np.uint16)
    yc, _ = oracle.encode_stream_chained(frames, eye, 4, B)
    yk, _ = oracle.encode_stream(frames, eye, 4, B)
    order = [(k, t) for k, cs in oracle.gop_partition(9, 4) for t in cs]
    run = None
    for i, (k, t) in enumerate(order):
        run = yc[i] if t == k + 1 else run + yc[i]
        assert np.array_equal(run, yk[i]), (i, k, t)


def test_gop_phis_variant():
    """Per-GOP matrices: one matrix repeated == encode_stream; GOP g's rows equal encode_stream
    with phi_g on that GOP (index g % n)."""
    rng = np.random.default_rng(61)
    frames = rng.integers(0, 256, (11, 8, 12), dtype=np.uint8)
    B, M, G = 4, 5, 3
    phis = [synth.phi_from_seed(100 ^ g, M, B * B) for g in range(2)]
    y1, _ = oracle.encode_stream_gop_phis(frames, [phis[0]], G, B)
    y0, _ = oracle.encode_stream(frames, phis[0], G, B)
    assert np.array_equal(y1, y0)
    y2, _ = oracle.encode_stream_gop_phis(frames, phis, G, B)
    i = 0
    for g, (k, cs) in enumerate(oracle.gop_partition(11, G)):
        yg, _ = oracle.encode_stream(frames[k:k + 1 + len(cs)], phis[g % 2], G, B)
        assert np.array_equal(y2[i:i + len(cs)], yg)
        i += len(cs)
