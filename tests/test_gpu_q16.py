"""GPU parity of the fused 16-bit quantisation.

The kernel quantises ITS fp32 measurements y_gpu (|y_gpu - y| <= 1e-5 * S, BASELINE.json:5)
with an fp32 scale and an fp32 rounding decision (R17-R19).  Against the exact y of the
fp64 oracle this fixes, per scale group with exact maximum a and tolerance scale Smax:
  * scale:  |scale - a/32767| <= 1e-5 * Smax / 32767 + 2^-22 * scale;  all-zero group -> 1.0
  * codes:  with t = y * inv (exact y, inv = fl32(1/scale) of the kernel's scale; the decision
            rule of DESIGN.md R18) and d = 1e-5 * S * inv + |t| 2^-22,
            |code - t| <= 0.5 + d, and code == round(t) wherever t is farther than d from a tie
            (entries with S == 0 are exactly 0);  |code| <= 32767.
Both sides decide in fp32 on their own y, so codes may differ from the oracle's only at ties
within the tolerance band.  Two further bitwise checks tie q16 to the fp32 path: the codes equal
round(y_gpu * inv) computed on the host from the fp32 output of the same kernel, and the
per-frame scale equals the maximum of the per-row scales.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1311_1419_b200 as P  # noqa: E402

REL = 1e-5
QMAX = 32767


def kernel_fp32_decision(y, scale):
    """EMULATION of the kernel's rounding decision (R18), kept here in the test, not in
    the oracle: code = round-half-even of fl32(y) * fl32(1 / scale) (one FFMA against 1.5 * 2^23 in
    the kernel; an fp32 x fp32 product is exact in fp64, so np.rint of it is that rounding).  Used
    only to check the kernel bitwise against ITS OWN fp32 output; against the exact oracle the tie
    band of check_group applies."""
    inv = (np.float32(1.0) / np.asarray(scale, dtype=np.float32)).astype(np.float64)
    return np.clip(np.rint(np.asarray(y, dtype=np.float32).astype(np.float64) * inv), -QMAX, QMAX).astype(np.int16)


def check_group(codes, scale, y, S):
    """codes int [n], scale float32, exact y / S fp64 [n] of one scale group."""
    codes = np.asarray(codes, dtype=np.int64)
    scale = float(scale)
    a = float(np.max(np.abs(y))) if y.size else 0.0
    if a == 0.0:
        assert np.all(codes == 0) and scale == 1.0
        return
    smax = float(np.max(S))
    assert abs(scale - a / QMAX) <= REL * smax / QMAX + 2.0 ** -22 * scale, (scale, a / QMAX)
    inv = float(np.float32(1.0) / np.float32(scale))
    t = y * inv
    d = REL * S * inv + np.abs(t) * 2.0 ** -22
    assert np.all(np.abs(codes) <= QMAX)
    assert np.all(np.abs(codes - t) <= 0.5 + d + 1e-12), float(np.max(np.abs(codes - t) - d))
    away = np.abs(np.abs(t - np.floor(t)) - 0.5) > d + 1e-9
    assert np.array_equal(codes[away], np.rint(t[away]).astype(np.int64))
    assert np.all(codes[S == 0] == 0)
    # dequantisation error (widened by the tolerance band)
    assert np.all(np.abs(codes * scale - y) <= scale * (0.5 + 2.0 ** -21) + REL * S + 2.0 ** -22 * np.abs(y))


def check_q16(codes, scales, y, S, nby, nbx, granularity):
    n_cs = y.shape[0]
    M = y.shape[2]
    assert codes.shape == y.shape
    for i in range(n_cs):
        if granularity == P.Encoder.Q16_FRAME:
            check_group(codes[i].ravel(), scales[i], y[i].ravel(), S[i].ravel())
        else:
            for r in range(nby):
                sl = slice(r * nbx, (r + 1) * nbx)
                check_group(codes[i, sl].ravel(), scales[i, r], y[i, sl].ravel(), S[i, sl].ravel())
    del M


def run_q16(enc, fd, granularity):
    codes, scales = enc.encode_batch_q16(fd, granularity)
    torch.cuda.synchronize()
    return codes, scales


def fp32_consistency(enc, fd, codes_f, scales_f, codes_r, scales_r):
    """Bitwise: q16 codes == round-half-even(y_gpu * fl32(1/scale)) from the fp32 output of the same
    kernel (exact fp64 product), and the frame scale == max of the row scales."""
    y32 = enc.encode_batch(fd)
    torch.cuda.synchronize()
    y32 = y32.cpu().numpy().astype(np.float64)
    sf, sr = scales_f.cpu().numpy(), scales_r.cpu().numpy()
    assert np.array_equal(kernel_fp32_decision(y32, sf[:, None, None]), codes_f.cpu().numpy())
    sr_blk = np.repeat(sr, enc.nbx, axis=1)[:, :enc.nblk, None]
    assert np.array_equal(kernel_fp32_decision(y32, sr_blk), codes_r.cpu().numpy())
    assert np.array_equal(sf, sr.max(axis=1))


CASES = [
    # name, W, H, T, G, B, M   (store paths: M=4 direct 8-byte, M%8==0 staged, else scalar)
    ("c1_m64", 176, 144, 4, 4, 16, 64),
    ("b8_m4", 160, 72, 7, 4, 8, 4),
    ("b8_m8", 96, 40, 5, 4, 8, 8),
    ("b16_m12", 112, 50, 5, 3, 16, 12),
    ("b16_m24", 176, 144, 3, 2, 16, 24),
    ("b16_m40", 64, 33, 4, 4, 16, 40),
    ("b16_m128", 352, 288, 3, 3, 16, 128),
    ("b32_m64", 640, 100, 3, 3, 32, 64),
    ("b32_m72", 96, 64, 3, 3, 32, 72),
    # row-scale register paths (one fold, M = 16/32 and 48/64): multi-row tiles, ragged last tile
    ("b16_m16", 208, 90, 5, 4, 16, 16),
    ("b16_m32", 400, 150, 4, 2, 16, 32),
    ("b16_m48", 176, 60, 4, 3, 16, 48),
    ("b8_m16", 128, 56, 5, 3, 8, 16),
    # per-frame store path not applicable (nblk * M not a multiple of 8): two passes
    ("b8_m3", 48, 40, 5, 4, 8, 3),
    ("b8_m5", 48, 24, 5, 4, 8, 5),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_q16_parity(case):
    name, W, H, T, G, B, M = case
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, T=T, G=G, B=B, Ms=(M,), S=2)
    frames = synth.gen_video(cfg)
    phi = synth.phi_from_seed(synth.phi_seed() + M, M, B * B)
    y, S = oracle.encode(frames, phi, G, B)
    enc = P.Encoder(W, H, G, B, M, phi)
    fd = torch.from_numpy(frames).cuda()
    cf, sf = run_q16(enc, fd, P.Encoder.Q16_FRAME)
    check_q16(cf.cpu().numpy(), sf.cpu().numpy(), y, S, enc.nby, enc.nbx, P.Encoder.Q16_FRAME)
    cr, sr = run_q16(enc, fd, P.Encoder.Q16_ROW)
    assert sr.shape == (y.shape[0], enc.nby)
    check_q16(cr.cpu().numpy(), sr.cpu().numpy(), y, S, enc.nby, enc.nbx, P.Encoder.Q16_ROW)
    fp32_consistency(enc, fd, cf, sf, cr, sr)
    # agreement with the oracle's own quantiser (exact y): codes equal except inside tie bands
    oc, osc = oracle.quantize_frames(y)
    diff = np.abs(cf.cpu().numpy().astype(np.int64) - oc)
    assert diff.max() <= 1 and (diff != 0).mean() < 1e-2


def test_q16_zero_and_static():
    """key == every CS frame: y = 0 -> codes 0, scale 1; one static block row
    (zero residual) inside a moving frame gets scale 1 in row mode."""
    W, H, B, M, G = 64, 48, 16, 32, 4
    phi = synth.phi_from_seed(5, M, B * B)
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, (H, W), dtype=np.uint8)
    frames = np.repeat(f[None, None], G, axis=1).copy()
    frames[0, 2, 16:] = rng.integers(0, 256, (H - 16, W), dtype=np.uint8)   # rows 1,2 move in frame 2
    enc = P.Encoder(W, H, G, B, M, phi)
    fd = torch.from_numpy(frames).cuda()
    cf, sf = run_q16(enc, fd, P.Encoder.Q16_FRAME)
    cr, sr = run_q16(enc, fd, P.Encoder.Q16_ROW)
    sf, sr, cf, cr = sf.cpu().numpy(), sr.cpu().numpy(), cf.cpu().numpy(), cr.cpu().numpy()
    assert sf[0] == 1.0 and sf[2] == 1.0 and np.all(cf[[0, 2]] == 0)
    assert sf[1] != 1.0
    assert sr[1, 0] == 1.0 and np.all(cr[1, :enc.nbx] == 0) and np.all(sr[1, 1:] != 1.0)
    y, S = oracle.encode(frames, phi, G, B)
    check_q16(cf, sf, y, S, enc.nby, enc.nbx, P.Encoder.Q16_FRAME)
    check_q16(cr, sr, y, S, enc.nby, enc.nbx, P.Encoder.Q16_ROW)


def test_q16_saturating_values():
    """Largest residuals (+-255) with large Phi entries: scale near its maximum, the max entry
    code exactly +-32767."""
    W, H, B, M, G = 32, 32, 16, 16, 2
    phi = (np.sign(synth.phi_from_seed(8, M, B * B).view(np.float16).astype(np.float64)) * 1024.0)
    phi_bits = phi.astype(np.float16).view(np.uint16)
    frames = np.zeros((1, 2, H, W), np.uint8)
    frames[0, 1] = 255
    frames[0, 1, :8] = 0
    enc = P.Encoder(W, H, G, B, M, phi_bits)
    fd = torch.from_numpy(frames).cuda()
    cf, sf = run_q16(enc, fd, P.Encoder.Q16_FRAME)
    y, S = oracle.encode(frames, phi_bits, G, B)
    c = cf.cpu().numpy()
    check_q16(c, sf.cpu().numpy(), y, S, enc.nby, enc.nbx, P.Encoder.Q16_FRAME)
    assert np.abs(c).max() == QMAX


@pytest.mark.parametrize("name,Ms", [("C4", (16, 128)), ("C5", (4,))])
def test_q16_full_size(name, Ms):
    """Full-size frames in the bench launch; a few CS frames checked whole against the oracle
    (the per-frame maximum needs every block of the frame)."""
    cfg = synth.CONFIGS[name]
    if name == "C5":
        cfg = cfg.with_(S=8)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    rng = np.random.default_rng(11)
    n_cs_s = oracle.cs_frame_count(cfg.T, cfg.G)
    order = [(k, t) for k, cs in oracle.gop_partition(cfg.T, cfg.G) for t in cs]
    for M in Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        cf, sf = run_q16(enc, fd, P.Encoder.Q16_FRAME)
        cr, sr = run_q16(enc, fd, P.Encoder.Q16_ROW)
        cf, sf, cr, sr = cf.cpu().numpy(), sf.cpu().numpy(), cr.cpu().numpy(), sr.cpu().numpy()
        picks = [n_cs_s - 1] + list(rng.integers(0, n_cs_s, 2))
        for s in sorted({0, cfg.S - 1}):
            for i in picks:
                key, t = order[i]
                y, S = oracle.encode_stream(frames[s][[key, t]], phi, 2, cfg.B)
                gi = s * n_cs_s + i
                check_q16(cf[gi:gi + 1], sf[gi:gi + 1], y, S, enc.nby, enc.nbx, P.Encoder.Q16_FRAME)
                check_q16(cr[gi:gi + 1], sr[gi:gi + 1], y, S, enc.nby, enc.nbx, P.Encoder.Q16_ROW)


def test_q16_plans_bitwise_identical():
    """Every candidate plan gives the same codes and scales (both granularities)."""
    cfg = synth.CONFIGS["C2"].with_(T=10)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, cfg.M, phi)
    ref = None
    for k in range(enc.num_candidates()):
        enc.set_candidate(k)
        got = []
        for gran in (P.Encoder.Q16_FRAME, P.Encoder.Q16_ROW):
            try:
                got += list(run_q16(enc, fd, gran))
            except P.CSError as e:
                assert gran == P.Encoder.Q16_ROW and e.code == P.CS_ERR_UNSUPPORTED
                got += [None, None]
        if ref is None:
            ref = got
            continue
        for a, b in zip(ref, got):
            if a is not None and b is not None:
                assert torch.equal(a, b), k


def test_q16_bad_args():
    enc = P.Encoder(64, 32, 4, 16, 16, synth.phi_from_seed(1, 16, 256))
    fd = torch.zeros((1, 4, 32, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(P.CSError):
        enc.encode_batch_q16(fd, granularity=7)
    codes = torch.empty((3, 8, 16), dtype=torch.int16, device="cuda")
    scales = torch.empty(3, dtype=torch.float32, device="cuda")
    rc = P.lib().cs_encode_batch_q16(enc._h, fd.data_ptr(), 1, 4, 0, codes.data_ptr() + 2, scales.data_ptr(), 0)
    assert rc == P.CS_ERR_ARG
    rc = P.lib().cs_encode_batch_q16(enc._h, fd.data_ptr(), 1, 4, 0, None, scales.data_ptr(), 0)
    assert rc == P.CS_ERR_ARG
    # G = 1: nothing to encode, success
    enc1 = P.Encoder(64, 32, 1, 16, 16, synth.phi_from_seed(1, 16, 256))
    c, s = enc1.encode_batch_q16(fd)
    assert c.numel() == 0 and s.numel() == 0


@pytest.mark.parametrize("name,M", [("C4", 16), ("C4", 32), ("C5", 4), ("C3", 64)])
def test_q16_frame_store_path_bitwise(name, M):
    """CS_Q16_FRAME with 8 M <= N stores y and re-quantises it (one measurement pass).  Bitwise: the
    scales are fl32(max|y_gpu| / 32767) of the fp32 kernel's own output and the codes are the kernel's
    fp32 decision on that output (kernel_fp32_decision); and the oracle check with the tie band."""
    base = synth.CONFIGS[name]
    cfg = base.with_(T=min(base.T, 2 * base.G + 3), S=min(base.S, 2))
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    assert 8 * M <= cfg.B ** 2
    c1, s1 = run_q16(enc, fd, P.Encoder.Q16_FRAME)
    y32 = enc.encode_batch(fd)
    torch.cuda.synchronize()
    y32 = y32.cpu().numpy()
    amax = np.abs(y32).reshape(y32.shape[0], -1).max(axis=1)
    want_s = np.where(amax > 0, (amax / np.float32(32767)).astype(np.float32), np.float32(1.0))
    assert np.array_equal(s1.cpu().numpy(), want_s)
    assert np.array_equal(c1.cpu().numpy(), kernel_fp32_decision(y32, want_s[:, None, None]))
    y, S = oracle.encode(frames, phi, cfg.G, cfg.B)
    check_q16(c1.cpu().numpy(), s1.cpu().numpy(), y, S, enc.nby, enc.nbx, P.Encoder.Q16_FRAME)
