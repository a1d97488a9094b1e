"""GPU parity of the closed-loop key frame (Eq. 2-4).

The key codec is integer arithmetic end to end (R21), so coefficients and decoded key
frames must be bit-identical to the oracle's.  The measurement against the decoded keys keeps the
north-star tolerance (|dy| <= 1e-5 * sum |Phi r|).
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


def oracle_keys(frames, G, qsteps):
    """[S][ceil(T/G)] decoded keys and coefficients from the oracle."""
    S, T, H, W = frames.shape
    keys, coefs = [], []
    for s in range(S):
        for k, _ in oracle.gop_partition(T, G):
            c = oracle.intra_forward(frames[s, k], qsteps)
            coefs.append(c)
            keys.append(oracle.intra_inverse(c, qsteps, W, H))
    ng = -(-T // G)
    return (np.stack(keys).reshape(S, ng, H, W), np.stack(coefs).reshape(S, ng, *coefs[0].shape))


@pytest.mark.parametrize("W,H,T,G,qs", [(176, 144, 9, 4, 1.0), (64, 20, 5, 2, 0.05), (96, 43, 7, 3, 8.0),
                                        (352, 288, 17, 8, 2.5)])
def test_key_codec_bit_exact(W, H, T, G, qs):
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, T=T, G=G, S=2)
    frames = synth.gen_video(cfg)
    qst = oracle.key_qsteps(qs)
    enc = P.Encoder(W, H, G, 16, 16, synth.phi_from_seed(1, 16, 256))
    keys, coef = enc.key_codec(torch.from_numpy(frames).cuda(), P.key_qsteps(qs))
    torch.cuda.synchronize()
    ok, oc = oracle_keys(frames, G, qst)
    assert np.array_equal(coef.cpu().numpy(), oc)
    assert np.array_equal(keys.cpu().numpy(), ok)


def test_key_codec_extremes():
    """Noise, 0/255 checkerboards (largest AC coefficients), flat 0 and 255 frames, minimum and
    maximum steps: still bit-exact (clamping of the decoded pixels exercised)."""
    W, H = 32, 24
    rng = np.random.default_rng(5)
    yy, xx = np.mgrid[0:H, 0:W]
    f = np.stack([rng.integers(0, 256, (H, W)), ((yy + xx) % 2) * 255, np.zeros((H, W)), np.full((H, W), 255),
                  ((xx // 1) % 2) * 255, ((yy % 2) * 255)]).astype(np.uint8)[None]
    enc = P.Encoder(W, H, 1, 8, 8, synth.phi_from_seed(2, 8, 64))
    fd = torch.from_numpy(f).cuda()
    for q in (np.ones((8, 8), np.int64), np.full((8, 8), 4096, np.int64), oracle.key_qsteps(0.7)):
        keys, coef = enc.key_codec(fd, q)
        torch.cuda.synchronize()
        ok, oc = oracle_keys(f, 1, q)
        assert np.array_equal(coef.cpu().numpy(), oc)
        assert np.array_equal(keys.cpu().numpy(), ok)


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_closed_loop_encode_parity(name):
    """Residuals against the GPU-decoded keys (Eq. 3), measured, vs the oracle's closed loop."""
    cfg = synth.CONFIGS[name].with_(T=min(synth.CONFIGS[name].T, 11))
    frames = synth.gen_video(cfg)
    qst = oracle.key_qsteps(1.0)
    M = cfg.Ms[0]
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    y_gpu, keys, _ = enc.encode_batch_closed_loop(torch.from_numpy(frames).cuda(), P.key_qsteps(1.0))
    torch.cuda.synchronize()
    y, S = oracle.encode_stream_closed_loop(frames[0], phi, cfg.G, cfg.B, qst)
    ok, st = oracle.check_tolerance(y_gpu.cpu().numpy(), y, S, REL)
    assert ok, st


def test_eq4_cancellation_on_gpu():
    """Phi = I (M = N = 64, B = 8): the GPU measurement of the closed-loop residual plus the
    GPU-decoded key reproduces every CS frame exactly, at every key quality (Eq. 4, P:93;
    SPEC.md:371)."""
    B = 8
    cfg = synth.CONFIGS["C1"].with_(T=10, G=5, B=B, S=1)
    frames = synth.gen_video(cfg)
    eye = np.eye(64).astype(np.float16).view(np.uint16)
    enc = P.Encoder(cfg.W, cfg.H, 5, B, 64, eye)
    fd = torch.from_numpy(frames).cuda()
    for qs in (0.2, 3.0, 30.0):
        y, keys, _ = enc.encode_batch_closed_loop(fd, P.key_qsteps(qs))
        torch.cuda.synchronize()
        y, keys = y.cpu().numpy().astype(np.float64), keys.cpu().numpy()
        order = [(gi, t) for gi, (k, cs) in enumerate(oracle.gop_partition(cfg.T, 5)) for t in cs]
        for i, (gi, t) in enumerate(order):
            rec = oracle.frame_unblocks(y[i], cfg.W, cfg.H, B) + keys[0, gi]
            assert np.array_equal(rec, frames[0, t].astype(np.float64)), (qs, i)


def test_raw_keys_reproduce_open_loop():
    """encode_batch_keys with the raw key frames as `keys` == encode_batch, bitwise."""
    cfg = synth.CONFIGS["C2"].with_(T=12)
    frames = synth.gen_video(cfg)
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, cfg.M, phi)
    fd = torch.from_numpy(frames).cuda()
    raw = fd[:, ::cfg.G].contiguous()
    a = enc.encode_batch(fd)
    b = enc.encode_batch_keys(fd, raw)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_key_codec_args():
    enc = P.Encoder(64, 32, 4, 16, 16, synth.phi_from_seed(1, 16, 256))
    fd = torch.zeros((1, 4, 32, 64), dtype=torch.uint8, device="cuda")
    keys = torch.empty((1, 1, 32, 64), dtype=torch.uint8, device="cuda")
    bad = np.zeros(64, np.int32)
    assert P.lib().cs_key_codec(enc._h, fd.data_ptr(), 1, 4, bad.ctypes.data, None, keys.data_ptr(), None) \
        == P.CS_ERR_ARG
    good = P.key_qsteps(1.0).ravel().copy()
    assert P.lib().cs_key_codec(enc._h, fd.data_ptr(), 1, 4, good.ctypes.data, None, keys.data_ptr() + 1, None) \
        == P.CS_ERR_ARG
    assert P.lib().cs_key_codec(enc._h, fd.data_ptr(), 1, 4, good.ctypes.data, None, keys.data_ptr(), None) == P.CS_OK
    torch.cuda.synchronize()
    assert int(keys.max()) == int(keys.min())          # all-zero frame decodes to a flat frame


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_chained_reference_parity(name):
    """f4 variant, Eq. 3 literal: every CS frame against the previous raw frame."""
    base = synth.CONFIGS[name]
    cfg = base.with_(T=min(base.T, 2 * base.G + 3), S=min(base.S, 2))
    frames = synth.gen_video(cfg)
    M = base.Ms[-1]
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    y_gpu = enc.encode_batch_chained(torch.from_numpy(frames).cuda())
    torch.cuda.synchronize()
    y_gpu = y_gpu.cpu().numpy()
    n_cs = oracle.cs_frame_count(cfg.T, cfg.G)
    for s in range(cfg.S):
        y, S = oracle.encode_stream_chained(frames[s], phi, cfg.G, cfg.B)
        ok, st = oracle.check_tolerance(y_gpu[s * n_cs:(s + 1) * n_cs], y, S, REL)
        assert ok, st


@pytest.mark.parametrize("name,M", [("C2", 32), ("C4", 128), ("C5", 4), ("C3", 64)])
def test_gop_phis_parity(name, M):
    """f4 variant, per-GOP seeds: GOP g measured with Phi(seed ^ g); the resident
    Phi is reloaded per unit.  Then n = 0 restores the single Phi (bitwise equal to a fresh run)."""
    base = synth.CONFIGS[name]
    cfg = base.with_(T=min(base.T, 3 * base.G + 2), S=min(base.S, 3))
    frames = synth.gen_video(cfg)
    n_g = -(-cfg.T // cfg.G)
    phis = [synth.phi_from_seed(synth.phi_seed() ^ g, M, cfg.B ** 2) for g in range(n_g)]
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phis[0])
    fd = torch.from_numpy(frames).cuda()
    ref = enc.encode_batch(fd).clone()
    enc.set_gop_phis(phis)
    y_gpu = enc.encode_batch(fd)
    torch.cuda.synchronize()
    yg = y_gpu.cpu().numpy()
    n_cs = oracle.cs_frame_count(cfg.T, cfg.G)
    for s in range(cfg.S):
        y, S = oracle.encode_stream_gop_phis(frames[s], phis, cfg.G, cfg.B)
        ok, st = oracle.check_tolerance(yg[s * n_cs:(s + 1) * n_cs], y, S, REL)
        assert ok, st
    enc.set_gop_phis(None)
    again = enc.encode_batch(fd)
    torch.cuda.synchronize()
    assert torch.equal(again, ref)


@pytest.mark.parametrize("M", [16, 64])
def test_gop_phis_slot_reuse(M):
    """Per-GOP Phi with the two resident Phi slots: 500 one-CS-frame GOPs of a one-tile frame over 148 CTAs,
    so every CTA switches matrices at every unit and reuses each slot several times (the slot's previous
    matrix must be released by the MMA's commit before it is overwritten)."""
    cfg = synth.CONFIGS["C1"].with_(W=64, H=32, G=2, T=1000, S=1, B=16)
    frames = synth.gen_video(cfg)
    phis = [synth.phi_from_seed(synth.phi_seed() ^ (7 * g + 1), M, 256) for g in range(5)]
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, 16, M, phis[0])
    enc.set_gop_phis(phis)
    y_gpu = enc.encode_batch(torch.from_numpy(frames).cuda()).cpu().numpy()
    y, S = oracle.encode_stream_gop_phis(frames[0], phis, cfg.G, 16)
    ok, st = oracle.check_tolerance(y_gpu, y, S, REL)
    assert ok, st
