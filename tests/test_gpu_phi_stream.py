"""Plans that stream Phi's K-slices through the stages (phi_stream = 1) give the same bits as the
resident-Phi plans: plain encode, per-GOP matrices (S:174 variant) and the q16 row epilogue."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_1311_1419_b200 as P  # noqa: E402


def stream_candidates(enc):
    out = []
    for i in range(enc.num_candidates()):
        if enc.set_candidate(i)["phi_stream"]:
            out.append(i)
    return out


@pytest.mark.parametrize("name,M,T", [("C3", 64, 17), ("C1", 64, 4), ("C2", 32, 9)])
def test_phi_stream_plans_bitwise(name, M, T):
    cfg = synth.CONFIGS[name].with_(T=T, S=1)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    cands = stream_candidates(enc)
    assert cands, "no phi-streaming plan for this geometry"
    ref_i = next(i for i in range(enc.num_candidates()) if not enc.set_candidate(i)["phi_stream"])
    enc.set_candidate(ref_i)
    ref = enc.encode_batch(fd).clone()
    y, S = oracle.encode(frames, phi, cfg.G, cfg.B)
    ok, stats = oracle.check_tolerance(ref.cpu().numpy(), y, S)
    assert ok, stats
    for i in cands[:6]:
        plan = enc.set_candidate(i)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), plan


def test_phi_stream_gop_phis_and_q16():
    cfg = synth.CONFIGS["C3"].with_(T=40, S=1)     # 3 GOPs (16, 16, 8 frames): 3 matrices
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    M = 64
    phis = [synth.phi_from_seed(synth.phi_seed() ^ g, M, cfg.B ** 2) for g in range(3)]
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phis[0])
    cands = stream_candidates(enc)
    assert cands
    ref_i = next(i for i in range(enc.num_candidates()) if not enc.set_candidate(i)["phi_stream"])
    enc.set_gop_phis(phis)
    enc.set_candidate(ref_i)
    ref = enc.encode_batch(fd).clone()
    # per-GOP oracle: GOP g measured with phis[g]
    n_cs_g = cfg.G - 1
    got = ref.cpu().numpy()
    for g in range(3):
        sub = frames[:, g * cfg.G:(g + 1) * cfg.G]
        y, S = oracle.encode(sub, phis[g], cfg.G, cfg.B)
        ok, stats = oracle.check_tolerance(got[g * n_cs_g:g * n_cs_g + y.shape[0]], y, S)
        assert ok, (g, stats)
    enc.set_candidate(cands[0])
    assert torch.equal(enc.encode_batch(fd), ref)
    enc.set_gop_phis(None)
    # q16 row epilogue on a streaming plan == on a resident plan
    enc.set_candidate(ref_i)
    c0, s0 = enc.encode_batch_q16(fd, P.Encoder.Q16_ROW)
    enc.set_candidate(cands[0])
    c1, s1 = enc.encode_batch_q16(fd, P.Encoder.Q16_ROW)
    torch.cuda.synchronize()
    assert torch.equal(c0, c1) and torch.equal(s0, s1)
    assert np.isfinite(s0.cpu().numpy()).all()


@pytest.mark.parametrize("W,H,T,G,M", [(640, 480, 5, 4, 96), (640, 100, 6, 3, 128), (160, 72, 7, 4, 256),
                                       (96, 40, 3, 3, 200)])
def test_b32_large_m(W, H, T, G, M):
    """B = 32 with M up to 256 (M <= min(N, 256)): Phi (up to 512 KB) no longer fits
    shared memory, so every plan streams its K-slices; parity with the oracle for fp32 (every candidate
    plan bitwise equal), the 16-bit row / frame codes and the adjoint."""
    cfg = synth.CONFIGS["C3"].with_(W=W, H=H, T=T, G=G, Ms=(M,), S=2)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed() + M, M, 1024)
    enc = P.Encoder(W, H, G, 32, M, phi)
    assert enc.plan()["phi_stream"] == 1
    out = enc.encode_batch(fd)
    torch.cuda.synchronize()
    y, S = oracle.encode(frames, phi, G, 32)
    ok, stats = oracle.check_tolerance(out.cpu().numpy(), y, S)
    assert ok, stats
    for i in range(min(6, enc.num_candidates())):
        enc.set_candidate(i)
        assert torch.equal(enc.encode_batch(fd), out), enc.plan()
    enc.set_candidate(0)
    for gran in (P.Encoder.Q16_FRAME, P.Encoder.Q16_ROW):
        codes, scales = enc.encode_batch_q16(fd, gran)
        torch.cuda.synchronize()
        c = codes.cpu().numpy().astype(np.float64)
        sc = scales.cpu().numpy().astype(np.float64)
        sc = np.repeat(sc, enc.nbx, axis=1)[:, :, None] if gran == P.Encoder.Q16_ROW else sc[:, None, None]
        assert np.all(np.abs(c * sc - y) <= sc * (0.5 + 2.0 ** -21) + 1e-5 * S + 2.0 ** -22 * np.abs(y))
    if M % 4 == 0:
        x = enc.adjoint(out)
        torch.cuda.synchronize()
        yv = out.cpu().numpy().astype(np.float64)
        xo = oracle.adjoint(yv, phi, W, H, 32)
        Sx = oracle.adjoint_tolerance_scale(yv, phi, W, H, 32)
        assert np.all(np.abs(x.cpu().numpy() - xo) <= 1e-5 * Sx)
