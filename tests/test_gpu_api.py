"""The binding's argument checks and the C ABI's device / plan rules, and the
host-buffer 16-bit path (f1 e2e): every case either raises before anything is launched or gives
exactly the device-path result."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1311_1419_b200 as P  # noqa: E402


def small_encoder(W=64, H=40, G=4, B=8, M=8):
    return P.Encoder(W, H, G, B, M, synth.phi_from_seed(3, M, B * B))


def test_wrappers_reject_bad_buffers():
    enc = small_encoder()
    good = torch.zeros((1, 5, 40, 64), dtype=torch.uint8, device="cuda")
    bad_shapes = [torch.zeros((1, 5, 40, 48), dtype=torch.uint8, device="cuda"),     # wrong W
                  torch.zeros((5, 40, 64), dtype=torch.uint8, device="cuda"),        # not 4-D
                  torch.zeros((1, 5, 40, 128), dtype=torch.uint8, device="cuda")[..., ::2],   # non-contiguous
                  torch.zeros((1, 5, 40, 64), dtype=torch.int16, device="cuda"),     # dtype
                  torch.zeros((1, 5, 40, 64), dtype=torch.uint8)]                    # host
    calls = [lambda f: enc.encode_batch(f), lambda f: enc.encode_batch_q16(f), lambda f: enc.encode_batch_chained(f),
             lambda f: enc.key_codec(f, P.key_qsteps(1.0)), lambda f: enc.autotune(f),
             lambda f: enc.encode_batch_gops(f, 0, 1, torch.empty(10**5, device="cuda"))]
    for bad in bad_shapes:
        for call in calls:
            with pytest.raises(ValueError):
                call(bad)
    small = torch.empty(10, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        enc.encode_batch(good, small)                      # undersized out
    with pytest.raises(ValueError):
        enc.encode_batch_gops(good, 0, 2, small)
    with pytest.raises(ValueError):
        enc.encode_batch_q16(good, codes=torch.empty(10, dtype=torch.int16, device="cuda"))
    with pytest.raises(ValueError):
        enc.encode_batch_keys(good, torch.zeros((1, 1, 40, 64), dtype=torch.uint8, device="cuda"))   # 2 GOPs
    with pytest.raises(ValueError):
        enc.adjoint(torch.zeros(7, dtype=torch.float32, device="cuda"))
    host = np.zeros((1, 5, 40, 128), dtype=np.uint8)[..., ::2]
    with pytest.raises(ValueError):
        enc.encode_batch_host(host)                        # non-contiguous host frames
    with pytest.raises(ValueError):
        enc.encode_batch_host(np.zeros((1, 5, 40, 64), np.uint8), np.zeros(3, np.float32))
    torch.cuda.synchronize()   # nothing bad was launched


def test_adjoint_refuses_per_gop_phis():
    """cs_adjoint back-projects with the create-time Phi: with per-GOP matrices set it must refuse
    (CS_ERR_UNSUPPORTED) instead of silently using the wrong matrix; restoring the single Phi
    re-enables it."""
    enc = small_encoder()
    y = torch.zeros((2, enc.nblk, enc.M), dtype=torch.float32, device="cuda")
    enc.adjoint(y)
    enc.set_gop_phis([synth.phi_from_seed(5 + g, enc.M, 64) for g in range(2)])
    with pytest.raises(P.CSError) as ei:
        enc.adjoint(y)
    assert ei.value.code == P.CS_ERR_UNSUPPORTED
    enc.set_gop_phis(None)
    enc.adjoint(y)
    torch.cuda.synchronize()


def test_q16_row_uses_a_qualifying_plan():
    """A current plan with tiles taller than 40 block rows no longer makes CS_Q16_ROW fail: the call
    runs the best qualifying candidate, bit-identical to running that plan explicitly."""
    W, H, G, B, M = 64, 720, 4, 8, 8      # nbx = 8: tiles of up to 128 block rows exist
    enc = P.Encoder(W, H, G, B, M, synth.phi_from_seed(11, M, B * B))
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, T=6, G=G, B=B, Ms=(M,), S=1)
    fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
    tall = [i for i in range(enc.num_candidates()) if enc.set_candidate(i)["tile_block_rows"] > 40]
    short = [i for i in range(enc.num_candidates()) if enc.set_candidate(i)["tile_block_rows"] <= 40]
    assert tall and short
    enc.set_candidate(short[0])
    ref_c, ref_s = enc.encode_batch_q16(fd, P.Encoder.Q16_ROW)
    enc.set_candidate(tall[0])
    c, s = enc.encode_batch_q16(fd, P.Encoder.Q16_ROW)
    torch.cuda.synchronize()
    assert torch.equal(c, ref_c) and torch.equal(s, ref_s)


@pytest.mark.parametrize("S,T", [(1, 37), (3, 19)])
@pytest.mark.parametrize("gran", [0, 1])
def test_host_q16_equals_device_q16(S, T, gran):
    """cs_encode_batch_host(_multi)_q16 (groups of GOPs for one stream, of streams otherwise) gives the
    device call's codes and scales bit for bit."""
    cfg = synth.CONFIGS["C2"].with_(T=T, S=S)
    frames = synth.gen_video(cfg)
    encs = [P.Encoder(cfg.W, cfg.H, cfg.G, 16, M, synth.phi_from_seed(7 + M, M, 256)) for M in (16, 64)]
    outs = P.encode_batch_host_multi_q16(encs, frames, gran)
    c1, s1 = encs[0].encode_batch_host_q16(frames, gran)
    fd = torch.from_numpy(frames).cuda()
    for e, (c, sc) in zip(encs, outs):
        rc, rs = e.encode_batch_q16(fd, gran)
        torch.cuda.synchronize()
        assert np.array_equal(c, rc.cpu().numpy()) and np.array_equal(sc, rs.cpu().numpy())
    assert np.array_equal(c1, outs[0][0]) and np.array_equal(s1, outs[0][1])


def test_device_mismatch_is_refused():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with torch.cuda.device(0):
        enc = small_encoder()
    f1 = torch.zeros((1, 5, 40, 64), dtype=torch.uint8, device="cuda:1")
    with pytest.raises(ValueError):
        enc.encode_batch(f1)
    f0 = torch.zeros((1, 5, 40, 64), dtype=torch.uint8, device="cuda:0")
    out = torch.empty(enc.out_shape(1, 5), dtype=torch.float32, device="cuda:0")
    with torch.cuda.device(1):   # raw ABI call with the wrong current device: CS_ERR_ARG, nothing launched
        rc = P.lib().cs_encode_batch(enc._h, f0.data_ptr(), 1, 5, out.data_ptr(), None)
    assert rc == P.CS_ERR_ARG
    enc.encode_batch(f0)   # the binding switches to the encoder's device itself
    torch.cuda.synchronize()
