"""CUDA-graph capture of the encode calls (no allocation inside encode calls,
so they are graph-capturable): capture once, replay on new frame contents, compare bitwise with
direct calls."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1311_1419_b200 as P  # noqa: E402


def test_encode_paths_in_a_cuda_graph():
    cfg = synth.CONFIGS["C2"].with_(T=17, S=2)
    frames_a = torch.from_numpy(synth.gen_video(cfg)).cuda()
    frames_b = torch.from_numpy(synth.gen_video(cfg, seed=synth.BASE_SEED + 99)).cuda()
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, cfg.M, phi)
    fd = frames_a.clone()
    y = torch.empty(enc.out_shape(cfg.S, cfg.T), dtype=torch.float32, device="cuda")
    codes = torch.empty(y.shape, dtype=torch.int16, device="cuda")
    scales = torch.empty(enc.q16_scale_shape(cfg.S, cfg.T, P.Encoder.Q16_ROW), dtype=torch.float32, device="cuda")
    x = torch.empty((y.shape[0], cfg.H, cfg.W), dtype=torch.float32, device="cuda")
    # warm-up outside the graph (lazy module loading), then capture
    enc.encode_batch(fd, y)
    enc.encode_batch_q16(fd, P.Encoder.Q16_ROW, codes, scales)
    enc.adjoint(y, x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        enc.encode_batch(fd, y)
        enc.encode_batch_q16(fd, P.Encoder.Q16_ROW, codes, scales)
        enc.adjoint(y, x)
    for src in (frames_b, frames_a):
        fd.copy_(src)
        g.replay()
        torch.cuda.synchronize()
        y_ref = enc.encode_batch(src)
        c_ref, s_ref = enc.encode_batch_q16(src, P.Encoder.Q16_ROW)
        x_ref = enc.adjoint(y_ref)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref) and torch.equal(codes, c_ref) and torch.equal(scales, s_ref)
        assert torch.equal(x, x_ref)
