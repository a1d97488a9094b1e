"""Programmatic dependent launch of the encode kernels (include/cs_encoder.h, cs_encoder_set_stable_inputs):
kernels queued back to back overlap; with stable inputs the loads of a launch start before the previous
kernel has completed and only its stores wait.  Checks: results are bitwise those of isolated launches,
write-after-write order on a shared output buffer is kept, and a launch whose input IS produced by the
preceding kernel (default setting) sees that kernel's output."""
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1311_1419_b200 as P  # noqa: E402


def _encoders(cfg, Ms, stable):
    encs = []
    for M in Ms:
        e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed() + M, M, cfg.B ** 2))
        e.set_stable_inputs(frames=stable)
        encs.append(e)
    return encs


@pytest.mark.parametrize("wl,T", [("C4", 27), ("C3", 50), ("C2", 41)])
def test_back_to_back_launches_match_isolated_ones(wl, T):
    cfg = synth.CONFIGS[wl].with_(T=T, S=1)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    Ms = (16, 64) if cfg.B == 16 else (cfg.M, 32)
    ref = []
    for e in _encoders(cfg, Ms, False):
        ref.append(e.encode_batch(fd).clone())
        torch.cuda.synchronize()
    y, S = oracle.encode(frames, synth.phi_from_seed(synth.phi_seed() + Ms[0], Ms[0], cfg.B ** 2), cfg.G, cfg.B)
    ok, st = oracle.check_tolerance(ref[0].cpu().numpy(), y, S)
    assert ok, st
    for stable in (False, True):
        encs = _encoders(cfg, Ms, stable)
        outs = [torch.empty_like(r) for r in ref]
        for _ in range(6):                      # 12 kernels queued without a host sync in between
            for e, o in zip(encs, outs):
                e.encode_batch(fd, o)
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r), stable


def test_shared_output_buffer_keeps_launch_order():
    """Two encoders (same shape, different Phi) write the SAME output buffer alternately: after the queue
    drains it holds the last writer's measurements, whichever launch overlapped which."""
    cfg = synth.CONFIGS["C4"].with_(T=19, S=1)
    fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
    a, b = _encoders(cfg, (32, 32), True)
    b2 = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, 32, synth.phi_from_seed(synth.phi_seed() + 777, 32, cfg.B ** 2))
    b2.set_stable_inputs(frames=True)
    ra, rb = a.encode_batch(fd).clone(), b2.encode_batch(fd).clone()
    torch.cuda.synchronize()
    assert not torch.equal(ra, rb)
    out = torch.empty_like(ra)
    for _ in range(5):
        a.encode_batch(fd, out)
        b2.encode_batch(fd, out)
    torch.cuda.synchronize()
    assert torch.equal(out, rb)
    a.encode_batch(fd, out)
    torch.cuda.synchronize()
    assert torch.equal(out, ra)


def test_input_written_by_the_preceding_kernel_default_setting():
    """Default (inputs not promised stable): frames produced by the kernel right before the encode are
    seen complete (the encode kernel waits for it before its first load)."""
    cfg = synth.CONFIGS["C4"].with_(T=17, S=1)
    frames = synth.gen_video(cfg)
    src = torch.from_numpy(frames).cuda()
    (e,) = _encoders(cfg, (32,), False)
    ref = e.encode_batch(src).clone()
    fd = torch.zeros_like(src)
    out = torch.empty_like(ref)
    for _ in range(4):
        fd.zero_()                # a kernel
        fd.add_(src)              # the kernel right before the encode writes its input
        e.encode_batch(fd, out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_q16_two_pass_and_store_paths_back_to_back_with_stable_inputs():
    cfg = synth.CONFIGS["C4"].with_(T=19, S=1)
    fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
    for M in (16, 64):            # store-and-requantise path / two measuring passes
        (e,) = _encoders(cfg, (M,), False)
        c0, s0 = e.encode_batch_q16(fd, P.Encoder.Q16_FRAME)
        r0, t0 = e.encode_batch_q16(fd, P.Encoder.Q16_ROW)
        torch.cuda.synchronize()
        (e2,) = _encoders(cfg, (M,), True)
        for _ in range(4):
            c1, s1 = e2.encode_batch_q16(fd, P.Encoder.Q16_FRAME)
            r1, t1 = e2.encode_batch_q16(fd, P.Encoder.Q16_ROW)
        torch.cuda.synchronize()
        assert torch.equal(c0, c1) and torch.equal(s0, s1) and torch.equal(r0, r1) and torch.equal(t0, t1), M


def test_adjoint_back_to_back_with_stable_inputs():
    cfg = synth.CONFIGS["C4"].with_(T=19, S=1)
    fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
    (e,) = _encoders(cfg, (32,), False)
    y = e.encode_batch(fd)
    x0 = e.adjoint(y).clone()
    torch.cuda.synchronize()
    e.set_stable_inputs(frames=True, measurements=True)
    x = torch.empty_like(x0)
    for _ in range(6):
        e.adjoint(y, x)
    torch.cuda.synchronize()
    assert torch.equal(x, x0)
    # frames promised stable, measurements not: y produced by the kernel right before the adjoint
    e.set_stable_inputs(frames=True, measurements=False)
    y2 = torch.empty_like(y)
    for _ in range(3):
        e.encode_batch(fd, y2)
        e.adjoint(y2, x)
    torch.cuda.synchronize()
    assert torch.equal(x, x0)


def test_stable_inputs_inside_a_cuda_graph():
    """The overlapping launches keep their order when captured into a CUDA graph (programmatic edges)."""
    cfg = synth.CONFIGS["C4"].with_(T=19, S=1)
    fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
    encs = _encoders(cfg, (16, 64), True)
    ref = [e.encode_batch(fd).clone() for e in encs]
    torch.cuda.synchronize()
    outs = [torch.zeros_like(r) for r in ref]
    shared = torch.zeros_like(ref[1])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(3):
            for e, o in zip(encs, outs):
                e.encode_batch(fd, o)
        encs[1].encode_batch(fd, shared)
    for _ in range(3):
        for o in outs:
            o.zero_()
        shared.zero_()
        g.replay()
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)
        assert torch.equal(shared, ref[1])
