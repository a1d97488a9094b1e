"""GPU parity of the block back-projection x0 = Phi^T y.

Acceptance (the form BASELINE.json:5 gives for y, applied to the adjoint): per pixel
|x_gpu - x| <= 1e-5 * sum_m |Phi_mj| |y_m| against the fp64 oracle on the same fp32 input y.  The
kernel splits y into two tf32 terms (Phi is exact in tf32) and accumulates in fp32, so the expected
error is ~1e-7 of that scale; a layout bug (wrong block, wrong in-block index, transposed Phi,
wrong K chunk) produces O(1) errors.
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


def check(x_gpu, meas, phi, W, H, B):
    x = oracle.adjoint(meas, phi, W, H, B)
    S = oracle.adjoint_tolerance_scale(meas, phi, W, H, B)
    assert x_gpu.shape == x.shape
    err = np.abs(x_gpu.astype(np.float64) - x)
    bad = err > REL * S
    assert not bad.any(), (int(bad.sum()), float(np.max(err / np.maximum(S, 1e-300))))
    assert np.all(x_gpu[S == 0] == 0)
    return float(np.max(err / np.where(S > 0, S, 1.0)))


def run(enc, meas_np):
    x = enc.adjoint(torch.from_numpy(np.ascontiguousarray(meas_np, dtype=np.float32)).cuda())
    torch.cuda.synchronize()
    return x.cpu().numpy()


CASES = [
    # W, H, B, M, n_frames   (Kc = 8 / 16 / 32, K chunks, ragged H, W % 32 == 16, two parts per row)
    (176, 144, 16, 64, 3),
    (64, 40, 8, 4, 5),
    (96, 24, 8, 12, 2),
    (80, 33, 16, 16, 2),
    (112, 50, 16, 24, 2),
    (64, 48, 16, 40, 2),
    (352, 288, 16, 128, 2),
    (48, 70, 32, 64, 2),
    (32, 32, 16, 256, 2),
    (1280, 24, 8, 16, 3),       # nbx = 160 > 128: two 80-block parts per block row
    (2096, 16, 16, 32, 1),      # nbx = 131: parts of 66 / 65 blocks
    # nbx % 32 == 0: flat 128-block tiles across block rows
    (512, 40, 16, 32, 3),       # nbx = 32, ragged H, one partial tile per frame
    (2048, 16, 32, 64, 2),      # nbx = 64, B = 32 (4 output chunks)
    (1024, 72, 8, 8, 2),        # nbx = 128, 9 whole tiles per frame
]


@pytest.mark.parametrize("case", CASES, ids=[f"W{c[0]}H{c[1]}B{c[2]}M{c[3]}" for c in CASES])
def test_adjoint_parity_random(case):
    W, H, B, M, n = case
    phi = synth.phi_from_seed(synth.phi_seed() + M + B, M, B * B)
    enc = P.Encoder(W, H, 2, B, M, phi)
    rng = np.random.default_rng(M * 7 + B)
    meas = (rng.normal(size=(n, enc.nblk, M)) * 10.0 ** rng.uniform(-2, 4, size=(n, enc.nblk, 1)))
    meas[:, ::7] = 0.0                                         # some all-zero blocks
    meas = meas.astype(np.float32)
    rel = check(run(enc, meas), meas.astype(np.float64), phi, W, H, B)
    assert rel < 1e-6, rel


@pytest.mark.parametrize("B,M", [(8, 4), (16, 64), (32, 64)])
def test_adjoint_unit_vectors(B, M):
    """v = e_(frame, block, m) -> row m of Phi laid into that block, exactly (one product of
    exact values); every m, blocks in every position of the warp / tile, including the last."""
    W, H = {8: (48, 20), 16: (48, 40), 32: (80, 40)}[B]   # ragged bottom row; B = 32: half last column
    phi = synth.phi_from_seed(3, M, B * B)
    phiv = oracle.phi_values(phi)
    enc = P.Encoder(W, H, 2, B, M, phi)
    nblk = enc.nblk
    meas = np.zeros((M, nblk, M), np.float32)
    blocks = [(m * 5 + 3) % nblk for m in range(M)]
    blocks[-1] = nblk - 1
    for m in range(M):
        meas[m, blocks[m], m] = 1.0
    x = run(enc, meas)
    for m in range(M):
        want = np.zeros((enc.nby * B, enc.nbx * B))
        by, bx = divmod(blocks[m], enc.nbx)
        want[by * B:(by + 1) * B, bx * B:(bx + 1) * B] = phiv[m].reshape(B, B)
        assert np.array_equal(x[m], want[:H, :W].astype(np.float32)), m


def test_adjoint_identity_phi():
    """Phi = I (M = N = 256): x is the unblocked y, up to the lo term's tf32 rounding."""
    B, M = 16, 256
    eye = np.eye(M).astype(np.float16).view(np.uint16)
    W, H = 48, 40
    enc = P.Encoder(W, H, 2, B, M, eye)
    meas = np.random.default_rng(1).normal(size=(2, enc.nblk, M)).astype(np.float32)
    x = run(enc, meas)
    for k in range(2):
        want = oracle.frame_unblocks(meas[k].astype(np.float64), W, H, B)
        assert np.all(np.abs(x[k] - want) <= 2.0 ** -20 * np.abs(want))


def test_adjoint_of_encoder_output_and_inner_product():
    """x0 = Phi^T y of the GPU's own measurements (the decoder's start point), checked against
    the oracle, and the adjoint identity <Phi r, v> = <r, Phi^T v> through both GPU kernels."""
    cfg = synth.CONFIGS["C2"].with_(T=9)
    frames = synth.gen_video(cfg)
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, cfg.M, phi)
    fd = torch.from_numpy(frames).cuda()
    y = enc.encode_batch(fd)
    x = enc.adjoint(y)
    torch.cuda.synchronize()
    y_np = y.cpu().numpy()
    check(x.cpu().numpy(), y_np.astype(np.float64), phi, cfg.W, cfg.H, cfg.B)
    # <y, v> with v = y (any v works) equals <R, Phi^T v>: R = residual frames of the CS frames
    order = [(k, t) for k, cs in oracle.gop_partition(cfg.T, cfg.G) for t in cs]
    xv = x.cpu().numpy().astype(np.float64)
    for i, (k, t) in enumerate(order):
        R = frames[0, t].astype(np.float64) - frames[0, k].astype(np.float64)
        lhs = float(np.sum(y_np[i].astype(np.float64) ** 2))
        rhs = float(np.sum(R * xv[i]))
        assert abs(lhs - rhs) <= 1e-4 * lhs, (i, lhs, rhs)


@pytest.mark.parametrize("name,Ms", [("C4", (16, 128)), ("C5", (4,))])
def test_adjoint_full_size(name, Ms):
    """Full-size frames: the adjoint of all CS frames of a reduced-T batch; every pixel of three
    frames against the oracle."""
    cfg = synth.CONFIGS[name].with_(T=9, S=2)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    for M in Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        y = enc.encode_batch(fd)
        x = enc.adjoint(y)
        torch.cuda.synchronize()
        y_np, x_np = y.cpu().numpy(), x.cpu().numpy()
        n = y_np.shape[0]
        for i in sorted({0, n // 2, n - 1}):
            check(x_np[i:i + 1], y_np[i:i + 1].astype(np.float64), phi, cfg.W, cfg.H, cfg.B)


def test_adjoint_args():
    phi = synth.phi_from_seed(1, 16, 256)
    enc = P.Encoder(64, 32, 4, 16, 16, phi)
    x = torch.empty((1, 32, 64), dtype=torch.float32, device="cuda")
    y = torch.zeros((1, 8, 16), dtype=torch.float32, device="cuda")
    assert P.lib().cs_adjoint(enc._h, y.data_ptr(), 0, x.data_ptr(), None) == P.CS_OK
    assert P.lib().cs_adjoint(enc._h, y.data_ptr() + 4, 1, x.data_ptr(), None) == P.CS_ERR_ARG
    assert P.lib().cs_adjoint(enc._h, None, 1, x.data_ptr(), None) == P.CS_ERR_ARG
    assert P.lib().cs_adjoint(enc._h, y.data_ptr(), -1, x.data_ptr(), None) == P.CS_ERR_ARG
    enc6 = P.Encoder(64, 32, 4, 16, 6, synth.phi_from_seed(1, 6, 256))
    y6 = torch.zeros((1, 8, 6), dtype=torch.float32, device="cuda")
    with pytest.raises(P.CSError) as ei:
        enc6.adjoint(y6)
    assert ei.value.code == P.CS_ERR_UNSUPPORTED
