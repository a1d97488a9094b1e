"""GPU parity of the paper-faithful frame-level measurement (Eq. 1).

Acceptance (R24, derived from the arithmetic): products A_ij r_j are exact in fp32
(fp16 x integer <= 255), the tensor core accumulates n/16 partial sums of 16 products in fp32, and
split-K adds at most 16 partials, so |y_gpu - y| <= (n/16 + 16) * 2^-23 * sum_j |A_ij r_j|.
A layout bug (transposed A, wrong pixel order, wrong key) gives O(1) relative errors.
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


def rel_bound(n):
    return (n / 16 + 16) * 2.0 ** -23


def check(y_gpu, y, S, n):
    assert y_gpu.shape == y.shape
    err = np.abs(y_gpu.astype(np.float64) - y)
    bad = err > rel_bound(n) * S
    assert not bad.any(), (int(bad.sum()), float(np.max(err / np.maximum(S, 1e-300))))
    assert np.all(y_gpu[S == 0] == 0)
    return float(np.max(err / np.where(S > 0, S, 1.0)))


@pytest.mark.parametrize("W,H,G,T,S,m", [(32, 16, 3, 7, 2, 37), (48, 20, 2, 9, 1, 130), (64, 8, 5, 23, 3, 256),
                                          (16, 16, 8, 17, 2, 5), (176, 144, 5, 10, 2, 507),
                                          (32, 16, 4, 8, 5, 300), (96, 32, 3, 300, 3, 64)])
def test_frame_parity(W, H, G, T, S, m):
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
    frames = synth.gen_video(cfg)
    A = synth.phi_from_seed(synth.phi_seed() + m, m, W * H)
    fe = P.FrameEncoder(W, H, G, m, A)
    y_gpu = fe.encode_batch(torch.from_numpy(frames).cuda())
    torch.cuda.synchronize()
    y_gpu = y_gpu.cpu().numpy()
    n_cs = oracle.cs_frame_count(T, G)
    for s in range(S):
        y, Sc = oracle.measure_frame(frames[s], A, G)
        check(y_gpu[s * n_cs:(s + 1) * n_cs], y, Sc, W * H)


def test_frame_identity_and_unit_columns():
    """A = I (m = n): y is the residual exactly (one nonzero product per row); a unit residual at
    pixel j gives exactly v * A[:, j] (localises pixel-order / permutation bugs)."""
    W, H, G = 32, 8, 2
    n = W * H
    eye = np.eye(n).astype(np.float16).view(np.uint16)
    rng = np.random.default_rng(2)
    frames = rng.integers(0, 256, (1, 6, H, W), dtype=np.uint8)
    fe = P.FrameEncoder(W, H, G, n, eye)
    y = fe.encode_batch(torch.from_numpy(frames).cuda()).cpu().numpy()
    for i, t in enumerate([1, 3, 5]):
        assert np.array_equal(y[i], (frames[0, t].astype(np.float32) - frames[0, t - 1]).ravel())
    A = synth.phi_from_seed(3, 40, n)
    Av = oracle.phi_values(A).astype(np.float32)
    fe2 = P.FrameEncoder(W, H, 2, 40, A)
    f = np.full((1, 2 * n, H, W), 100, np.uint8)
    for j in range(n):
        f[0, 2 * j + 1].flat[j] = 180
    y = fe2.encode_batch(torch.from_numpy(f).cuda()).cpu().numpy()
    for j in range(n):
        assert np.array_equal(y[j], 80 * Av[:, j]), j


def test_frame_block_structured_matches_block_path():
    """A assembled from Phi block by block: the frame-level GPU path and the block GPU path compute
    the same measurements (different summation orders: within both tolerances)."""
    B, M = 16, 8
    W, H, G, T = 64, 40, 4, 9
    phi = synth.phi_from_seed(4, M, B * B)
    A = oracle.block_matrix_as_frame(phi, W, H, B)
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=1)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    yf = P.FrameEncoder(W, H, G, A.shape[0], A).encode_batch(fd).cpu().numpy()
    yb = P.Encoder(W, H, G, B, M, phi).encode_batch(fd).cpu().numpy()
    y, S = oracle.measure_frame(frames[0], A, G)
    check(yf, y, S, W * H)
    assert np.allclose(yf, yb.reshape(yb.shape[0], -1), rtol=0, atol=float(np.max(S)) * 1e-5)


def test_frame_paper_config_full_batch():
    """The paper's configuration (QCIF, GOP = key + 4 CS frames, CR 50 -> m = 507) in the
    bench launch shape (64 streams: one full tile per SM, no split-K); every CS frame of 3 streams
    against the oracle."""
    W, H, G, m, T, S = 176, 144, 5, 507, 40, 64
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
    frames = synth.gen_video(cfg)
    A = synth.phi_from_seed(synth.phi_seed(), m, W * H)
    fe = P.FrameEncoder(W, H, G, m, A)
    y_gpu = fe.encode_batch(torch.from_numpy(frames).cuda()).cpu().numpy()
    n_cs = oracle.cs_frame_count(T, G)
    for s in (0, 31, 63):
        y, Sc = oracle.measure_frame(frames[s], A, G)
        check(y_gpu[s * n_cs:(s + 1) * n_cs], y, Sc, W * H)


def test_frame_bench_batch_parity():
    """The bench's exact launch (64 streams x 400 QCIF frames, m = 507; bench.py --op frame, R25):
    three streams' CS frames (320 each) against the oracle.  Prints the observed max |dy|/S next to
    the R24 worst-case bound (accumulation-order guarantee) and the north star's 1e-5."""
    W, H, G, m, T, S = 176, 144, 5, 507, 400, 64
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
    frames = synth.gen_video(cfg)
    A = synth.phi_from_seed(synth.phi_seed(), m, W * H)
    fe = P.FrameEncoder(W, H, G, m, A)
    y_gpu = fe.encode_batch(torch.from_numpy(frames).cuda()).cpu().numpy()
    n_cs = oracle.cs_frame_count(T, G)
    worst = 0.0
    for s in (0, 31, 63):
        y, Sc = oracle.measure_frame(frames[s], A, G)
        worst = max(worst, check(y_gpu[s * n_cs:(s + 1) * n_cs], y, Sc, W * H))
    print(f"f2 bench batch: observed max |dy|/S = {worst:.3e}; R24 bound {rel_bound(W * H):.3e}; north star 1e-5")
    assert worst < rel_bound(W * H)


def test_frame_args():
    A = synth.phi_from_seed(1, 4, 32 * 16)
    with pytest.raises(P.CSError):
        P.FrameEncoder(24, 16, 2, 4, synth.phi_from_seed(1, 4, 24 * 16))      # W % 16
    bad = A.copy()
    bad[0, 0] = 0x7C00                                                        # +inf
    with pytest.raises(P.CSError):
        P.FrameEncoder(32, 16, 2, 4, bad)
    fe = P.FrameEncoder(32, 16, 1, 4, A)                                      # G = 1: no CS frames
    y = fe.encode_batch(torch.zeros((2, 3, 16, 32), dtype=torch.uint8, device="cuda"))
    assert y.numel() == 0


def test_frame_windows_and_split_k():
    """K4 gives the oracle's measurements with windows within and across streams and split-K."""
    for (W, H, G, T, S, m) in [(176, 144, 5, 40, 4, 507), (64, 16, 3, 8, 3, 100), (48, 32, 4, 11, 2, 300)]:
        cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
        frames = synth.gen_video(cfg)
        A = synth.phi_from_seed(11 + m, m, W * H)
        y_gpu = P.FrameEncoder(W, H, G, m, A).encode_batch(torch.from_numpy(frames).cuda()).cpu().numpy()
        n_cs = oracle.cs_frame_count(T, G)
        for s in range(S):
            y, Sc = oracle.measure_frame(frames[s], A, G)
            check(y_gpu[s * n_cs:(s + 1) * n_cs], y, Sc, W * H)
