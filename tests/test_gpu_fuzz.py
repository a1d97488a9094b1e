"""Seeded shape fuzzing of the device paths against the oracle: random frame sizes (any H, W a
multiple of 16), block sizes, measurement counts (any M allowed by the Phi SMEM limit), GOP sizes
(including G = 1 and short final GOPs), frame counts and stream counts.  Each case checks the fp32
encode (north-star tolerance), the per-frame q16 codes (within 1 of the oracle's quantiser) and, when
M % 4 == 0, the adjoint."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1311_1419_b200 as P  # noqa: E402


def random_case(rng):
    B = int(rng.choice([8, 16, 32]))
    N = B * B
    m_max = min(N, 256)
    while True:
        M = int(rng.integers(1, m_max + 1))
        mpad = max(16, -(-M // 16) * 16)
        if mpad * N * 2 <= 160 * 1024:
            break
    W = 16 * int(rng.integers(1, 25))
    H = int(rng.integers(1, 200))
    G = int(rng.integers(1, 12))
    T = int(rng.integers(1, 3 * G + 3))
    S = int(rng.integers(1, 4))
    return W, H, T, G, B, M, S


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_encode_q16_adjoint(seed):
    rng = np.random.default_rng(1000 + seed)
    W, H, T, G, B, M, S = random_case(rng)
    frames = rng.integers(0, 256, size=(S, T, H, W), dtype=np.uint8)
    if rng.random() < 0.5:                       # static background + moving patch: sparse residuals
        frames[:] = frames[:, :1]
        frames[:, :, : max(1, H // 3), : max(16, W // 4)] = rng.integers(0, 256, size=(S, T, max(1, H // 3), max(16, W // 4)))
    phi = synth.phi_from_seed(seed, M, B * B)
    enc = P.Encoder(W, H, G, B, M, phi)
    fd = torch.from_numpy(frames).cuda()
    y_gpu = enc.encode_batch(fd)
    torch.cuda.synchronize()
    y, Sc = oracle.encode(frames, phi, G, B)
    assert y_gpu.shape == y.shape, (W, H, T, G, B, M, S)
    ok, st = oracle.check_tolerance(y_gpu.cpu().numpy(), y, Sc)
    assert ok, ((W, H, T, G, B, M, S), st)
    if y.shape[0] == 0:
        return
    codes, scales = enc.encode_batch_q16(fd)
    torch.cuda.synchronize()
    oc, _ = oracle.quantize_frames(y)
    assert np.abs(codes.cpu().numpy().astype(np.int64) - oc).max() <= 1, (W, H, T, G, B, M, S)
    if M % 4 == 0:
        x = enc.adjoint(y_gpu)
        torch.cuda.synchronize()
        yv = y_gpu.cpu().numpy().astype(np.float64)
        xo = oracle.adjoint(yv, phi, W, H, B)
        Sx = oracle.adjoint_tolerance_scale(yv, phi, W, H, B)
        assert np.all(np.abs(x.cpu().numpy() - xo) <= 1e-5 * Sx), (W, H, T, G, B, M, S)
