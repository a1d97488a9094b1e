"""Input-generator checks (synth/): determinism and the statistics SPEC.md asks of Phi."""
import hashlib
import math

import numpy as np

import synth


def test_phi_deterministic_and_shape():
    a = synth.phi_from_seed(42, 64, 256)
    b = synth.phi_from_seed(42, 64, 256)
    assert a.dtype == np.uint16 and a.shape == (64, 256)
    assert np.array_equal(a, b)                                  # SPEC.md:133 bit-identical rebuild
    assert not np.array_equal(a, synth.phi_from_seed(43, 64, 256))


def test_phi_statistics():
    """Column means ~0 within 4/sqrt(M); row energy E[sum_j Phi_mj^2] = N/M."""
    for M, N in [(16, 256), (64, 256), (128, 256), (64, 1024), (4, 64)]:
        phi = synth.phi_from_seed(synth.phi_seed(), M, N).view(np.float16).astype(np.float64)
        assert np.all(np.isfinite(phi))
        assert np.all(np.abs(phi.mean(axis=0)) <= 4.0 / math.sqrt(M))
        energy = (phi ** 2).sum(axis=1).mean()
        assert abs(energy - N / M) < 0.15 * N / M
        assert np.abs(phi).max() <= 2048


def test_phi_has_subnormals_at_large_M():
    """fp16 subnormals occur for M >= 64 -- the parity tests rely on them."""
    phi = synth.phi_from_seed(synth.phi_seed(), 128, 256)
    mag = phi & 0x7FFF
    assert np.any((mag > 0) & (mag < 0x0400))


def test_video_deterministic_and_plausible():
    cfg = synth.CONFIGS["C1"]
    a = synth.gen_video(cfg)
    b = synth.gen_video(cfg)
    assert a.shape == (1, 4, 144, 176) and a.dtype == np.uint8
    assert np.array_equal(a, b)
    # mostly static background: residual small away from the object, large on it
    r = a[0, 1].astype(int) - a[0, 0].astype(int)
    assert 1.5 < np.median(np.abs(r)) + 1 < 6
    assert np.abs(r).max() > 60
    # rendering a stream in pieces gives the same frames (counter-based noise)
    cfg2 = synth.CONFIGS["C2"].with_(T=12)
    full = synth.gen_stream(cfg2, 0)
    part = synth.gen_stream(cfg2, 0, t0=5, T=4)
    assert np.array_equal(full[5:9], part)


def test_streams_differ():
    cfg = synth.CONFIGS["C5"].with_(T=2, S=2, W=64, H=48)
    v = synth.gen_video(cfg)
    assert not np.array_equal(v[0], v[1])
    h = hashlib.sha256(v.tobytes()).hexdigest()
    assert h == hashlib.sha256(synth.gen_video(cfg).tobytes()).hexdigest()
