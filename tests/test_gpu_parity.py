"""GPU parity: the sm_100a kernel (through the C ABI) against the fp64 oracle, entry by entry.

Acceptance (BASELINE.json:5): |y_gpu - y| <= 1e-5 * sum_j |Phi_mj r_j|; entries with a zero
scale must be exactly 0.  Products are exact and accumulation is fp32, so the simulated
worst case is ~2e-7; anything near 1e-5 is a layout bug, not rounding.
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


def encode_gpu(frames, phi, G, B, M):
    S, T, H, W = frames.shape
    enc = P.Encoder(W, H, G, B, M, phi)
    out = enc.encode_batch(torch.from_numpy(np.ascontiguousarray(frames)).cuda())
    torch.cuda.synchronize()
    return out.cpu().numpy(), enc


def assert_parity(y_gpu, frames, phi, G, B):
    y, S = oracle.encode(frames, phi, G, B)
    assert y_gpu.shape == y.shape
    ok, st = oracle.check_tolerance(y_gpu, y, S, REL)
    assert ok, st
    return st


# ------------------------------------------------------------------ the five configs, reduced T
# (ragged tails: T not a multiple of G where possible; full frame size, several tiles)
REDUCED = {
    "C1": dict(T=4, S=1),
    "C2": dict(T=19, S=1),    # GOPs 8,8,3
    "C3": dict(T=35, S=1),    # GOPs 16,16,3
    "C4": dict(T=11, S=1),    # GOPs 8,3; H=1080 has a half-outside last block row
    "C5": dict(T=37, S=2),    # GOPs 32,5 per stream, two streams
}


@pytest.mark.parametrize("name", list(REDUCED))
def test_config_parity_reduced(name):
    base = synth.CONFIGS[name]
    cfg = base.with_(**REDUCED[name])
    frames = synth.gen_video(cfg)
    for M in base.Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        y_gpu, _ = encode_gpu(frames, phi, cfg.G, cfg.B, M)
        assert_parity(y_gpu, frames, phi, cfg.G, cfg.B)


# ------------------------------------------------------------------ full sizes, sampled outputs
def sample_check(y_gpu_stream, frames_stream, phi, G, B, rng, n=400):
    n_cs, nblk, M = y_gpu_stream.shape
    ci = rng.integers(0, n_cs, n)
    bi = rng.integers(0, nblk, n)
    # always include the last CS frame and the last block (ragged corners)
    ci[:2] = n_cs - 1
    bi[:2] = [nblk - 1, 0]
    y, S = oracle.measure_entries(frames_stream, phi, G, B, ci, bi)
    ok, st = oracle.check_tolerance(y_gpu_stream[ci, bi], y, S, REL)
    assert ok, st


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_full_size_sampled(name):
    cfg = synth.CONFIGS[name]
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    rng = np.random.default_rng(7)
    for M in cfg.Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        y_gpu = out.cpu().numpy()
        assert np.isfinite(y_gpu).all()
        sample_check(y_gpu, frames[0], phi, cfg.G, cfg.B, rng)


def test_c5_full_batch_sampled():
    """All 64 streams of C5 in one launch (the bench launch); sampled per stream."""
    cfg = synth.CONFIGS["C5"]
    M = cfg.M
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    frames = synth.gen_video(cfg)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    out = enc.encode_batch(torch.from_numpy(frames).cuda())
    torch.cuda.synchronize()
    y = out.cpu().numpy()
    n_cs = y.shape[0] // cfg.S
    rng = np.random.default_rng(8)
    for s in range(0, cfg.S, 9):
        sample_check(y[s * n_cs:(s + 1) * n_cs], frames[s], phi, cfg.G, cfg.B, rng, n=60)


# ------------------------------------------------------------------ layout localisation
@pytest.mark.parametrize("B", [8, 16, 32])
def test_unit_residual_every_position(B):
    """One pixel per block differs (at a different in-block position per block): each
    output must be exactly v * Phi[:, j] -- a single exact product, no rounding at all."""
    M = 16
    N = B * B
    nbx = 4 * 16 // B if B < 32 else 4
    W = nbx * B
    nby = -(-N // nbx)
    H = nby * B
    key = np.full((H, W), 90, np.uint8)
    cs = key.copy()
    for b in range(nby * nbx):
        j = b % N
        by, bx = divmod(b, nbx)
        yy, xx = divmod(j, B)
        cs[by * B + yy, bx * B + xx] = 90 + (b % 150) + 1
    phi = synth.phi_from_seed(3, M, N)
    frames = np.stack([key, cs])[None]
    y_gpu, _ = encode_gpu(frames, phi, 2, B, M)
    phiv = oracle.phi_values(phi)
    for b in range(nby * nbx):
        v = (b % 150) + 1
        assert np.array_equal(y_gpu[0, b].astype(np.float64), v * phiv[:, b % N]), b


def test_identity_phi_lossless():
    """M = N identity (SPEC.md:113 lossless mode): y is the residual block, exactly."""
    B, N = 16, 256
    rng = np.random.default_rng(4)
    frames = rng.integers(0, 256, size=(1, 3, 2 * B, 3 * B), dtype=np.uint8)
    phi = np.eye(N).astype(np.float16).view(np.uint16)
    y_gpu, enc = encode_gpu(frames, phi, 3, B, N)
    assert enc.plan()["m_pad"] == 256
    y, _ = oracle.encode(frames, phi, 3, B)
    assert np.array_equal(y_gpu.astype(np.float64), y)


def test_zero_residual_exact_zero():
    rng = np.random.default_rng(5)
    f = rng.integers(0, 256, size=(1, 1, 144, 176), dtype=np.uint8)
    frames = np.repeat(f, 6, axis=1)
    phi = synth.phi_from_seed(9, 64, 256)
    y_gpu, _ = encode_gpu(frames, phi, 3, 16, 64)
    assert np.all(y_gpu == 0)


def test_saturation_and_subnormal():
    for B in (8, 16, 32):
        N = B * B
        frames = np.stack([np.zeros((B, 32), np.uint8), np.full((B, 32), 255, np.uint8)])[None]
        ones = np.ones((16, N)).astype(np.float16).view(np.uint16)
        y_gpu, _ = encode_gpu(frames, ones, 2, B, 16)
        assert np.all(y_gpu == 255.0 * N)
    # smallest subnormal times 255 -> exactly 255 * 2^-24 (no flush to zero)
    phi = np.zeros((16, 256), np.uint16)
    phi[:, 5] = 0x0001
    frames = np.zeros((1, 2, 16, 16), np.uint8)
    frames[0, 1, 0, 5] = 255
    y_gpu, _ = encode_gpu(frames, phi, 2, 16, 16)
    assert np.all(y_gpu[0, 0] == np.float32(255 * 2.0 ** -24))


def test_real_subnormals_in_phi_parity():
    """Phi at M=128 contains fp16 subnormals; sparse residual makes them matter."""
    phi = synth.phi_from_seed(synth.phi_seed(), 128, 256)
    assert np.any(((phi & 0x7FFF) > 0) & ((phi & 0x7FFF) < 0x400))
    rng = np.random.default_rng(6)
    key = rng.integers(0, 256, (64, 96), dtype=np.uint8)
    cs = key.copy()
    mask = rng.random((64, 96)) < 0.03
    cs[mask] = rng.integers(0, 256, mask.sum())
    frames = np.stack([key, cs])[None]
    y_gpu, _ = encode_gpu(frames, phi, 2, 16, 128)
    assert_parity(y_gpu, frames, phi, 2, 16)


@pytest.mark.parametrize("W,H,B,M,G,T", [
    (16, 1, 16, 16, 2, 2),        # one block, 15 rows of padding
    (48, 40, 32, 5, 3, 7),        # partial block in x and y, M not a multiple of 4
    (32, 24, 8, 17, 4, 9),        # M = 17 (scalar epilogue), ragged GOP
    (2048, 8, 8, 64, 2, 3),       # 256 blocks per row -> folds
    (128, 200, 16, 48, 5, 12),    # several tile rows, short last GOP
    (64, 64, 32, 80, 2, 4),       # largest B=32 M
    (64, 48, 16, 256, 3, 5),      # M = N = 256: the largest M (UMMA N limit), lossless mode
    (16, 300, 8, 4, 4, 9),        # one block column, tall frame, many tile rows
    (640, 96, 32, 64, 4, 9),      # C3-like rows with H % B == 0: 4-D strip boxes / Phi streaming plans
])
def test_edge_shapes(W, H, B, M, G, T):
    rng = np.random.default_rng(W * 7 + H)
    frames = rng.integers(0, 256, size=(2, T, H, W), dtype=np.uint8)
    phi = synth.phi_from_seed(W + H + M, M, B * B)
    y_gpu, _ = encode_gpu(frames, phi, G, B, M)
    assert_parity(y_gpu, frames, phi, G, B)


def test_gop_of_one_writes_nothing():
    frames = torch.zeros((1, 5, 32, 32), dtype=torch.uint8, device="cuda")
    enc = P.Encoder(32, 32, 1, 16, 16, synth.phi_from_seed(1, 16, 256))
    assert enc.measurement_count(1, 5) == 0
    sentinel = torch.full((8,), float("nan"), device="cuda")
    enc.encode_batch(frames, out=sentinel)
    torch.cuda.synchronize()
    assert torch.isnan(sentinel).all()


# ------------------------------------------------------------------ API consistency / determinism
def test_batch_gop_range_host_paths_agree_bitwise():
    cfg = synth.CONFIGS["C2"].with_(T=27, S=2)
    frames = synth.gen_video(cfg)
    phi = synth.phi_from_seed(synth.phi_seed(), cfg.M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, cfg.M, phi)
    fd = torch.from_numpy(frames).cuda()
    a = enc.encode_batch(fd)
    b = enc.encode_batch(fd)
    torch.cuda.synchronize()
    assert torch.equal(a, b)                          # deterministic
    a = a.cpu().numpy()
    # per-GOP calls through cs_encode_gop
    n_cs = a.shape[0] // 2
    for s in range(2):
        i = 0
        for key_t, cs_ts in oracle.gop_partition(cfg.T, cfg.G):
            g = enc.encode_gop(fd[s, key_t:key_t + 1 + len(cs_ts)].contiguous())
            torch.cuda.synchronize()
            assert np.array_equal(g.cpu().numpy(), a[s * n_cs + i:s * n_cs + i + len(cs_ts)])
            i += len(cs_ts)
    # GOP ranges [1, 4): 7 + 7 + 2 CS frames per stream
    rng_out = enc.encode_batch_gops(fd, 1, 4, torch.empty((2 * (7 + 7 + 2), enc.nblk, cfg.M), device="cuda"))
    torch.cuda.synchronize()
    r = rng_out.cpu().numpy()
    for s in range(2):
        assert np.array_equal(r[s * 16:(s + 1) * 16], a[s * n_cs + 7:s * n_cs + 23])
    # host path (pinned and pageable)
    h = enc.encode_batch_host(frames)
    assert np.array_equal(h, a)
    pinned = torch.from_numpy(frames).pin_memory()
    h2 = enc.encode_batch_host(pinned)
    assert np.array_equal(h2, a)


def test_bad_arguments_fail_loudly():
    phi = synth.phi_from_seed(1, 16, 256)
    enc = P.Encoder(64, 32, 4, 16, 16, phi)
    fd = torch.zeros((1, 4, 32, 64), dtype=torch.uint8, device="cuda")
    out = torch.empty(enc.out_shape(1, 4), device="cuda")
    with pytest.raises(P.CSError):
        P.lib()  # loaded
        rc = P.lib().cs_encode_batch(enc._h, fd.data_ptr() + 1, 1, 4, out.data_ptr(), None)
        P._check(rc)
    with pytest.raises(P.CSError):
        enc.encode_gop(fd[0, :1].expand(5, 32, 64).contiguous())
    with pytest.raises(P.CSError):
        P.Encoder(64, 32, 4, 12, 16, np.zeros((16, 144), np.uint16))
    bad = phi.copy()
    bad[0, 0] = 0x7C00  # +inf
    with pytest.raises(P.CSError) as e:
        P.Encoder(64, 32, 4, 16, 16, bad)
    assert e.value.code == P.CS_ERR_PHI


def test_encoders_with_different_plans_coexist():
    """Regression: creating a second encoder with a smaller shared-memory plan must not break
    launches of the first (the max-dynamic-smem attribute is per kernel, not per encoder)."""
    cfg = synth.CONFIGS["C4"].with_(T=3)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    encs = [P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, 256))
            for M in (16, 128)]
    assert encs[0].plan()["smem_bytes"] != encs[1].plan()["smem_bytes"]
    for M, e in zip((16, 128), encs):
        out = e.encode_batch(fd)
        torch.cuda.synchronize()
        phi = synth.phi_from_seed(synth.phi_seed(), M, 256)
        assert_parity(out.cpu().numpy(), frames, phi, cfg.G, cfg.B)


def test_all_candidate_plans_bitwise_identical():
    """Every feasible plan (tile rows, folds, K-chunk, key mode, ring depths) computes the same
    per-block MMA chain, so outputs are bit-identical -- the autotuner can pick any of them."""
    for name, M in (("C4", 64), ("C5", 4), ("C3", 64)):
        base = synth.CONFIGS[name]
        cfg = base.with_(T=min(base.T, 9 if name != "C3" else 17), S=1)
        frames = synth.gen_video(cfg)
        fd = torch.from_numpy(frames).cuda()
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        n = min(enc.num_candidates(), 8)
        assert n >= 2
        ref = None
        seen = set()
        for i in range(n):
            plan = enc.set_candidate(i)
            seen.add((plan["tile_block_rows"], plan["chunk_rows"], plan["key_resident"]))
            out = enc.encode_batch(fd)
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
                assert_parity(out.cpu().numpy(), frames, phi, cfg.G, cfg.B)
            else:
                assert torch.equal(out, ref), (name, plan)
        assert len(seen) >= 2
        chosen = enc.autotune(fd, max_candidates=3, reps=1)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        assert torch.equal(out, ref) and chosen["smem_bytes"] > 0


@pytest.mark.parametrize("M", [16, 32, 64, 128])
def test_bench_candidate_plans_bitwise_identical_c4(M):
    """bench.py autotunes among the top 12 plans of every C4 M; each of them gives the same bits as the
    first, which is checked against the oracle -- so whichever plan the bench times is a checked plan.
    T = 2G + 3 = 19: two full GOPs and a ragged third."""
    base = synth.CONFIGS["C4"]
    cfg = base.with_(T=2 * base.G + 3, S=1)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    n = min(enc.num_candidates(), 12)
    ref = None
    for i in range(n):
        plan = enc.set_candidate(i)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
            assert_parity(out.cpu().numpy(), frames, phi, cfg.G, cfg.B)
        else:
            assert torch.equal(out, ref), (M, i, plan)


def test_host_multi_encoder_path():
    """cs_encode_batch_host_multi: several encoders (different M and B) over the same host frames
    give exactly the device-path outputs; mismatched geometry is rejected."""
    cfg = synth.CONFIGS["C2"].with_(T=19, S=3)
    frames = synth.gen_video(cfg)
    encs = [P.Encoder(cfg.W, cfg.H, cfg.G, B, M, synth.phi_from_seed(7 + M, M, B * B))
            for B, M in ((16, 16), (16, 64), (8, 12), (32, 40))]
    outs = P.encode_batch_host_multi(encs, frames)
    fd = torch.from_numpy(frames).cuda()
    for e, o in zip(encs, outs):
        ref = e.encode_batch(fd)
        torch.cuda.synchronize()
        assert np.array_equal(o, ref.cpu().numpy())
    other = P.Encoder(cfg.W, cfg.H, cfg.G + 1, 16, 16, synth.phi_from_seed(1, 16, 256))
    with pytest.raises(ValueError):
        P.encode_batch_host_multi([encs[0], other], frames)
    with pytest.raises(P.CSError):
        P.encode_batch_host_multi([encs[0], encs[0]], frames)
