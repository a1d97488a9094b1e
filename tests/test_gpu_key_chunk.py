"""KEY_CHUNK plans (chunk-outer / frame-inner units): every CS frame of a unit
accumulates in its own TMEM accumulator while the key chunk (in converter registers) and Phi's
K-slice cross L2 -> SMEM once per unit and chunk.  The per-block MMA chain is the same K order as
every other plan, so the outputs must be bitwise those of the other plans, and the oracle's within
the north-star tolerance -- for resident and streamed Phi, ragged frames, short GOPs, per-GOP
matrices, decoded keys and the q16 epilogues."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_1311_1419_b200 as P  # noqa: E402


def split_candidates(enc):
    kc, other = [], []
    for i in range(enc.num_candidates()):
        (kc if enc.set_candidate(i)["key_resident"] == 3 else other).append(i)
    return kc, other


CASES = [
    # W, H, T, G, M   (B = 32)
    (640, 480, 17, 16, 64),     # C3 geometry, one full GOP + a 1-frame GOP
    (640, 200, 11, 4, 64),      # H % 32 != 0: bulk-copied strips + zero rows
    (208, 96, 9, 3, 32),        # W % 32 = 16: right halves outside the frame
    (320, 128, 10, 2, 16),      # G = 2: one CS frame per GOP (U = 1)
    (640, 480, 12, 8, 96),      # Phi > resident budget: streamed slices only
    (192, 64, 7, 7, 128),
]


@pytest.mark.parametrize("W,H,T,G,M", CASES)
def test_key_chunk_plans_bitwise_and_parity(W, H, T, G, M):
    cfg = synth.CONFIGS["C3"].with_(W=W, H=H, T=T, G=G, Ms=(M,), S=2)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phi = synth.phi_from_seed(synth.phi_seed() + 3 * M, M, 1024)
    enc = P.Encoder(W, H, G, 32, M, phi)
    kc, other = split_candidates(enc)
    assert kc and other
    enc.set_candidate(other[0])
    ref = enc.encode_batch(fd).clone()
    y, S = oracle.encode(frames, phi, G, 32)
    ok, st = oracle.check_tolerance(ref.cpu().numpy(), y, S)
    assert ok, st
    seen = set()
    for i in kc[:8]:
        plan = enc.set_candidate(i)
        seen.add((plan["phi_stream"], plan["a_bufs"], plan["tile_block_rows"], plan["chunk_rows"]))
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), plan
    # 16-bit epilogues on the best KEY_CHUNK plan == on the reference plan
    enc.set_candidate(other[0])
    q_ref = [enc.encode_batch_q16(fd, g) for g in (0, 1)]
    enc.set_candidate(kc[0])
    for g, (c0, s0) in zip((0, 1), q_ref):
        c1, s1 = enc.encode_batch_q16(fd, g)
        torch.cuda.synchronize()
        assert torch.equal(c0, c1) and torch.equal(s0, s1), g


def test_key_chunk_gop_phis_and_decoded_keys():
    W, H, T, G, M = 640, 160, 40, 16, 64
    cfg = synth.CONFIGS["C3"].with_(W=W, H=H, T=T, G=G, Ms=(M,), S=1)
    frames = synth.gen_video(cfg)
    fd = torch.from_numpy(frames).cuda()
    phis = [synth.phi_from_seed(synth.phi_seed() ^ g, M, 1024) for g in range(3)]
    enc = P.Encoder(W, H, G, 32, M, phis[0])
    kc, other = split_candidates(enc)
    both = {enc.set_candidate(i)["phi_stream"]: i for i in kc}
    # per-GOP matrices: resident reload and streamed slices
    enc.set_gop_phis(phis)
    enc.set_candidate(other[0])
    ref = enc.encode_batch(fd).clone()
    got = ref.cpu().numpy()
    for g in range(3):
        sub = frames[:, g * G:(g + 1) * G]
        y, S = oracle.encode(sub, phis[g], G, 32)
        ok, st = oracle.check_tolerance(got[g * (G - 1):g * (G - 1) + y.shape[0]], y, S)
        assert ok, (g, st)
    for ps, i in both.items():
        enc.set_candidate(i)
        assert torch.equal(enc.encode_batch(fd), ref), ps
    enc.set_gop_phis(None)
    # closed loop: residuals against decoded keys (Eq. 2-3) through the keys buffer
    qs = P.key_qsteps(2.0)
    enc.set_candidate(other[0])
    keys, _ = enc.key_codec(fd, qs)
    ref = enc.encode_batch_keys(fd, keys).clone()
    for ps, i in both.items():
        enc.set_candidate(i)
        assert torch.equal(enc.encode_batch_keys(fd, keys), ref), ps
    y, S = oracle.encode_stream_closed_loop(frames[0], phis[0], G, 32, oracle.key_qsteps(2.0))
    ok, st = oracle.check_tolerance(ref.cpu().numpy(), y, S)
    assert ok, st
