"""Small runs of every device path for the CSENC_CHECKS bounds-check build (the memory-safety gate:
compute-sanitizer is not available on this pool): every key mode, block size, folds, partial
blocks, ragged GOPs, the q16 modes, closed-loop / chained keys, per-GOP Phi, the adjoint and the
frame-level GEMM (split-K).  Results are checked against the oracle; a bound violation traps (the
process dies).  Prints ALL_OK at the end.  With CSENC_STRESS=<seed> (the race gate: random delays after
every mbarrier wait in K1) and SANITIZE_K1_ONLY=1 only the K1 plan sweep runs, every candidate plan
of each case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
import paper_1311_1419_b200 as P

cases = [(64, 16, 3, 2, 16, 16), (176, 144, 5, 4, 16, 64), (96, 40, 7, 3, 32, 16), (1280, 24, 5, 4, 8, 4),
         (352, 40, 9, 8, 16, 32), (48, 40, 5, 3, 32, 5), (160, 72, 7, 4, 8, 12), (640, 96, 9, 4, 32, 64),
         (208, 70, 6, 3, 32, 96)]
K1_ONLY = os.environ.get("SANITIZE_K1_ONLY") == "1"
ok_all = True


def report(tag, ok):
    global ok_all
    ok_all &= bool(ok)
    print(tag, ok)


for W, H, T, G, B, M in cases:
    rng = np.random.default_rng(W + H)
    frames = rng.integers(0, 256, size=(2, T, H, W), dtype=np.uint8)
    phi = synth.phi_from_seed(W, M, B * B)
    enc = P.Encoder(W, H, G, B, M, phi)
    fd = torch.from_numpy(frames).cuda()
    y, S = oracle.encode(frames, phi, G, B)
    tag = f"{W}x{H} T{T} G{G} B{B} M{M}"
    # the first three candidates, plus every KEY_CHUNK (key_resident 3) and streamed-Phi candidate
    # among the first 24; all of them under the race gate
    cands = [i for i in range(enc.num_candidates())
             if i < 3 or K1_ONLY or (i < 24 and (enc.set_candidate(i)["key_resident"] == 3 or enc.plan()["phi_stream"]))]
    for i in cands[:40]:
        enc.set_candidate(i)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        report(f"{tag} plan {i} key {enc.plan()['key_resident']}", oracle.check_tolerance(out.cpu().numpy(), y, S)[0])
    if K1_ONLY:
        continue
    # Phi-streaming plans (and with them the 4-D strip boxes when H % B == 0): the first two
    streaming = [i for i in range(enc.num_candidates()) if enc.set_candidate(i)["phi_stream"]][:2]
    for i in streaming:
        enc.set_candidate(i)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        report(f"{tag} phi-stream plan {i}", oracle.check_tolerance(out.cpu().numpy(), y, S)[0])
    enc.set_candidate(0)
    enc.set_candidate(0)
    # f1: q16 modes (codes within +-1 of the oracle's quantisation of the exact y)
    oc, _ = oracle.quantize_frames(y)
    for gran in (P.Encoder.Q16_FRAME, P.Encoder.Q16_ROW):
        try:
            c, s = enc.encode_batch_q16(fd, gran)
            torch.cuda.synchronize()
        except P.CSError as e:
            report(f"{tag} q16 {gran} unsupported ({e.code})", e.code == P.CS_ERR_UNSUPPORTED)
            continue
        if gran == P.Encoder.Q16_ROW:
            report(f"{tag} q16 row", np.all(np.isfinite(s.cpu().numpy())))
        else:
            report(f"{tag} q16 {gran}", np.abs(c.cpu().numpy().astype(int) - oc).max() <= 1)
    # f4: closed loop, chained, per-GOP Phi
    qs = oracle.key_qsteps(1.0)
    yk, keys, _ = enc.encode_batch_closed_loop(fd, P.key_qsteps(1.0))
    torch.cuda.synchronize()
    yo, So = oracle.encode_stream_closed_loop(frames[0], phi, G, B, qs)
    n_cs = yo.shape[0]
    report(f"{tag} closed loop", oracle.check_tolerance(yk.cpu().numpy()[:n_cs], yo, So)[0])
    yc = enc.encode_batch_chained(fd)
    torch.cuda.synchronize()
    yo, So = oracle.encode_stream_chained(frames[1], phi, G, B)
    report(f"{tag} chained", oracle.check_tolerance(yc.cpu().numpy()[n_cs:], yo, So)[0])
    phis = [synth.phi_from_seed(W ^ g, M, B * B) for g in range(-(-T // G))]
    enc.set_gop_phis(phis)
    yg = enc.encode_batch(fd)
    torch.cuda.synchronize()
    enc.set_gop_phis(None)
    yo, So = oracle.encode_stream_gop_phis(frames[0], phis, G, B)
    report(f"{tag} gop phis", oracle.check_tolerance(yg.cpu().numpy()[:n_cs], yo, So)[0])
    # f3: adjoint of the measurements
    if M % 4 == 0:
        x = enc.adjoint(torch.from_numpy(y.astype(np.float32)).cuda())
        torch.cuda.synchronize()
        xo = oracle.adjoint(y.astype(np.float32).astype(np.float64), phi, W, H, B)
        Sx = oracle.adjoint_tolerance_scale(y.astype(np.float32).astype(np.float64), phi, W, H, B)
        report(f"{tag} adjoint", np.all(np.abs(x.cpu().numpy() - xo) <= 1e-5 * Sx))

# f2: frame-level GEMM (split-K, windows per stream and across streams)
for W, H, G, T, S, m in [] if K1_ONLY else [(32, 16, 3, 7, 2, 37), (64, 8, 5, 20, 3, 300), (176, 144, 5, 10, 2, 507)]:
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
    frames = synth.gen_video(cfg)
    A = synth.phi_from_seed(7 + m, m, W * H)
    fe = P.FrameEncoder(W, H, G, m, A)
    yg = fe.encode_batch(torch.from_numpy(frames).cuda())
    torch.cuda.synchronize()
    n_cs = oracle.cs_frame_count(T, G)
    good = True
    for s in range(S):
        yo, So = oracle.measure_frame(frames[s], A, G)
        good &= np.all(np.abs(yg.cpu().numpy()[s * n_cs:(s + 1) * n_cs] - yo) <= (W * H / 16 + 16) * 2.0 ** -23 * So)
    report(f"frame {W}x{H} G{G} T{T} S{S} m{m}", good)
print("ALL_OK" if ok_all else "FAILURES")
