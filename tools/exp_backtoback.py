"""Back-to-back launches without per-launch events: `python tools/exp_backtoback.py WL [reps]` -> us per
step (all M of the workload) timed with one event pair around reps steps.  Shows what programmatic
dependent launch (CSENC_LIB=... for the A/B) is worth when nothing sits between the launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1311_1419_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = synth.CONFIGS[wl]
Ms = [16, 32, 64, 128] if wl == "C4" else [cfg.M]
frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
encs = [P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)) for M in Ms]
outs = [e.encode_batch(frames) for e in encs]
for e, o in zip(encs, outs):
    e.autotune(frames, out=o, max_candidates=12, reps=3)
torch.cuda.synchronize()
res = []
for trial in range(3):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        for e, o in zip(encs, outs):
            e.encode_batch(frames, out=o)
    t1.record()
    torch.cuda.synchronize()
    res.append(t0.elapsed_time(t1) / reps * 1e3)
print(os.path.basename(os.environ.get("CSENC_LIB", "default")), wl, "us/step", [round(r, 2) for r in res])
