"""Minimal launcher for ncu: `python tools/run_one.py WL M [reps] [candidate] [f32|q16row|q16frame]` encodes
workload WL at M reps times with the planner's (or the given) candidate plan -- no autotune, no oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1311_1419_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
M = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.M
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cand = int(sys.argv[4]) if len(sys.argv) > 4 else -1
out_kind = sys.argv[5] if len(sys.argv) > 5 else "f32"
frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
if cand >= 0:
    e.set_candidate(cand)
for _ in range(reps):
    if out_kind == "f32":
        e.encode_batch(frames)
    else:
        e.encode_batch_q16(frames, {"q16frame": 0, "q16row": 1}[out_kind])
torch.cuda.synchronize()
print("ok", wl, M, e.plan())
