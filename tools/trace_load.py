import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_1311_1419_b200 as P
cfg = synth.CONFIGS["C4"]
frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
M = 16
enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(1, M, 256))
out = enc.encode_batch(frames)
cap = 256
ev = enc.TRACE_EVENTS
buf = torch.zeros(len(ev) * cap, dtype=torch.int64, device="cuda")
enc.set_trace(buf, cap)
torch.cuda.synchronize()
enc.encode_batch(frames, out)
torch.cuda.synchronize()
t = buf.view(len(ev), cap).cpu().numpy()
t0 = t[t > 0].min()
print(enc.plan())
print("   i  p_empty p_issued   c_full  (relative cycles)   lat=c_full-p_issued")
for i in range(40):
    pe, pi, cf = t[0, i] - t0, t[1, i] - t0, t[2, i] - t0
    print(f"{i:4d} {pe:8d} {pi:8d} {cf:8d}   {cf - pi:8d}")
