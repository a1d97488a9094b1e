import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_1311_1419_b200 as P
wl, M = sys.argv[1], int(sys.argv[2])
cfg = synth.CONFIGS[wl]
frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
y = e.encode_batch(frames)
del frames
x = e.adjoint(y)
for _ in range(3):
    e.adjoint(y, x)
torch.cuda.synchronize()
print("ok")
