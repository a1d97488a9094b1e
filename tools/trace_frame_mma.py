"""MMA-warp wait breakdown of the frame-level GEMM (needs a build whose trace events 0/1 are recorded
after the A-tile and residual-operand waits in the MMA loop; see DESIGN.md sec.7 f2)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, paper_1311_1419_b200 as P
W, H, G, S, T = 176, 144, 5, 64, 400
n = W * H; m = round(n / 50)
cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
fe = P.FrameEncoder(W, H, G, m, synth.phi_from_seed(synth.phi_seed(), m, n))
y = fe.encode_batch(fd)
cap = 400
buf = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
fe.set_trace(buf, cap); torch.cuda.synchronize()
fe.encode_batch(fd, y); torch.cuda.synchronize(); fe.set_trace(None, 0)
t = buf.view(4, cap).cpu().numpy().astype(np.int64)
k = int((t[3] > 0).sum()); t = t[:, 1:k] - t[t > 0].min()
med = lambda x: float(np.median(x))
print("period", med(np.diff(t[3])))
print("A wait (gotA[i] - issued[i-1])", med(t[0][1:] - t[3][:-1]))
print("B wait (gotB[i] - gotA[i])", med(t[1] - t[0]))
print("issue (issued[i] - gotB[i])", med(t[3] - t[1]))
print("conv done -> gotB", med(t[1] - t[2]))
