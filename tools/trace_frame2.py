"""Per-chunk timeline of the 2-SM frame GEMM (pair 0): producer issue -> leader / peer residual
written -> MMAs issued."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
k = int((t[3] > 0).sum())
t = t[:, :k] - t[t > 0].min()
med = lambda x: float(np.median(x))
print("chunks traced", k)
print("chunk period (MMA issued diff)", med(np.diff(t[3])))
print("leader conversion (done - start)", med(t[1] - t[2]), " start - issue", med(t[2] - t[0]))
print("MMA issued - conv done", med(t[3] - t[1]))
for i in range(0, min(k, 12)):
    print(i, t[:, i].tolist())
