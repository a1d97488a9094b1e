"""Timeline of the single-pass per-frame q16 epilogue (CTA 0): d_full -> contribution published ->
(look-back wait done for the item 2 back) -> item done; plus the producer/converter/MMA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_1311_1419_b200 as P
cfg = synth.CONFIGS["C4"]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
gran = int(sys.argv[2]) if len(sys.argv) > 2 else 0
enc.encode_batch_q16(fd, gran)
cap = 128
ev = enc.TRACE_EVENTS
buf = torch.zeros(len(ev) * cap, dtype=torch.int64, device="cuda")
enc.set_trace(buf, cap)
torch.cuda.synchronize()
enc.encode_batch_q16(fd, gran)
torch.cuda.synchronize()
enc.set_trace(None, 0)
t = buf.view(len(ev), cap).cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
d = {k: np.where(t[i] > 0, t[i] - t0, -1) for i, k in enumerate(ev)}
n = int((d["e_done"] >= 0).sum())
print(f"M={M} gran={gran} items traced {n}")
med = lambda x: float(np.median(x)) if len(x) else float("nan")
e = lambda k: d[k][:n]
print("item period (e_done diff)", med(np.diff(e("e_done"))))
print("dfull -> published (pass A + atomics)", med(e("m_afull") - e("e_dfull")))
print("published -> wait done (look-back wait, item-2)", med(e("c_aempty")[:n] - e("m_afull")[:n]))
print("wait done -> done (quantise)", med(e("e_done") - e("c_aempty")))
print("done -> next dfull (waiting for MMA)", med(e("e_dfull")[1:n] - e("e_done")[:n - 1]))
print("first 10 items:")
for i in range(min(10, n)):
    print(i, " ".join(f"{k}={d[k][i]}" for k in ("e_dfull", "m_afull", "c_aempty", "e_done")))
