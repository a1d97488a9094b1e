"""Per-event pipeline timeline of CTA 0 (cs_encoder_set_trace) for one config; prints the
median latency of every handoff so the slowest stage of the pipeline is visible."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_1311_1419_b200 as P

def main(workload="C4", M=None, cap=256, T=None, q16=None):
    cfg = synth.CONFIGS[workload]
    M = M or cfg.M
    if T:
        cfg = cfg.with_(T=T)
    frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
    tf = os.environ.get("TUNE_FILE")
    if tf and os.path.exists(tf):
        k = json.load(open(tf)).get(f"{workload}:{M}")
        if k is not None:
            enc.set_candidate(int(k))
    run = (lambda: enc.encode_batch(frames, out)) if q16 is None else (lambda: enc.encode_batch_q16(frames, q16))
    out = enc.encode_batch(frames)
    run()
    ev = enc.TRACE_EVENTS
    buf = torch.zeros(len(ev) * cap, dtype=torch.int64, device="cuda")
    enc.set_trace(buf, cap)
    torch.cuda.synchronize()
    run()
    torch.cuda.synchronize()
    enc.set_trace(None, 0)
    t = buf.view(len(ev), cap).cpu().numpy().astype(np.int64)
    n = int((t[ev.index("c_done")] > 0).sum())
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    print(f"{workload} M={M} plan={enc.plan()} items_traced={n}")
    d = {k: t[i, :n] for i, k in enumerate(ev)}
    def med(x):
        x = x[np.isfinite(x)]
        return float(np.median(x)) if x.size else float("nan")
    rep = {
        "stage period (c_done[i]-c_done[i-1])": med(np.diff(d["c_done"])),
        "convert (c_done - c_aempty)": med(d["c_done"] - d["c_aempty"]),
        "  of which ALU+st issue (c_conv - c_aempty)": med(d["c_conv"] - d["c_aempty"]),
        "  of which wait::st (c_done - c_conv)": med(d["c_done"] - d["c_conv"]),
        "converter wait A free (c_aempty - c_full)": med(d["c_aempty"] - d["c_full"]),
        "handoff c_done -> m_afull": med(d["m_afull"] - d["c_done"]),
        "mma issue (m_issued - m_afull)": med(d["m_issued"] - d["m_afull"]),
        "A round trip (c_aempty[i+2] - m_issued[i])": med(d["c_aempty"][2:] - d["m_issued"][:-2]),
        "tma latency (c_full - p_issued)": med(d["c_full"] - d["p_issued"]),
        "epilogue (e_done - e_dfull)": med(d["e_done"] - d["e_dfull"]),
    }
    if q16 == 0 and (d["e_rows"] > 0).any():   # q16frame fused (EPI_F32Q): re-quantisation warps
        ne = int((t[ev.index("e_done")] > 0).sum())
        ea, er, ed = t[ev.index("e_arrived"), :ne], t[ev.index("e_rows"), :ne], t[ev.index("e_done"), :ne]
        rep["requant wait (ready - epilogue done)"] = med(ea - ed)
        rep["requant item (done - ready)"] = med(er - ea)
        rep["requant lag at the end (last done - last epilogue)"] = float(er[-1] - ed[-1])
    elif (d["e_arrived"] > 0).any():
        rep["  epilogue ld+reduce (e_arrived - e_dfull)"] = med(d["e_arrived"] - d["e_dfull"])
        rep["  epilogue row wait (e_rows - e_arrived)"] = med(d["e_rows"] - d["e_arrived"])
        rep["  epilogue scale+codes (e_done - e_rows)"] = med(d["e_done"] - d["e_rows"])
    if "k_start" in ev and t[ev.index("k_end"), 0] > 0:
        ks, ke = t[ev.index("k_start"), 0], t[ev.index("k_end"), 0]
        ne_ = int((t[ev.index("e_done")] > 0).sum())
        rep["CTA 0 kernel (k_end - k_start)"] = float(ke - ks)
        rep["  prologue (first p_issued - k_start)"] = float(d["p_issued"][0] - ks)
        rep["  fill (first e_done - first p_issued)"] = float(t[ev.index("e_done"), 0] - d["p_issued"][0])
        rep["  drain (k_end - last e_done)"] = float(ke - t[ev.index("e_done"), ne_ - 1]) if ne_ else float("nan")
        rep["  CS items / epilogue items of CTA 0"] = float(n * 1000 + ne_)
        kst = t[ev.index("k_start")]
        for j, what in ((1, "barriers initialised"), (2, "TMEM allocated"), (4, "offset table written"),
                        (3, "prologue barrier passed"), (5, "producer: Phi issued"),
                        (6, "producer: first unit decoded"), (7, "producer: first Phi slice issued")):
            if kst[j] >= 0:
                rep[f"    prologue: {what} (since k_start)"] = float(kst[j] - ks)
    for k, v in rep.items():
        print(f"  {k:45s} {v:9.0f} cycles")
    # utilisation over the traced window (items 2..n-2 to skip the prologue)
    lo, hi = 2, n - 2
    span = float(d["c_done"][hi] - d["c_done"][lo])
    per = span / (hi - lo)
    util = {
        "converter busy": np.sum(d["c_done"][lo:hi] - d["c_aempty"][lo:hi]) / span,
        "converter wait stage": np.sum(d["c_full"][lo + 1:hi + 1] - d["c_done"][lo:hi]) / span,
        "converter wait A": np.sum(d["c_aempty"][lo:hi] - d["c_full"][lo:hi]) / span,
        "mma busy (issue)": np.sum(d["m_issued"][lo:hi] - d["m_afull"][lo:hi]) / span,
        "mma wait A": np.sum(d["m_afull"][lo + 1:hi + 1] - d["m_issued"][lo:hi]) / span,
        "producer wait slot": np.sum(d["p_empty"][lo + 1:hi + 1] - d["p_issued"][lo:hi]) / span,
    }
    ne = int((t[ev.index("e_done")] > 0).sum())
    if ne > 4:
        e0 = d["e_dfull"][:ne] if len(d["e_dfull"]) >= ne else d["e_dfull"]
        espan = float(t[ev.index("e_done"), ne - 2] - t[ev.index("e_done"), 1])
        util["epilogue busy"] = float(np.sum(t[ev.index("e_done"), 2:ne - 1] - t[ev.index("e_dfull"), 2:ne - 1]) / espan)
    print(f"  period/item {per:.0f} cycles = {30720 if False else 0}", " ".join(f"{k}={v:.2f}" for k, v in util.items()))
    print("first 12 items (cycles since first event):")
    print("   i " + " ".join(f"{k:>9s}" for k in ev))
    for i in range(min(int(os.environ.get("TRACE_ROWS", "12")), n)):
        print(f"{i:4d} " + " ".join(f"{t[j, i]:9d}" for j in range(len(ev))))
    return rep

if __name__ == "__main__":
    w = sys.argv[1] if len(sys.argv) > 1 else "C4"
    Ms = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else [None]
    q16 = None if len(sys.argv) <= 3 or sys.argv[3] == "f32" else {"q16frame": 0, "q16row": 1}[sys.argv[3]]
    for M in Ms:
        main(w, M, q16=q16)
