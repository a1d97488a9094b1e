"""Time every K1 plan candidate of a workload (outputs are bitwise identical across plans), L2
flushed before each launch when the input fits in L2.  usage: python tools/plan_scan.py C3 [M] [top]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1311_1419_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
Ms = [int(sys.argv[2])] if len(sys.argv) > 2 and sys.argv[2] != "all" else list(cfg.Ms)
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
dev = torch.device("cuda", 0)
frames = torch.from_numpy(synth.gen_video(cfg)).to(dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if frames.numel() < (256 << 20) else None
s = torch.cuda.current_stream(dev)
for M in Ms:
    phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
    e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
    out = torch.empty(e.out_shape(cfg.S, cfg.T), dtype=torch.float32, device=dev)
    res = []
    for i in range(e.num_candidates()):
        pl = e.set_candidate(i)
        for _ in range(3):
            e.encode_batch(frames, out, s)
        ts = []
        for _ in range(20):
            if flush is not None:
                flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            e.encode_batch(frames, out, s)
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
        res.append((ms, i, pl))
    res.sort(key=lambda r: r[0])
    n_cs = cfg.S * (cfg.T - -(-cfg.T // cfg.G))
    for ms, i, pl in res[:top]:
        print(f"{wl} M={M} cand {i:3d} {ms * 1e3:8.1f} us {n_cs * cfg.W * cfg.H / ms / 1e6:7.0f} Gpx/s",
              {k: pl[k] for k in ("tile_block_rows", "folds", "lanes", "chunk_rows", "stages", "key_resident",
                                  "a_bufs", "d_bufs", "phi_stream")})
    print(f"{wl} M={M}: {len(res)} candidates; planner's rank of the best: {res[0][1]}", flush=True)
