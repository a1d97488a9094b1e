"""C3 launch-rate experiment: per-launch time of back-to-back encodes (a) plain Python calls, (b) one CUDA
graph of the same calls, with and without stable inputs; and the CPU cost of one binding call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1311_1419_b200 as P

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
M = cfg.M
frames = torch.from_numpy(synth.gen_video(cfg)).cuda()
e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
out = e.encode_batch(frames)
e.autotune(frames, out=out, max_candidates=12, reps=3)
R = 50
for stable in (False, True):
    e.set_stable_inputs(stable)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        e.encode_batch(frames, out)
    t_cpu = (time.perf_counter() - t0) / R * 1e6
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        e.encode_batch(frames, out)
    e1.record(); torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / R * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(R):
            e.encode_batch(frames, out)
    g.replay(); torch.cuda.synchronize()
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / R * 1e3
    print(f"{wl} stable={stable}: CPU {t_cpu:.1f} us per call (queueing), plain {plain:.1f} us/launch, graph {graph:.1f} us/launch")
