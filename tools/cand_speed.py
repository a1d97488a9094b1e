"""Time every candidate plan of C4 (fp32 encode) for the given Ms: which plans are fast."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1311_1419_b200 as P
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
Ms = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(cfg.Ms)
fd = torch.from_numpy(synth.gen_video(cfg)).cuda()
for M in Ms:
    enc = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2))
    out = enc.encode_batch(fd)
    for k in range(min(8, enc.num_candidates())):
        pl = enc.set_candidate(k)
        for _ in range(3): enc.encode_batch(fd, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): enc.encode_batch(fd, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        npx = out.shape[0] * cfg.W * cfg.H
        print(f"M={M} cand {k}: {npx / ms / 1e6:7.0f} Gpx/s  T_r={pl['tile_block_rows']} F={pl['folds']} chunk={pl['chunk_rows']} "
              f"stages={pl['stages']} key={pl['key_resident']} a={pl['a_bufs']} d={pl['d_bufs']}")
