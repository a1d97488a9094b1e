"""Small GPU smoke/debug run: tiny cases vs the oracle, printing where they differ."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle, synth
import paper_1311_1419_b200 as P

def run(W, H, T, G, B, M, seed=0, kind="random", S=1):
    rng = np.random.default_rng(seed)
    if kind == "random":
        frames = rng.integers(0, 256, size=(S, T, H, W), dtype=np.uint8)
    elif kind == "unit":
        frames = np.full((S, T, H, W), 100, np.uint8)
        frames[0, 1, 0, 0] = 101
    phi = synth.phi_from_seed(seed + 5, M, B * B)
    enc = P.Encoder(W, H, G, B, M, phi)
    print("plan", enc.plan())
    fd = torch.from_numpy(frames).cuda()
    out = enc.encode_batch(fd)
    torch.cuda.synchronize()
    y_gpu = out.cpu().numpy().astype(np.float64)
    y, Sc = oracle.encode(frames, phi, G, B)
    ok, st = oracle.check_tolerance(y_gpu, y, Sc)
    print(f"W={W} H={H} T={T} G={G} B={B} M={M} kind={kind}: ok={ok} {st}")
    if not ok:
        bad = np.argwhere(np.abs(y_gpu - y) > 1e-5 * Sc + 0)
        print("first bad", bad[:10])
        i = tuple(bad[0])
        print("gpu", y_gpu[i[0], i[1], :8], "\nref", y[i[0], i[1], :8])
    return ok

if __name__ == "__main__":
    t = time.time()
    run(64, 16, 2, 2, 16, 16, kind="unit")
    run(64, 16, 2, 2, 16, 16)
    run(176, 144, 4, 4, 16, 64)
    run(352, 288, 20, 8, 16, 32)
    run(640, 480, 20, 16, 32, 64)
    run(1920, 1080, 9, 8, 16, 128)
    run(1280, 720, 33, 32, 8, 4, S=2)
    print("elapsed", time.time() - t)
