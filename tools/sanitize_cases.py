"""Small encodes for compute-sanitizer (memcheck / racecheck / synccheck): every key mode,
block size, folds, partial blocks, ragged GOPs -- kept tiny so the sanitizer finishes quickly."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_1311_1419_b200 as P

cases = [(64, 16, 3, 2, 16, 16), (176, 144, 5, 4, 16, 64), (96, 40, 7, 3, 32, 16), (1280, 24, 5, 4, 8, 4),
         (352, 40, 9, 8, 16, 32), (48, 40, 5, 3, 32, 5)]
ok_all = True
for W, H, T, G, B, M in cases:
    rng = np.random.default_rng(W + H)
    frames = rng.integers(0, 256, size=(1, T, H, W), dtype=np.uint8)
    phi = synth.phi_from_seed(W, M, B * B)
    enc = P.Encoder(W, H, G, B, M, phi)
    fd = torch.from_numpy(frames).cuda()
    for i in range(min(enc.num_candidates(), 3)):
        enc.set_candidate(i)
        out = enc.encode_batch(fd)
        torch.cuda.synchronize()
        y, S = oracle.encode(frames, phi, G, B)
        ok, st = oracle.check_tolerance(out.cpu().numpy(), y, S)
        ok_all &= ok
        print(W, H, T, G, B, M, "plan", i, enc.plan()["key_resident"], ok)
print("ALL_OK" if ok_all else "FAILURES")
