import ctypes, torch, paper_1311_1419_b200 as P, synth
W,H,G,m=176,144,5,507
fe=P.FrameEncoder(W,H,G,m,synth.phi_from_seed(1,m,W*H))
cfg=synth.CONFIGS["C1"].with_(W=W,H=H,G=G,T=40,S=4)
fe.encode_batch(torch.from_numpy(synth.gen_video(cfg)).cuda()); torch.cuda.synchronize(); print("ok")
