import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, ttgen, paper_2109_00626_b200 as ttc
X, Y = ttgen.config_batch("C5", kind="corr", B=1)
XD, YD = ttc.TTDevice.from_batch(X, "cuda"), ttc.TTDevice.from_batch(Y, "cuda")
print("ranks", X.ranks[0][:12], XD.ranks_np is not None, XD.offsets_np)
got = ttc.ttc_inner(XD, YD).cpu().numpy()
torch.cuda.synchronize()
print("got", got, "want", oracle.tt_inner(X.train(0), Y.train(0))[0])
