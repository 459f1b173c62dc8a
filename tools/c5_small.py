"""A C5-shaped batch with every bond rank 8 (N = 64, I = 2): the FP32 kernel's per-step fixed cost (ncu target)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2109_00626_b200 as ttc  # noqa: E402
import ttgen  # noqa: E402

dev = torch.device("cuda:0")
N, I, B = 64, 2, 16384
r = np.full((B, N + 1), 8, np.int32)
r[:, 0] = r[:, -1] = 1
X = ttgen.gaussian_batch(1, 0, 0, 0, r, (I,) * N, "geo")
Y = ttgen.gaussian_batch(2, 0, 1, 0, r.copy(), (I,) * N, "geo")
XD, YD = ttc.TTDevice.from_batch(X, dev), ttc.TTDevice.from_batch(Y, dev)
for _ in range(3):
    ttc.ttc_inner(XD, YD)
torch.cuda.synchronize()
print("ok")
