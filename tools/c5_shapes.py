"""C5-shaped batches (N = 64, I = 2) with the rank profile varied: the FP32 kernel's MAC rate by tile shape."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2109_00626_b200 as ttc  # noqa: E402
import ttgen  # noqa: E402

dev = torch.device("cuda:0")
N, I, B = 64, 2, 16384
rng = np.random.default_rng(7)
for label, choices in (("mix 8-32", [8, 16, 24, 32]), ("all 32", [32]), ("all 16", [16]), ("all 8", [8]),
                       ("8/32", [8, 32])):
    def ranks():
        r = rng.choice(choices, size=(B, N + 1)).astype(np.int32)
        r[:, 0] = r[:, -1] = 1
        return r
    X = ttgen.gaussian_batch(1, 0, 0, 0, ranks(), (I,) * N, "geo")
    Y = ttgen.gaussian_batch(2, 0, 1, 0, ranks(), (I,) * N, "geo")
    XD, YD = ttc.TTDevice.from_batch(X, dev), ttc.TTDevice.from_batch(Y, dev)
    mac, byt = ttc.ttc_pair_cost(XD, YD)
    for _ in range(2):
        ttc.ttc_inner(XD, YD)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ttc.ttc_inner(XD, YD)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 5 / 1e3
    print(f"{label:10s} {B / s / 1e6:6.2f} M pairs/s  {float(np.sum(mac)) / s / 1e12:6.2f} TMAC/s  "
          f"{float(np.sum(byt)) / s / 1e9:7.1f} GB/s")
