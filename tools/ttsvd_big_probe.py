"""Timing probe of the workspace TT-SVD kernel (ttsvd_big.cu) on single unfoldings and Example 2 shapes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2109_00626_b200 as ttc  # noqa: E402

dev = torch.device("cuda", 0)
for dims, B in [((400, 400), 8), ((400, 400), 1), ((20, 8000), 8), ((8000, 20), 8), ((400, 100), 64),
                ((20, 20, 20, 5), 64), ((20, 20, 20, 5, 4), 8), ((200, 200), 8), ((100, 100), 8)]:
    n = int(np.prod(dims))
    x = torch.randn(B * n, device=dev)
    T = ttc.ttc_tt_svd(x, dims, 0.0)
    torch.cuda.synchronize()
    cap = ttc.ttc_tt_svd_capacity(dims)
    cores = torch.zeros(B * cap, device=dev)
    ranks = torch.zeros((B, len(dims) + 1), dtype=torch.int32, device=dev)
    ws = torch.empty(ttc.ttc_tt_svd_workspace(B, dims), dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        ttc.ttc_tt_svd_into(x, dims, 0.0, cores, ranks, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    # sync ints after the B per-tensor double regions: [b * 32] barrier arrivals, [b * 32 + 16] rotating CTA-sweeps
    g = max(min(int(np.prod(dims[:k + 1])), int(np.prod(dims[k + 1:]))) for k in range(len(dims) - 1))
    per = 2 * n + g * g + 2 * g + 80
    sync = ws[8 * B * per:].view(torch.int32).cpu().numpy()
    print(dims, "B", B, f"{e0.elapsed_time(e1) / reps:.3f} ms per call", "ranks", ranks[0].tolist(),
          "barriers", int(sync[0]), "rotating CTA-sweeps", int(sync[16]), flush=True)
