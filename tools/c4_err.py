"""C4 self / correlated pairs: relative error distribution of the tcgen05 kernel against the fp64 oracle
(margin below the 1e-5 |oracle| gate of tests/test_gpu_inner.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, ttgen
import paper_2109_00626_b200 as ttc
dev = "cuda:0"
for N in (16, 21):
    for kind in ("self", "corr"):
        B = 48
        X, Y = ttgen.make_pair(kind, 5 + N, 4, 0, ttgen.uniform_ranks(B, N, 64), (4,) * N, device=dev)
        got = ttc.ttc_inner(ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)).cpu().numpy().astype(np.float64)
        rel = []
        for b in range(B):
            want, _ = oracle.tt_inner(X.train(b), Y.train(b))
            rel.append((got[b] - want) / abs(want))
        rel = np.array(rel)
        print(f"N={N} {kind}: max |rel| {np.abs(rel).max():.2e}  mean rel {rel.mean():+.2e}")
