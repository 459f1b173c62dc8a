"""Write-only, read-only and copy HBM bandwidth with torch ops (context for write-bound kernels: C3, R1).
Usage: python tools/hbm_rw.py  -> one JSON line (GB/s, best of 10, CUDA events)."""
import json

import torch

n = 1 << 30  # 1 Gi fp32 = 4 GiB
a = torch.empty(n, device="cuda", dtype=torch.float32)
b = torch.empty(n, device="cuda", dtype=torch.float32)
a.fill_(1.0)


def best(fn, nbytes):
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return nbytes / min(ts) / 1e9


out = {"write_gbs": best(lambda: b.fill_(2.0), 4 * n),
       "read_gbs": best(lambda: a.sum(), 4 * n),
       "copy_gbs": best(lambda: b.copy_(a), 8 * n)}
print(json.dumps(out))
