"""One small launch of every hot kernel (for compute-sanitizer memcheck / racecheck / synccheck runs; one tool per
gpurun call, B200_PROFILING.md).  Checks nothing numerically (the -m gpu tests do); exits 0 when every call returns."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2109_00626_b200 as ttc  # noqa: E402
import ttgen  # noqa: E402

dev = torch.device("cuda:0")


def inner(cfg, B, kind="corr", env=None):
    if env:
        os.environ["TTC_KERNEL"] = env
    X, Y = ttgen.config_batch(cfg, kind=kind, B=B)
    out = ttc.ttc_inner(ttc.TTDevice.from_batch(X, dev), ttc.TTDevice.from_batch(Y, dev))
    torch.cuda.synchronize()
    os.environ.pop("TTC_KERNEL", None)
    print(cfg, B, env or "default", float(out[0]))


inner("C1", 1)                  # inner_small_kernel
inner("C2", 6)                  # inner_r16_kernel
inner("C4", 6)                  # inner_r64tc_kernel (tcgen05, TMA)
inner("C4", 5, env="mmasync")   # inner_r64_kernel
inner("C5", 12)                 # inner_ffma_kernel
inner("C2", 5, env="fast")      # inner_tc_kernel
inner("C5", 3, env="generic")   # inner_generic_kernel
c = ttgen.CONFIGS["C3"]
X, Y = ttgen.config_batch("C3", B=3)
XD, YD = ttc.TTDevice.from_batch(X, dev), ttc.TTDevice.from_batch(Y, dev)
plan = ttc.ttc_contract_plan_create(XD, YD, c["x_modes"], c["y_modes"])
cores, _, _ = ttc.ttc_contract(plan, XD, YD)   # contract_kernel
sp = ttc.ttc_splice_plan_create(XD, YD, 1, 1)
zc, zr, zo = ttc.ttc_contract(sp, XD, YD)      # splice_kernel
torch.cuda.synchronize()
R = ttgen.uniform_ranks(3, 4, 5)
T = ttgen.gaussian_batch(1, 0, 0, 0, R, (6, 5, 4, 3))
dense = ttc.ttc_reconstruct(ttc.TTDevice.from_batch(T, dev))   # reconstruct_kernel
rng = np.random.default_rng(0)
d = torch.from_numpy(rng.standard_normal(2 * 6 * 5 * 4).astype(np.float32)).to(dev)
S = ttc.ttc_tt_svd(d, (6, 5, 4), 0.0)                           # ttsvd pipeline
torch.cuda.synchronize()
print("sanitize cases ok", float(cores[0]), float(zc[0]), float(dense[0]))
