import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, ttgen, paper_2109_00626_b200 as ttc
cases = [((7,), [1, 1], [1, 1]), ((2, 2), [1, 8, 1], [1, 8, 1]), ((2, 2), [1, 16, 1], [1, 8, 1]),
         ((2, 2, 2), [1, 8, 8, 1], [1, 8, 8, 1]), ((2, 2, 2), [1, 24, 16, 1], [1, 8, 32, 1]),
         ((3, 2), [1, 4, 1], [1, 4, 1]), ((10,) * 5, [1, 4, 4, 4, 4, 1], [1, 4, 4, 4, 4, 1])]
cases = [((2, 2, 2, 2), [1, 8, 32, 8, 1], [1, 32, 8, 32, 1]), ((2, 2, 2), [1, 32, 8, 1], [1, 8, 32, 1]),
         ((2, 2, 2), [1, 8, 32, 1], [1, 32, 8, 1]), ((2, 2), [1, 32, 1], [1, 8, 1]), ((2,) * 6, [1, 8, 32, 8, 32, 8, 1], [1, 32, 8, 32, 8, 32, 1])]
for dims, rx, ry in cases:
    B = 3
    xr = np.tile(np.array(rx, np.int32), (B, 1)); yr = np.tile(np.array(ry, np.int32), (B, 1))
    X = ttgen.gaussian_batch(1, 0, 0, 0, xr, dims, "geo"); Y = ttgen.gaussian_batch(1, 0, 1, 0, yr, dims, "geo")
    XD, YD = ttc.TTDevice.from_batch(X, "cuda"), ttc.TTDevice.from_batch(Y, "cuda")
    got = ttc.ttc_inner(XD, YD).cpu().numpy()
    os.environ["TTC_KERNEL"] = "generic"; gen = ttc.ttc_inner(XD, YD).cpu().numpy(); del os.environ["TTC_KERNEL"]
    want = [oracle.tt_inner(X.train(b), Y.train(b))[0] for b in range(B)]
    print(dims, rx, ry, "wpp", got, "gen", gen, "oracle", np.array(want))

for B in (1, 3, 16):
    X, Y = ttgen.config_batch("C5", kind="corr", B=B)
    XD, YD = ttc.TTDevice.from_batch(X, "cuda"), ttc.TTDevice.from_batch(Y, "cuda")
    got = ttc.ttc_inner(XD, YD).cpu().numpy()
    os.environ["TTC_KERNEL"] = "generic"; gen = ttc.ttc_inner(XD, YD).cpu().numpy(); del os.environ["TTC_KERNEL"]
    print("C5 corr B", B, "wpp", got[:4], "gen", gen[:4])
