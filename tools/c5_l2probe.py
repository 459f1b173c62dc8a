"""C5 launch timing: one launch per host sync vs back-to-back launches (same batch)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_00626_b200 as ttc
import ttgen
dev = torch.device("cuda:0")
B = 65536
X, Y = ttgen.config_batch("C5", "iid", 0, B, device=dev)
XD, YD = ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)
order = ttc.ttc_cost_order(XD, YD)
out = torch.empty(B, device=dev)
for mode in ("synced", "b2b", "synced", "b2b"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
    torch.cuda.synchronize()
    for it in range(6):
        ev[2 * it].record()
        ttc.ttc_inner(XD, YD, out=out, order=order)
        ev[2 * it + 1].record()
        if mode == "synced":
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    ts = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(6)]
    print(mode, " ".join(f"{t:.2f}" for t in ts), "ms")
