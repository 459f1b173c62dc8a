"""Multi-process (gloo, world size 2 and 3, CPU) coverage of the sharded path's host logic: identical
cost-balanced bounds on every rank, per-rank shard views addressing exactly their pairs, and the padded
all-gather + compaction returning results in pair order.  Oracle results stand in for the kernel output
(no GPU here); the GPU path is covered by test_gpu_inner.py::test_virtual_shards_are_bitwise_equal."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, B, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2109_00626_b200 as ttc
        from paper_2109_00626_b200 import dist as tdist
        import ttgen
        X, Y = ttgen.config_batch(cfg, kind="corr", B=B)
        XD, YD = ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)
        mac, _ = ttc.ttc_pair_cost(XD, YD)
        bounds = tdist.shard_bounds(mac, world)
        # every rank must hold the same plan
        bt = torch.tensor(bounds, dtype=torch.int64)
        allb = [torch.zeros_like(bt) for _ in range(world)]
        dist.all_gather(allb, bt)
        same = all(torch.equal(allb[0], b) for b in allb)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        xs, ys = tdist.shard_view(XD, lo, hi), tdist.shard_view(YD, lo, hi)
        # the shard view addresses exactly pairs lo..hi-1 of the batch (checked through the oracle on its data)
        local = []
        for j in range(hi - lo):
            xc = ttgen.TTBatch(xs.cores, xs.rank_rows(), xs.offsets_np if xs.offsets_np is not None else xs._packed_offsets(), X.dims).train(j)
            yc = ttgen.TTBatch(ys.cores, ys.rank_rows(), ys.offsets_np if ys.offsets_np is not None else ys._packed_offsets(), Y.dims).train(j)
            local.append(oracle.tt_inner(xc, yc)[0])
        full = tdist.gather_results(torch.tensor(local, dtype=torch.float64), bounds)
        if rank == 0:
            want = oracle.tt_inner_batch(X, Y, nthreads=1)
            q.put((same, bounds.tolist(), full.numpy().tolist(), want.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,B", [(2, "C2", 7), (2, "C5", 9), (3, "C5", 10)])
def test_sharded_gather_matches_unsharded(world, cfg, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    same, bounds, full, want = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert same
    assert bounds[0] == 0 and bounds[-1] == B and all(b2 > b1 for b1, b2 in zip(bounds, bounds[1:]))
    assert np.array_equal(np.array(full), np.array(want))   # pair order, bitwise (same oracle, same data)
