"""GPU parity for ttc_inner (through the C ABI) against the fp64 oracle, on the BASELINE.json configs.

Error measure (BASELINE.json north_star): |gpu - oracle| / (||X||_F ||Y||_F) <= 1e-4, with the norms from
the oracle.  Because that bound is nearly vacuous for iid pairs (|<X,Y>| / (||X|| ||Y||) ~ 1e-5 .. 1e-10,
DESIGN.md reading R12), parity is gated on non-vacuous batches of the same shapes: self pairs (Y = X),
correlated pairs, integer cores (bitwise exact) and tagged rank-1 pairs (bitwise exact, order check); on
iid batches the error must also be far below |oracle| itself."""
import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
import ttgen

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL = 1e-4


def _run(X, Y):
    out = ttc.ttc_inner(ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV))
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _check(X, Y, got, idx, kind):
    worst = 0.0
    for b in idx:
        xc, yc = X.train(b), Y.train(b)
        want, _ = oracle.tt_inner(xc, yc)
        nrm = oracle.normaliser(xc, yc)
        err = abs(got[b] - want) / nrm
        worst = max(worst, err)
        assert err <= TOL, f"{kind} pair {b}: normalised error {err:.3e}"
        if kind in ("self", "corr"):
            assert abs(want) / nrm > 0.5            # the control is not vacuous here
            assert abs(got[b] - want) <= 1e-5 * abs(want)
        if kind == "iid" and abs(want) / nrm > 1e-7:
            assert abs(got[b] - want) <= 1e-2 * abs(want), f"iid pair {b}: {got[b]} vs {want}"
    return worst


def _sample(B, k, seed=0):
    if B <= k:
        return list(range(B))
    rng = np.random.default_rng(seed)
    return sorted(set([0, B - 1] + list(rng.choice(B, k - 2, replace=False))))


@pytest.mark.parametrize("kind", ["iid", "self", "corr"])
def test_c1(kind):
    X, Y = ttgen.config_batch("C1", kind=kind)
    got = _run(X, Y)
    _check(X, Y, got, [0], kind)


@pytest.mark.parametrize("kind", ["iid", "self", "corr"])
def test_c2_small_all_pairs(kind):
    """C2 shape, 67 pairs (several waves' worth of CTAs per SM is not needed here: a ragged batch)."""
    X, Y = ttgen.config_batch("C2", kind=kind, B=67)
    got = _run(X, Y)
    _check(X, Y, got, range(67), kind)


def test_c2_full_size_sampled():
    """BASELINE.json configs[1] at full size (4096 pairs, the bench workload), sampled pairs vs the oracle."""
    X, Y = ttgen.config_batch("C2", kind="iid", device=DEV)
    got = _run(X, Y)
    _check(X, Y, got, _sample(X.B, 24), "iid")
    Xs, Ys = ttgen.config_batch("C2", kind="self", device=DEV)
    got = _run(Xs, Ys)
    _check(Xs, Ys, got, _sample(Xs.B, 16, 1), "self")


def _run_sentinel(X, Y, order=False):
    """ttc_inner into a NaN-filled output on the device: every pair must be written (finite afterwards)."""
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    out = torch.full((X.B,), float("nan"), dtype=torch.float32, device=DEV)
    ttc.ttc_inner(XD, YD, out=out, order=ttc.ttc_cost_order(XD, YD) if order else None)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got)), f"{int(np.sum(~np.isfinite(got)))} of {X.B} pairs never written"
    return got, XD, YD


@pytest.mark.parametrize("B", [8192])
def test_c4_full_batch(B):
    """BASELINE.json configs[3] (R = 64) at its full single-GPU batch (8,192 pairs), the bench's launch: iid pairs
    and the non-vacuous self / correlated controls, 64 sampled pairs each (first and last pair included)."""
    for kind, k in (("self", 64), ("corr", 64), ("iid", 16)):
        X, Y = ttgen.config_batch("C4", kind=kind, B=B, device=DEV)
        got, _, _ = _run_sentinel(X, Y)
        _check(X, Y, got, _sample(X.B, k, 7), kind)
        del X, Y
        torch.cuda.empty_cache()


@pytest.mark.parametrize("B,kinds", [(8192, ("self", "corr", "iid")), (65536, ("corr",))])
def test_c5_full_batch(B, kinds):
    """BASELINE.json configs[4] (ranks {8..32}, N = 64, I = 2) at one 8-GPU shard (8,192 pairs) and at the full
    65,536-pair batch on one GPU, with the cost-descending work list the bench uses (ttc_inner_ordered): the
    first and last tickets (the most and least expensive pairs) and the first / last pair indices are among
    >= 64 sampled pairs on non-vacuous self / correlated batches; the ordered and natural-order launches agree
    bitwise on every pair; a NaN sentinel shows that every pair was written."""
    for kind in kinds:
        X, Y = ttgen.config_batch("C5", kind=kind, B=B, device=DEV)
        got, XD, YD = _run_sentinel(X, Y, order=True)
        order = ttc.ttc_cost_order(XD, YD).host
        idx = sorted(set(_sample(X.B, 64, 3)) | {int(order[0]), int(order[1]), int(order[-2]), int(order[-1])})
        _check(X, Y, got, idx, kind)
        nat, _, _ = _run_sentinel(X, Y, order=False)
        assert np.array_equal(nat.view(np.uint64), got.view(np.uint64))
        del X, Y, XD, YD
        torch.cuda.empty_cache()


def test_c5_small_corr():
    X, Y = ttgen.config_batch("C5", kind="corr", B=256, device=DEV)
    got = _run(X, Y)
    _check(X, Y, got, _sample(X.B, 16, 2), "corr")


@pytest.mark.parametrize("cfg,B", [("C1", 1), ("C2", 33), ("C4", 8), ("C5", 16)])
def test_integer_cores_bitwise(cfg, B):
    """Cores in {-1, 0, 1}: when every partial sum is an integer below 2^24 (checked by running the oracle on
    |X|, |Y|, an upper bound for any summation order), fp32 is exact and the GPU must equal the oracle bitwise."""
    c = ttgen.CONFIGS[cfg]
    if cfg == "C5":
        xr = ttgen.random_ranks(1, 5, 0, 0, B, c["N"], c["rank_choices"])
        yr = ttgen.random_ranks(1, 5, 1, 0, B, c["N"], c["rank_choices"])
        dims = (c["I"],) * c["N"]
    else:
        xr = yr = ttgen.uniform_ranks(B, c["N"], c["R"])
        dims = (c["I"],) * c["N"]
    density = {"C1": 0.3, "C2": 0.05, "C4": 0.01, "C5": 0.1}[cfg]
    X, Y = ttgen.make_pair("int", 3, 9, 0, xr, dims, yr, density=density)
    got = _run(X, Y)
    exact = 0
    for b in range(B):
        xc, yc = X.train(b), Y.train(b)
        bound, _ = oracle.tt_inner([np.abs(a) for a in xc], [np.abs(a) for a in yc])
        if bound >= 2 ** 24:
            continue
        want, _ = oracle.tt_inner(xc, yc)
        assert got[b] == want, f"pair {b}: {got[b]} != {want}"
        exact += 1
    assert exact >= 1


def test_tagged_order():
    """<X_b, Y_b> = b exactly: results come back in pair order (C2 shape, 1000 pairs)."""
    B = 1000
    X, Y = ttgen.make_pair("tagged", 0, 2, 0, ttgen.uniform_ranks(B, 8, 16), (16,) * 8)
    got = _run(X, Y)
    assert np.array_equal(got, np.arange(B, dtype=np.float64))


def test_determinism_and_exact_scaling():
    X, Y = ttgen.config_batch("C2", kind="iid", B=64)
    a, b = _run(X, Y), _run(X, Y)
    assert np.array_equal(a, b)
    # scaling core 3 of every X by 2 scales every result by exactly 2
    X2 = ttgen.TTBatch(X.cores.clone(), X.ranks, X.offsets, X.dims)
    sz = [16 * 16 * 16] * 6
    start = 256 + sz[0] * 2  # core index 3 (0-based) starts after cores 0 (256), 1, 2
    per = int(X.offsets[1])
    for j in range(64):
        X2.cores[j * per + start: j * per + start + 4096] *= 2
    c = _run(X2, Y)
    assert np.array_equal(c, 2 * a)


def test_virtual_shards_are_bitwise_equal():
    """Sharding the batch (ttc_partition) and running the shards one after the other gives bitwise the
    unsharded result: per-pair work is independent of the split (multi-GPU correctness)."""
    X, Y = ttgen.config_batch("C5", kind="iid", B=200)
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    full = ttc.ttc_inner(XD, YD).cpu().numpy()
    mac, _ = ttc.ttc_pair_cost(XD, YD)
    for k in (2, 4, 8):
        bounds = ttc.ttc_partition(mac, k)
        parts = []
        for j in range(k):
            s, e = int(bounds[j]), int(bounds[j + 1])
            xs = ttc.TTDevice(X.cores.to(DEV), X.dims, ranks=X.ranks[s:e], offsets=X.offsets[s:e])
            ys = ttc.TTDevice(Y.cores.to(DEV), Y.dims, ranks=Y.ranks[s:e], offsets=Y.offsets[s:e])
            parts.append(ttc.ttc_inner(xs, ys).cpu().numpy())
        assert np.array_equal(np.concatenate(parts), full)


def test_edge_shapes():
    """N = 1 (a dot product), I = 1 modes, rank-1 trains, unequal X / Y ranks, odd sizes, large I."""
    rng = np.random.default_rng(5)
    for dims, rx, ry in [((7,), [1, 1], [1, 1]),
                         ((1, 1, 1), [1, 3, 2, 1], [1, 1, 5, 1]),
                         ((3, 1, 4, 2), [1, 5, 7, 3, 1], [1, 2, 9, 4, 1]),
                         ((300, 2), [1, 3, 1], [1, 5, 1]),
                         ((5, 5, 5), [1, 128, 128, 1], [1, 128, 128, 1]),
                         ((2,) * 10, [1] + [33] * 9 + [1], [1] + [31] * 9 + [1])]:
        B = 5
        xr = np.tile(np.array(rx, np.int32), (B, 1))
        yr = np.tile(np.array(ry, np.int32), (B, 1))
        X = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, xr, dims, "geo")
        Y = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 1, 0, yr, dims, "geo")
        got = _run(X, Y)
        _check(X, Y, got, range(B), "edge")
        Xs = ttgen.TTBatch(X.cores.clone(), X.ranks, X.offsets, X.dims)
        got = _run(Xs, Xs)
        _check(Xs, Xs, got, range(B), "self")


@pytest.mark.parametrize("dims", [(16, 16), (4, 16, 16), (16, 16, 16), (3, 5, 16, 7, 2), (13, 9, 11, 1),
                                  (1, 8, 1, 8, 1, 8), (6, 12, 16, 10, 14, 4, 2), (20, 20, 20), (3, 24, 5, 26, 2)])
def test_uniform_rank16_shapes(dims):
    """The uniform rank-16 kernel (first / last cores from L2, interior cores through the TMA ring) on mixed
    mode sizes: fewer slices than warps, odd slice counts, I = 1 cores, boundary I not a multiple of 4, a single
    interior core (N = 3), N = 2 (no interior core: served by another kernel), and mode sizes 17..26 (2 CTAs per
    SM instead of 3; with I_1 = I_N = 20 the boundary warp reads its cores from global memory, no scratch)."""
    rng = np.random.default_rng(sum(dims))
    B = 37
    N = len(dims)
    r = np.tile(np.array([1] + [16] * (N - 1) + [1], np.int32), (B, 1))
    X = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, r, dims, "geo")
    Y = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 1, 0, r, dims, "geo")
    got = _run(X, Y)
    _check(X, Y, got, range(B), "edge")
    got = _run(X, X)
    _check(X, X, got, range(B), "self")


@pytest.mark.parametrize("variant", ["generic", "fast", "ffma", "small"])
def test_kernel_variants_agree(monkeypatch, variant):
    """Every tt_inner kernel (default dispatch vs TTC_KERNEL=generic / fast / ffma / small) agrees within fp32 rounding."""
    for cfg, B in (("C2", 16), ("C5", 24), ("C1", 1), ("C4", 2)):
        X, Y = ttgen.config_batch(cfg, kind="corr", B=B)
        ref = _run(X, Y)
        monkeypatch.setenv("TTC_KERNEL", variant)
        got = _run(X, Y)
        monkeypatch.delenv("TTC_KERNEL")
        for b in range(B):
            nrm = oracle.normaliser(X.train(b), Y.train(b))
            assert abs(ref[b] - got[b]) <= 1e-5 * nrm, (cfg, b, ref[b], got[b])


def test_sharded_inner_nccl_single_rank():
    """dist.sharded_inner over an NCCL group (world size 1 on this box): partition + shard views +
    all_gather_into_tensor + compaction reproduce the unsharded call bitwise."""
    import os
    import torch.distributed as dist
    from paper_2109_00626_b200 import dist as tdist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        X, Y = ttgen.config_batch("C5", kind="iid", B=40)
        XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
        full = ttc.ttc_inner(XD, YD)
        got, bounds = tdist.sharded_inner(XD, YD)
        torch.cuda.synchronize()
        assert list(bounds) == [0, 40]
        assert torch.equal(got, full)
        # shard views of a 4-way plan, run one after another, gathered by hand
        mac, _ = ttc.ttc_pair_cost(XD, YD)
        b4 = tdist.shard_bounds(mac, 4)
        parts = [ttc.ttc_inner(tdist.shard_view(XD, int(b4[r]), int(b4[r + 1])),
                               tdist.shard_view(YD, int(b4[r]), int(b4[r + 1]))) for r in range(4)]
        assert torch.equal(torch.cat(parts), full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", range(6))
def test_ffma_rank_mult8_shapes(case):
    """The FP32 warp-per-pair kernel (interior ranks multiples of 8, <= 32): random rank profiles over every
    {8, 16, 24, 32} combination, mixed and odd mode sizes (boundary cores of odd size are copied without
    cp.async), N = 2 (no interior step), N = 3, uniform ranks (ranks_host NULL), and ragged batch sizes."""
    rng = np.random.default_rng(100 + case)
    dims = [(2, 2, 2, 2, 2, 2), (3, 1, 5, 2, 7), (2, 2), (4, 3, 2), (2,) * 24, (1, 2, 3, 4, 5, 6, 7)][case]
    B = [1, 5, 33, 130, 517, 64][case]
    N = len(dims)
    def ranks():
        r = rng.choice([8, 16, 24, 32], size=(B, N + 1)).astype(np.int32)
        r[:, 0] = 1
        r[:, -1] = 1
        return r
    X = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, ranks(), dims, "geo")
    Y = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 1, 0, ranks(), dims, "geo")
    got = _run(X, Y)
    _check(X, Y, got, _sample(B, 40, case), "edge")
    got = _run(X, X)
    _check(X, X, got, _sample(B, 40, case + 1), "self")
    # uniform ranks through the ranks_host == NULL path
    R = [8, 16, 24, 32, 24, 8][case]
    ur = np.tile(np.array([1] + [R] * (N - 1) + [1], np.int32), (B, 1))
    Xu = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, ur, dims, "geo")
    got = _run(Xu, Xu)
    _check(Xu, Xu, got, _sample(B, 24, case + 2), "self")


def test_cost_ordered_inner_is_bitwise_equal():
    """ttc_inner_ordered (cost-descending work list) returns exactly ttc_inner's values, pair by pair."""
    for cfg, B in (("C5", 300), ("C2", 40), ("C1", 3), ("C4", 6)):
        X, Y = ttgen.config_batch(cfg, kind="corr", B=B)
        XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
        ref = ttc.ttc_inner(XD, YD).cpu().numpy()
        order = ttc.ttc_cost_order(XD, YD)
        assert sorted(order.host.tolist()) == list(range(B))
        got = ttc.ttc_inner(XD, YD, order=order).cpu().numpy()
        assert np.array_equal(ref.view(np.uint32), got.view(np.uint32)), cfg


@pytest.mark.parametrize("N,B", [(3, 1), (3, 149), (4, 2), (16, 150), (16, 297), (21, 37)])
def test_r64_tcgen05_kernel(monkeypatch, N, B):
    """The tcgen05 rank-64 kernel (inner_r64tc.cu: uniform R = 64, I_n = 4, packed) on one interior step (N = 3),
    batches below / just above / about twice the CTA count (static pair assignment), and long chains (N = 21):
    self and correlated pairs against the oracle (1e-5 |oracle| gate) and against the legacy mma.sync kernel
    (TTC_KERNEL=mmasync) within fp32 rounding."""
    r = ttgen.uniform_ranks(B, N, 64)
    for kind in ("self", "corr"):
        X, Y = ttgen.make_pair(kind, 11 + N, 4, 0, r, (4,) * N, device=DEV)
        got = _run(X, Y)
        _check(X, Y, got, _sample(B, 12, N), kind)
        monkeypatch.setenv("TTC_KERNEL", "mmasync")
        ref = _run(X, Y)
        monkeypatch.delenv("TTC_KERNEL")
        for b in range(B):
            assert abs(got[b] - ref[b]) <= 2e-5 * abs(ref[b]), (kind, b, got[b], ref[b])


def test_graph_replay_and_concurrent_streams_are_reentrant():
    """No kernel keeps global state (ttc.h: re-entrant): ttc_inner captured in a CUDA graph and replayed gives the
    eager result bitwise, and the C5 kernel (formerly handing out pairs from global ticket counters) run on two
    streams at once, twice over, gives bitwise the single-stream result for both batches."""
    X, Y = ttgen.config_batch("C1", kind="corr")
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    eager = ttc.ttc_inner(XD, YD).clone()
    s = torch.cuda.Stream()
    out = torch.empty_like(eager)
    with torch.cuda.stream(s):
        ttc.ttc_inner(XD, YD, out=out, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ttc.ttc_inner(XD, YD, out=out, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    batches = [ttgen.config_batch("C5", kind="corr", b0=b0, B=300, device=DEV) for b0 in (0, 300)]
    devs = [(ttc.TTDevice.from_batch(Xb), ttc.TTDevice.from_batch(Yb)) for Xb, Yb in batches]
    ref = [ttc.ttc_inner(xd, yd).clone() for xd, yd in devs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.full((300,), float("nan"), device=DEV) for _ in range(2)]
    for rep in range(2):
        for k in range(2):
            ttc.ttc_inner(devs[k][0], devs[k][1], out=outs[k], stream=streams[k])
        torch.cuda.synchronize()
        for k in range(2):
            assert torch.equal(outs[k], ref[k]), (rep, k)


@pytest.mark.parametrize("case", ["c5", "gaps", "dims", "i1", "i3"])
def test_ffma_tma_staging_matches_cp_async(monkeypatch, case):
    """The FP32 kernel's two staging paths (TMA tensor boxes with zero-filled padding, TTC_FFMA_TMA=1, vs 16-byte
    cp.async, TTC_FFMA_TMA=0) stage the same values, so the results are bitwise equal: C5 correlated pairs; trains
    at gapped offsets (16-byte steps) with the last core ending at the buffer's end; mixed interior mode sizes
    (several G run lengths).  Both paths are also checked against the oracle."""
    rng = np.random.default_rng({"c5": 1, "gaps": 2, "dims": 3, "i1": 4, "i3": 5}[case])
    if case == "c5":
        X, Y = ttgen.config_batch("C5", kind="corr", B=300)
        XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    else:
        dims = {"gaps": (2,) * 12, "dims": (2, 3, 2, 3, 2, 2),   # 8 run lengths: a full map table
                "i1": (2, 1, 1, 1, 1, 2), "i3": (1, 3, 3, 3, 1)}[case]   # G runs of Ga (I = 1) / 3 Ga floats
        B, N = 97, len(dims)
        def ranks():
            r = rng.choice([8, 16, 24, 32], size=(B, N + 1)).astype(np.int32)
            r[:, 0] = r[:, -1] = 1
            return r
        X = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, ranks(), dims, "geo")
        Y = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 1, 0, ranks(), dims, "geo")
        def gapped(T):
            sizes = np.diff(np.append(T.offsets, T.cores.numel()))
            gaps = 4 * rng.integers(0, 5, size=B)
            offs = np.zeros(B, np.int64)
            pos = 0
            for b in range(B):
                pos += int(gaps[b])
                offs[b] = pos
                pos += int(sizes[b])
            buf = torch.full((pos,), float("nan"))   # gaps hold NaN: any stray read poisons a result
            for b in range(B):
                buf[offs[b]:offs[b] + sizes[b]] = T.cores[T.offsets[b]:T.offsets[b] + sizes[b]]
            return ttc.TTDevice(buf.to(DEV), T.dims, ranks=T.ranks, offsets=offs)
        XD, YD = gapped(X), gapped(Y)
    res = {}
    for t in ("0", "1"):
        monkeypatch.setenv("TTC_KERNEL", "ffma")
        monkeypatch.setenv("TTC_FFMA_TMA", t)
        res[t] = ttc.ttc_inner(XD, YD).cpu().numpy()
    monkeypatch.delenv("TTC_FFMA_TMA")
    monkeypatch.delenv("TTC_KERNEL")
    assert np.array_equal(res["0"], res["1"])
    _check(X, Y, res["1"].astype(np.float64), _sample(X.ranks.shape[0], 24, 7), "corr" if case == "c5" else "edge")
