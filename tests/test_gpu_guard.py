"""Out-of-bounds checks without compute-sanitizer (closed on this GPU pool: "runs under it have left GPUs needing a
reset"): every train sits between NaN guard bands (NaN-filled gaps between the trains of an offset batch, NaN before
and after a packed batch), every output between NaN sentinels.  A kernel that reads outside its trains picks up a
NaN and returns a non-finite value; one that writes outside its output range overwrites a sentinel.  Results must
also equal the plain (packed, unguarded) call bitwise: the layout of the batch does not change any sum."""
import numpy as np
import pytest
import torch

import paper_2109_00626_b200 as ttc
import ttgen

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GUARD = 1024   # floats of NaN before / after a batch; gaps between trains are 64 floats


def _guarded_copy(T: ttgen.TTBatch, gaps: bool):
    """(TTDevice over a NaN-guarded copy of batch T, the backing buffer)."""
    rows = T.ranks
    sizes = [ttgen.train_elems(rows[b], T.dims) for b in range(T.B)]
    gap = 64 if gaps else 0
    offs = np.zeros(T.B, np.int64)
    pos = GUARD
    for b in range(T.B):
        offs[b] = pos
        pos += sizes[b] + gap
    buf = torch.full((pos + GUARD,), float("nan"), dtype=torch.float32, device=DEV)
    src = T.cores.to(DEV)
    for b in range(T.B):
        buf[offs[b]: offs[b] + sizes[b]] = src[int(T.offsets[b]): int(T.offsets[b]) + sizes[b]]
    if gaps:
        return ttc.TTDevice(buf, T.dims, ranks=rows, offsets=offs), buf
    view = buf[GUARD: GUARD + sum(sizes)]   # packed, NaN on both sides of the region
    return ttc.TTDevice(view, T.dims, ranks=rows, offsets=offs - GUARD), buf


def _sentinel_out(n):
    full = torch.full((n + 64,), float("nan"), dtype=torch.float32, device=DEV)
    return full, full[32: 32 + n]


@pytest.mark.parametrize("cfg,B,env,gaps", [("C1", 1, None, True), ("C2", 7, None, False), ("C2", 7, "fast", True),
                                            ("C4", 9, None, False), ("C4", 5, "mmasync", True), ("C5", 21, None, True),
                                            ("C5", 6, "generic", True), ("C2", 3, "small", True)])
def test_inner_reads_and_writes_stay_in_bounds(monkeypatch, cfg, B, env, gaps):
    X, Y = ttgen.config_batch(cfg, kind="corr", B=B)
    ref = ttc.ttc_inner(ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV))
    if env:
        monkeypatch.setenv("TTC_KERNEL", env)
        ref = ttc.ttc_inner(ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV))
    XG, _bx = _guarded_copy(X, gaps)
    YG, _by = _guarded_copy(Y, gaps)
    full, out = _sentinel_out(B)
    ttc.ttc_inner(XG, YG, out=out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    f = full.cpu().numpy()
    assert np.all(np.isfinite(got)), "a kernel read outside its trains"
    assert np.all(np.isnan(f[:32])) and np.all(np.isnan(f[32 + B:])), "a kernel wrote outside out[0:B]"
    assert np.array_equal(got.view(np.uint32), ref.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("op", ["contract", "splice", "reconstruct"])
def test_contract_splice_reconstruct_stay_in_bounds(op):
    c = ttgen.CONFIGS["C3"]
    X, Y = ttgen.config_batch("C3", B=3)
    XG, _bx = _guarded_copy(X, True)
    YG, _by = _guarded_copy(Y, True)
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    if op == "reconstruct":
        R = ttgen.uniform_ranks(3, 4, 5)
        T = ttgen.gaussian_batch(1, 0, 0, 0, R, (6, 5, 4, 3))
        TG, _bt = _guarded_copy(T, True)
        ref = ttc.ttc_reconstruct(ttc.TTDevice.from_batch(T, DEV))
        full, out = _sentinel_out(ref.numel())
        ttc.ttc_reconstruct(TG, out=out)
    else:
        mk = (lambda a, b: ttc.ttc_contract_plan_create(a, b, c["x_modes"], c["y_modes"])) if op == "contract" else \
            (lambda a, b: ttc.ttc_splice_plan_create(a, b, 1, 1))
        ref, _, _ = ttc.ttc_contract(mk(XD, YD), XD, YD)
        plan = mk(XG, YG)
        full, out = _sentinel_out(plan.total)
        ttc.ttc_contract(plan, XG, YG, out=out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    f = full.cpu().numpy()
    n = got.size
    assert np.all(np.isfinite(got)), f"{op}: read outside the trains"
    assert np.all(np.isnan(f[:32])) and np.all(np.isnan(f[32 + n:])), f"{op}: wrote outside its output"
    assert np.array_equal(got.view(np.uint32), ref.cpu().numpy().view(np.uint32))


def _guarded_ws(nbytes):
    """(full buffer, the workspace view): 4 KB of 0xFF guard bytes before and after the caller's workspace."""
    full = torch.full((nbytes + 8192,), 255, dtype=torch.uint8, device=DEV)
    return full, full[4096: 4096 + nbytes]


def test_reconstruct_beyond_shared_memory_stays_in_bounds():
    """The workspace GEMM chain (reconstruct_big.cu): trains between NaN guard bands, output between NaN sentinels,
    workspace between guard bytes; result bitwise equal to the plain call."""
    r = np.tile(np.array([1, 7, 9, 1], np.int32), (3, 1))
    r[1, 1:-1] = [6, 8]
    T = ttgen.gaussian_batch(5, 0, 0, 0, r, (7, 2000, 9), "geo")
    ref = ttc.ttc_reconstruct(ttc.TTDevice.from_batch(T, DEV), [2, 3, 1])
    TG, _bt = _guarded_copy(T, True)
    nb = ttc.ttc_reconstruct_workspace(TG, [2, 3, 1])
    assert nb > 0
    wfull, ws = _guarded_ws(nb)
    full, out = _sentinel_out(ref.numel())
    ttc.ttc_reconstruct(TG, [2, 3, 1], out=out, workspace=ws)
    torch.cuda.synchronize()
    got, f, w = out.cpu().numpy(), full.cpu().numpy(), wfull.cpu().numpy()
    n = got.size
    assert np.all(np.isfinite(got)), "read outside the trains"
    assert np.all(np.isnan(f[:32])) and np.all(np.isnan(f[32 + n:])), "wrote outside the output"
    assert np.all(w[:4096] == 255) and np.all(w[4096 + nb:] == 255), "wrote outside the workspace"
    assert np.array_equal(got.view(np.uint32), ref.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("dims,perm", [((20, 20, 20, 5), None), ((5, 20, 20, 20), [2, 3, 4, 1]), ((70, 70), None)])
def test_tt_svd_beyond_shared_memory_stays_in_bounds(dims, perm):
    """The workspace TT-SVD (ttsvd_big.cu): dense batch between NaN guards, cores / ranks between sentinels, the
    workspace between guard bytes; cores and ranks bitwise equal to the plain call."""
    B = 3
    n = int(np.prod(dims))
    rng = np.random.default_rng(n)
    dense = torch.from_numpy(rng.standard_normal(B * n).astype(np.float32)).to(DEV)
    ref = ttc.ttc_tt_svd(dense, dims, 0.1, perm=perm)
    cap = ttc.ttc_tt_svd_capacity(dims, perm)
    dfull = torch.full((B * n + 2 * GUARD,), float("nan"), dtype=torch.float32, device=DEV)
    dfull[GUARD: GUARD + B * n] = dense
    cfull, cores = _sentinel_out(B * cap)
    rfull = torch.full((B * (len(dims) + 1) + 64,), -7, dtype=torch.int32, device=DEV)
    ranks = rfull[32: 32 + B * (len(dims) + 1)].view(B, len(dims) + 1)
    nb = ttc.ttc_tt_svd_workspace(B, dims, perm)
    wfull, ws = _guarded_ws(nb)
    ttc.ttc_tt_svd_into(dfull[GUARD: GUARD + B * n], dims, 0.1, cores, ranks, perm=perm, workspace=ws)
    torch.cuda.synchronize()
    rk = ranks.cpu().numpy()
    assert np.array_equal(rk, ref.rank_rows()), "ranks differ from the plain call"
    c, cf, rf, w = cores.cpu().numpy(), cfull.cpu().numpy(), rfull.cpu().numpy(), wfull.cpu().numpy()
    assert np.all(np.isnan(cf[:32])) and np.all(np.isnan(cf[32 + B * cap:])), "wrote outside the cores"
    assert np.all(rf[:32] == -7) and np.all(rf[32 + B * (len(dims) + 1):] == -7), "wrote outside the ranks"
    assert np.all(w[:4096] == 255) and np.all(w[4096 + nb:] == 255), "wrote outside the workspace"
    refc = ref.cores.cpu().numpy()
    for b in range(B):   # the written part of each train: finite (no read outside the dense batch) and bitwise equal
        used = sum(int(rk[b][k]) * (ref.dims_np[k]) * int(rk[b][k + 1]) for k in range(len(dims)))
        seg = c[b * cap: b * cap + used]
        assert np.all(np.isfinite(seg)), "read outside the dense batch"
        assert np.array_equal(seg.view(np.uint32), refc[b * cap: b * cap + used].view(np.uint32))
