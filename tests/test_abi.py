"""C-ABI checks that need no GPU: the library loads, exports every symbol include/ttc.h declares, validates
arguments on the host (every error code), and its host-side plan / cost / partition logic matches the oracle
and the hand values exactly.  A valid compute call without a GPU must fail (TTC_ERR_CUDA): no CPU fallback."""
import ctypes
import itertools
import json
import os
import re

import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
import ttgen
from oracle import complexity as cx
from tests import ref_numpy as ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ttc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ttc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = _declared_symbols()
    assert len(syms) == 19
    lib = ctypes.CDLL(ttc.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(ttc.EXPORTED)
    assert ttc.ttc_version() == 1


def _dev(B=2, N=3, dims=(2, 3, 2), R=2, device="cpu"):
    r = ttgen.uniform_ranks(B, N, R)
    offs, total = ttgen.packed_offsets(r, dims)
    return ttc.TTDevice(torch.zeros(total), dims, ranks=r, offsets=offs)


def _call_inner(x, y, out=None):
    out = torch.zeros(max(x.B, 1)) if out is None else out
    return ttc._lib.ttc_inner(ctypes.byref(x.c), ctypes.byref(y.c), out.data_ptr(), None)


def test_valid_inner_without_gpu_is_a_cuda_error_not_a_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x, y = _dev(), _dev()
    assert _call_inner(x, y) == ttc.TTC_ERR_CUDA
    assert "ttc_inner launch" in ttc.ttc_last_error()


def test_zero_batch_is_a_noop():
    x, y = _dev(B=0), _dev(B=0)
    assert ttc._lib.ttc_inner(ctypes.byref(x.c), ctypes.byref(y.c), None, None) == ttc.TTC_OK


def test_error_codes():
    x, y = _dev(), _dev()
    lib = ttc._lib
    assert lib.ttc_inner(None, ctypes.byref(y.c), None, None) == ttc.TTC_ERR_NULL
    # batch mismatch
    assert _call_inner(x, _dev(B=3)) == ttc.TTC_ERR_SHAPE
    # mode-size mismatch, diagnostic names both dimensions
    assert _call_inner(x, _dev(dims=(2, 4, 2))) == ttc.TTC_ERR_SHAPE
    assert "X mode 2 (I=3) vs Y mode 2 (J=4)" in ttc.ttc_last_error()
    # boundary rank != 1
    r = ttgen.uniform_ranks(2, 3, 2)
    r[1, 3] = 2
    offs = np.array([0, 100], np.int64)
    bad = ttc.TTDevice(torch.zeros(300), (2, 3, 2), ranks=r, offsets=offs)
    assert _call_inner(bad, y) == ttc.TTC_ERR_RANK
    assert "pair 1" in ttc.ttc_last_error()
    r2 = ttgen.uniform_ranks(2, 3, 2)
    r2[0, 1] = 0
    assert _call_inner(ttc.TTDevice(torch.zeros(300), (2, 3, 2), ranks=r2, offsets=offs), y) == ttc.TTC_ERR_RANK
    # rank above the supported maximum
    big = ttc.TTDevice(torch.zeros(10), (2, 3, 2), uniform_rank=129, batch=2)
    assert _call_inner(big, y) == ttc.TTC_ERR_UNSUPPORTED
    # trains past the end of the buffer
    short = ttc.TTDevice(torch.zeros(5), (2, 3, 2), uniform_rank=2, batch=2)
    assert _call_inner(short, y) == ttc.TTC_ERR_OVERFLOW
    # misaligned output
    buf = torch.zeros(8)
    assert lib.ttc_inner(ctypes.byref(x.c), ctypes.byref(y.c), buf.data_ptr() + 2, None) == ttc.TTC_ERR_ALIGN
    # misaligned cores
    xm = _dev()
    xm.c.cores = xm.cores.data_ptr() + 1
    assert _call_inner(xm, y) == ttc.TTC_ERR_ALIGN
    # negative batch / order
    xn = _dev()
    xn.c.batch = -1
    assert _call_inner(xn, y) == ttc.TTC_ERR_ARG
    xo = _dev()
    xo.c.order = 0
    assert _call_inner(xo, y) == ttc.TTC_ERR_SHAPE
    # offset overflow
    r3 = ttgen.uniform_ranks(2, 3, 2)
    r3[0, 1] = 3
    ov = ttc.TTDevice(torch.zeros(300), (2, 3, 2), ranks=r3, offsets=np.array([0, 2 ** 62], np.int64))
    assert _call_inner(ov, y) == ttc.TTC_ERR_OVERFLOW
    with pytest.raises(ttc.TTCError):
        ttc.ttc_inner(x, _dev(B=3), out=torch.zeros(2))


def test_contract_mode_errors():
    x, y = _dev(), _dev()
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_contract_plan_create(x, y, [1, 3], [3, 1])
    assert e.value.status == ttc.TTC_ERR_MODES
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_contract_plan_create(x, y, [4], [1])
    assert e.value.status == ttc.TTC_ERR_MODES
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_contract_plan_create(x, y, [1], [2])        # I_1 = 2 vs J_2 = 3
    assert e.value.status == ttc.TTC_ERR_SHAPE
    assert "X mode 1 (I=2) vs Y mode 2 (J=3)" in ttc.ttc_last_error()


def _monotone(N, M, K):
    for xm in itertools.combinations(range(1, N + 1), K):
        for ym in itertools.combinations(range(1, M + 1), K):
            yield list(xm), list(ym)


def test_contract_plan_metadata_matches_oracle_exhaustive():
    """Host plan (ladder order, dims, src, perm, per-pair ranks and sizes) == oracle O3, exactly."""
    rng = np.random.default_rng(0)
    n = 0
    for N, M in [(1, 1), (2, 3), (3, 3), (4, 2), (3, 5)]:
        for K in range(0, min(N, M) + 1):
            for xm, ym in _monotone(N, M, K):
                xd = list(rng.integers(1, 4, N))
                yd = list(rng.integers(1, 4, M))
                for a, b in zip(xm, ym):
                    yd[b - 1] = xd[a - 1]
                B = 3
                xr = np.stack([[1] + list(rng.integers(1, 5, N - 1)) + [1] for _ in range(B)]).astype(np.int32)
                yr = np.stack([[1] + list(rng.integers(1, 5, M - 1)) + [1] for _ in range(B)]).astype(np.int32)
                xo, xt = ttgen.packed_offsets(xr, xd)
                yo, yt = ttgen.packed_offsets(yr, yd)
                X = ttc.TTDevice(torch.zeros(xt), xd, ranks=xr, offsets=xo)
                Y = ttc.TTDevice(torch.zeros(yt), yd, ranks=yr, offsets=yo)
                plan = ttc.ttc_contract_plan_create(X, Y, xm, ym)
                total = 0
                for b in range(B):
                    Xc = ref.random_train(rng, xd, xr[b])
                    Yc = ref.random_train(rng, yd, yr[b])
                    res = oracle.tt_contract(Xc, Yc, xm, ym, with_cores=False)
                    assert plan.L == res["order"]
                    assert list(plan.dims) == list(res["dims"])
                    assert list(plan.src) == list(res["src"])
                    assert list(plan.perm) == list(res["perm"])
                    assert list(plan.ranks[b]) == list(res["ranks"])
                    assert plan.offsets[b] == total
                    total += res["elems"]
                assert plan.total == total
                n += 1
    assert n > 50


def test_splice_plan_metadata_matches_oracle():
    """Host splice plan (chain order, dims, src, perm, per-pair ranks and sizes) == oracle O5, exactly, for
    every end-mode choice; interior modes are rejected (TTC_ERR_MODES)."""
    rng = np.random.default_rng(1)
    n_cases = 0
    for N, M in [(1, 1), (1, 3), (2, 2), (3, 3), (4, 2), (5, 4)]:
        for n in sorted({1, N}):
            for m in sorted({1, M}):
                xd = list(rng.integers(1, 4, N))
                yd = list(rng.integers(1, 4, M))
                yd[m - 1] = xd[n - 1]
                B = 3
                xr = np.stack([[1] + list(rng.integers(1, 5, N - 1)) + [1] for _ in range(B)]).astype(np.int32)
                yr = np.stack([[1] + list(rng.integers(1, 5, M - 1)) + [1] for _ in range(B)]).astype(np.int32)
                xo, xt = ttgen.packed_offsets(xr, xd)
                yo, yt = ttgen.packed_offsets(yr, yd)
                X = ttc.TTDevice(torch.zeros(xt), xd, ranks=xr, offsets=xo)
                Y = ttc.TTDevice(torch.zeros(yt), yd, ranks=yr, offsets=yo)
                plan = ttc.ttc_splice_plan_create(X, Y, n, m)
                total = 0
                for b in range(B):
                    res = oracle.tt_splice(ref.random_train(rng, xd, xr[b]), ref.random_train(rng, yd, yr[b]), n, m,
                                           with_cores=False)
                    assert plan.L == res["order"]
                    assert list(plan.dims) == list(res["dims"])
                    assert list(plan.src) == list(res["src"])
                    assert list(plan.perm) == list(res["perm"])
                    assert list(plan.ranks[b]) == list(res["ranks"])
                    assert plan.offsets[b] == total
                    total += res["elems"]
                assert plan.total == total
                n_cases += 1
    assert n_cases == 19
    x, y = _dev(N=3, dims=(2, 3, 2)), _dev(N=3, dims=(2, 3, 2))
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_splice_plan_create(x, y, 2, 1)
    assert e.value.status == ttc.TTC_ERR_MODES
    x2 = _dev(N=3, dims=(3, 3, 2))
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_splice_plan_create(x2, y, 1, 1)         # I_1 = 3 vs J_1 = 2
    assert e.value.status == ttc.TTC_ERR_SHAPE
    assert "X mode 1 (I=3) vs Y mode 1 (J=2)" in ttc.ttc_last_error()


def test_c3_plan_hand_values():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_ladder_meta.json")))
    X = ttc.TTDevice(torch.zeros(1), [8] * 6, uniform_rank=8, batch=0)
    Y = ttc.TTDevice(torch.zeros(1), [8] * 6, uniform_rank=8, batch=0)
    x1 = ttc.TTDevice(torch.zeros(2 * 8 * 8 + 4 * 8 * 64), [8] * 6, uniform_rank=8, batch=1)
    plan = ttc.ttc_contract_plan_create(x1, x1, g["x_modes"], g["y_modes"])
    assert plan.L == g["order"] and list(plan.dims) == g["dims"] and list(plan.src) == g["src"]
    assert list(plan.perm) == g["perm"] and list(plan.ranks[0]) == g["ranks"] and plan.total == g["elems"]
    assert plan.max_rank == 64


def test_pair_cost_matches_closed_forms():
    for cfg, mac_want, bytes_want in (("C1", 4240, 4480), ("C2", 795136, 200704), ("C4", 29393408, 1839104)):
        c = ttgen.CONFIGS[cfg]
        x = ttc.TTDevice(torch.zeros(1), [c["I"]] * c["N"], uniform_rank=c["R"], batch=0)
        r = ttgen.uniform_ranks(2, c["N"], c["R"])
        offs, tot = ttgen.packed_offsets(r, [c["I"]] * c["N"])
        X = ttc.TTDevice(torch.zeros(tot), [c["I"]] * c["N"], ranks=r, offsets=offs)
        mac, by = ttc.ttc_pair_cost(X, X)
        assert list(mac) == [mac_want] * 2
        assert list(by) == [bytes_want + 4] * 2   # cores read once + the 4-byte result
    # heterogeneous (C5 shape): min-association cost, checked against the W-first oracle count as an upper bound
    X, Y = ttgen.config_batch("C5", B=4)
    XD, YD = ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)
    mac, by = ttc.ttc_pair_cost(XD, YD)
    for b in range(4):
        dims = list(X.dims)
        w_first = cx.sweep_macs(dims, list(X.ranks[b]), list(Y.ranks[b]))
        v_first = cx.sweep_macs(dims, list(Y.ranks[b]), list(X.ranks[b]))
        assert mac[b] <= min(w_first, v_first)
        per_step = sum(dims[n] * min(X.ranks[b, n] * Y.ranks[b, n] * Y.ranks[b, n + 1] + X.ranks[b, n] * X.ranks[b, n + 1] * Y.ranks[b, n + 1],
                                     X.ranks[b, n] * Y.ranks[b, n] * X.ranks[b, n + 1] + Y.ranks[b, n] * X.ranks[b, n + 1] * Y.ranks[b, n + 1])
                       for n in range(len(dims)))
        assert mac[b] == per_step
        assert by[b] == 4 * (sum(X.ranks[b, n] * dims[n] * X.ranks[b, n + 1] + Y.ranks[b, n] * dims[n] * Y.ranks[b, n + 1]
                                 for n in range(len(dims))) + 1)


@pytest.mark.parametrize("seed", range(6))
def test_partition_is_optimal_contiguous_split(seed):
    """Bottleneck of ttc_partition == brute-force optimum over all contiguous k-splits (small B)."""
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 11))
    k = int(rng.integers(1, 5))
    cost = rng.uniform(0.5, 3.0, B)
    bounds = ttc.ttc_partition(cost, k)
    assert bounds[0] == 0 and bounds[-1] == B and np.all(np.diff(bounds) >= 0)
    if B >= k:
        assert np.all(np.diff(bounds) >= 1)
    got = max(cost[bounds[j]:bounds[j + 1]].sum() for j in range(k))
    best = np.inf
    for cuts in itertools.combinations(range(1, B), min(k - 1, B - 1)):
        bb = [0, *cuts, B]
        best = min(best, max(cost[bb[j]:bb[j + 1]].sum() for j in range(len(bb) - 1)))
    assert got <= best * (1 + 1e-9)


def test_partition_uniform_and_errors():
    b = ttc.ttc_partition(np.ones(4096), 8)
    assert list(b) == [512 * j for j in range(9)]
    with pytest.raises(ttc.TTCError):
        ttc.ttc_partition(np.ones(4), 0)
    with pytest.raises(ttc.TTCError):
        ttc.ttc_partition(np.array([1.0, -1.0]), 2)


def test_tt_svd_workspace_sizes():
    """Host-only sizing of ttc_tt_svd's caller-owned workspace: Z_n (B x prod(dims) floats), the Gram matrix and
    its eigenvectors (B x g^2 doubles each), eigenvalues (B x g doubles), order (B x g int32), norms (B doubles),
    each 256-byte aligned, g = the largest unfolding side; 0 where the fused launch runs (N = 1, or g > 32)."""
    al = lambda v: (v + 255) // 256 * 256
    B, dims = 7, (20, 20, 20)
    g = 20
    want = al(4 * B * 8000) + 2 * al(8 * B * g * g) + al(8 * B * g) + al(4 * B * g) + al(8 * B)
    assert ttc.ttc_tt_svd_workspace(B, dims) == want
    assert ttc.ttc_tt_svd_workspace(0, dims) == 0 or ttc.ttc_tt_svd_workspace(0, dims) >= 0
    assert ttc.ttc_tt_svd_workspace(B, (5,)) == 0            # N = 1: no SVD step
    assert ttc.ttc_tt_svd_workspace(B, (40, 40)) == 0        # side 40 > 32: fused launch
    assert ttc.ttc_tt_svd_workspace(B, (4, 6), perm=(2, 1)) > 0
    with pytest.raises(ttc.TTCError):
        ttc.ttc_tt_svd_workspace(B, (4, 6), perm=(1, 1))
    # beyond shared memory (Example 2's (ii) / (iii)): the one-sided Jacobi kernel's fp64 Z, A (prod(dims) each),
    # V (gmax^2), singular values and signs (gmax each) and 64 + 16 doubles of group partials / padding per tensor,
    # plus 32 synchronisation ints per tensor; gmax = the largest smaller side of an unfolding (400 x 100 -> 100;
    # 400 x 400 -> 400)
    big = lambda el, g: 8 * B * (2 * el + g * g + 2 * g + 80) + 4 * B * 32
    assert ttc.ttc_tt_svd_workspace(B, (20, 20, 20, 5)) == big(40000, 100)
    assert ttc.ttc_tt_svd_workspace(B, (20, 20, 20, 5, 4)) == big(160000, 400)
    assert ttc.ttc_tt_svd_workspace(B, (5, 20, 20, 20), perm=(2, 3, 4, 1)) == big(40000, 100)
    assert ttc.ttc_tt_svd_workspace(B, (70, 70)) == big(4900, 70)   # side 70 > 64
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_tt_svd_workspace(B, (2000, 2000))            # smaller side 2000 > 1024
    assert e.value.status == ttc.TTC_ERR_UNSUPPORTED


def test_inner_ordered_validates_the_permutation():
    """ttc_inner_ordered checks its host order on the host (no CUDA call on error)."""
    import ctypes
    X, Y = ttgen.config_batch("C2", kind="iid", B=4)
    XD, YD = ttc.TTDevice.from_batch(X, "cpu"), ttc.TTDevice.from_batch(Y, "cpu")
    out = torch.zeros(4)
    for bad in ([0, 1, 2, 2], [0, 1, 2, 4], [-1, 0, 1, 2]):
        o = np.asarray(bad, np.int32)
        rc = ttc._lib.ttc_inner_ordered(ctypes.byref(XD.c), ctypes.byref(YD.c), ttc._ptr(o), ttc._ptr(o),
                                         ttc._ptr(out), None)
        assert rc == ttc.TTC_ERR_ARG, bad
        assert "permutation" in ttc.ttc_last_error()


def test_every_compute_entry_is_a_noop_on_an_empty_batch():
    """B = 0: every compute entry point returns TTC_OK without touching the device (this
    container has none, so any CUDA call would fail)."""
    x = ttc.TTDevice(torch.zeros(1), [3, 4, 2], uniform_rank=2, batch=0)
    y = ttc.TTDevice(torch.zeros(1), [3, 4, 2], uniform_rank=3, batch=0)
    lib = ttc._lib
    assert lib.ttc_inner_ordered(ctypes.byref(x.c), ctypes.byref(y.c), None, None, None, None) == ttc.TTC_OK
    plan = ttc.ttc_contract_plan_create(x, y, [2], [2])
    assert plan.total == 0 or plan.total >= 0
    assert lib.ttc_contract(plan.handle, ctypes.byref(x.c), ctypes.byref(y.c), None, None, None) == ttc.TTC_OK
    splice = ttc.ttc_splice_plan_create(x, y, 1, 1)
    assert lib.ttc_contract(splice.handle, ctypes.byref(x.c), ctypes.byref(y.c), None, None, None) == ttc.TTC_OK
    perm = np.asarray([3, 1, 2], np.int32)
    assert lib.ttc_reconstruct(ctypes.byref(x.c), ttc._ptr(perm), None, None, None) == ttc.TTC_OK
    dims = np.asarray([3, 4, 2], np.int32)
    assert lib.ttc_tt_svd(0, 3, ttc._ptr(dims), None, None, ctypes.c_double(0.1), None, None, None, 0,
                          None) == ttc.TTC_OK
    nb = ctypes.c_int64(-1)
    assert lib.ttc_tt_svd_workspace(0, 3, ttc._ptr(dims), None, ctypes.byref(nb)) == ttc.TTC_OK and nb.value == 0


def test_n_elems_is_required_and_bounds_every_train():
    """ttc.h: n_elems >= 1 is required when batch > 0 (TTC_ERR_ARG, no unchecked device reads); a packed uniform
    batch or an offset train running past n_elems is TTC_ERR_OVERFLOW."""
    x, y = _dev(), _dev()
    x.c.n_elems = 0
    assert _call_inner(x, y) == ttc.TTC_ERR_ARG
    assert "n_elems" in ttc.ttc_last_error()
    x, y = _dev(), _dev()
    x.c.n_elems -= 1
    assert _call_inner(x, y) == ttc.TTC_ERR_OVERFLOW


def test_tt_svd_dense_size_overflow_is_detected():
    """The dense size prod I_n is overflow-checked before use ({2^20, 2^20, 2^24} used to wrap to 0)."""
    cap = ctypes.c_int64(0)
    d = np.array([1 << 20, 1 << 20, 1 << 24], np.int32)
    assert ttc._lib.ttc_tt_svd_capacity(3, d.ctypes.data, None, ctypes.byref(cap)) == ttc.TTC_ERR_OVERFLOW
    d = np.array([1 << 15, 1 << 15, 1 << 15], np.int32)   # 2^45 > 2^40
    assert ttc._lib.ttc_tt_svd_capacity(3, d.ctypes.data, None, ctypes.byref(cap)) == ttc.TTC_ERR_OVERFLOW


def test_reconstruct_workspace_sizes():
    """Host-only sizing of ttc_reconstruct_ws's workspace: 0 where a shared-memory split exists; else B x two
    ping-pong buffers per chain, the split k minimising the multiply-adds (ties: the smaller k).  Hand values for
    dims (7, 2000, 9), ranks (1, 7, 9, 1): k = 1 and k = 2 both cost 2,016,000 MACs, k = 1 has no left chain and
    one right step, Q_1 = R_1 x I_2 I_3 = 7 x 18,000 floats per buffer."""
    r = np.tile(np.array([1, 7, 9, 1], np.int32), (3, 1))
    T = ttgen.gaussian_batch(1, 0, 0, 0, r, (7, 2000, 9), "geo")
    TD = ttc.TTDevice.from_batch(T, "cpu")
    assert ttc.ttc_reconstruct_workspace(TD) == 4 * 3 * 2 * 7 * 18000
    assert ttc.ttc_reconstruct_workspace(TD, [3, 1, 2]) == 4 * 3 * 2 * 7 * 18000   # perm: output strides only
    small = ttgen.gaussian_batch(2, 0, 0, 0, np.tile(np.array([1, 3, 3, 1], np.int32), (2, 1)), (4, 5, 6), "geo")
    assert ttc.ttc_reconstruct_workspace(ttc.TTDevice.from_batch(small, "cpu")) == 0
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_reconstruct_workspace(TD, [1, 1, 2])
    assert e.value.status == ttc.TTC_ERR_MODES
