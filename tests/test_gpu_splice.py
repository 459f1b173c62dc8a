"""GPU parity for the TTCP splice of end modes (ttc_splice_plan_create + ttc_contract)
against oracle O5 (core by core, same construction) and the dense Eq. 8 definition, plus exactness of the
copied / rank-transposed cores (pure data movement: bitwise)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
import ttgen
from tests import ref_numpy as ref

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _splice(X, Y, n, m):
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    plan = ttc.ttc_splice_plan_create(XD, YD, n, m)
    cores, ranks, offs = ttc.ttc_contract(plan, XD, YD)
    torch.cuda.synchronize()
    return plan, cores.cpu().numpy().astype(np.float64), ranks, offs


def _check_pair(plan, flat, offs, X, Y, b, n, m, dense=True):
    xc, yc = X.train(b), Y.train(b)
    res = oracle.tt_splice(xc, yc, n, m)
    assert list(plan.ranks[b]) == list(res["ranks"])
    seg = flat[offs[b]: offs[b] + res["elems"]]
    assert seg.shape == res["flat"].shape
    # fp32 rounding of each entry is bounded by a few ulps of the sum of |terms| (oracle on |X|, |Y|)
    bound = oracle.tt_splice([np.abs(c) for c in xc], [np.abs(c) for c in yc], n, m)["flat"]
    worst = np.max(np.abs(seg - res["flat"]) / np.maximum(bound, 1e-30))
    assert worst <= 1e-5, f"pair {b}: core-wise error {worst:.3e} of the |terms| bound"
    if res["order"] == 0:
        return seg, res
    # cores that only move data (no K absorbed) are bitwise equal to the (widened fp32) oracle cores
    pos = 0
    absorbing = {l for l in range(res["order"]) if l == int(np.sum(np.asarray(res["src"]) > 0)) or
                 (l == res["order"] - 1 and np.all(np.asarray(res["src"]) > 0))}
    for l in range(res["order"]):
        a, i, c = int(res["ranks"][l]), int(res["dims"][l]), int(res["ranks"][l + 1])
        if l not in absorbing:
            assert np.array_equal(seg[pos:pos + a * i * c], res["flat"][pos:pos + a * i * c]), f"core {l} not exact"
        pos += a * i * c
    if dense:
        cores, pos = [], 0
        for l in range(res["order"]):
            a, i, c = int(res["ranks"][l]), int(res["dims"][l]), int(res["ranks"][l + 1])
            cores.append(seg[pos:pos + a * i * c].reshape((a, i, c), order="F"))
            pos += a * i * c
        got = oracle.to_canonical(ref.dense_from_tt(cores), res["perm"])
        want = ref.tcp(ref.dense_from_tt(xc), ref.dense_from_tt(yc), [n], [m])
        err = np.linalg.norm(got - want) / oracle.normaliser(xc, yc)
        assert err <= 1e-4, f"pair {b}: dense normalised error {err:.3e}"
    return seg, res


def test_all_end_modes_heterogeneous():
    """Every end-mode choice, N, M in 1..5, per-pair different ranks (ragged layouts), odd mode sizes."""
    rng = np.random.default_rng(17)
    cases = 0
    for N, M in [(1, 1), (1, 3), (3, 1), (2, 2), (3, 3), (5, 4), (4, 5)]:
        for n in sorted({1, N}):
            for m in sorted({1, M}):
                xd = [int(v) for v in rng.integers(1, 6, N)]
                yd = [int(v) for v in rng.integers(1, 6, M)]
                yd[m - 1] = xd[n - 1]
                B = 5
                xr = np.stack([[1] + list(rng.integers(1, 9, N - 1)) + [1] for _ in range(B)]).astype(np.int32)
                yr = np.stack([[1] + list(rng.integers(1, 9, M - 1)) + [1] for _ in range(B)]).astype(np.int32)
                X = ttgen.gaussian_batch(cases, 0, 0, 0, xr, xd, "geo")
                Y = ttgen.gaussian_batch(cases, 0, 1, 0, yr, yd, "geo")
                plan, flat, ranks, offs = _splice(X, Y, n, m)
                for b in range(B):
                    _check_pair(plan, flat, offs, X, Y, b, n, m)
                cases += 1
    assert cases == 21


def test_s1_full_size_sampled():
    """The S1 workload bench.py --config S1 times (16,384 pairs of C3's operands, x_1^1), sampled pairs."""
    c = ttgen.CONFIGS["S1"]
    X, Y = ttgen.config_batch("S1", device=DEV)
    plan, flat, ranks, offs = _splice(X, Y, c["x_mode"], c["y_mode"])
    assert plan.total == c["B"] * 4224
    for b in (0, 1, 8191, 16383):
        _check_pair(plan, flat, offs, X, Y, b, c["x_mode"], c["y_mode"], dense=(b == 0))


def test_uniform_ranks_and_large_ranks():
    """ranks_host == NULL (uniform) path, and ranks up to 64 (K of 64 x 64 in shared memory)."""
    rng = np.random.default_rng(3)
    for R, dims in ((8, (4, 3, 5)), (64, (4, 2, 4))):
        B = 3
        r = np.tile(np.array([1, R, R, 1], np.int32), (B, 1))
        X = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, r, dims, "geo")
        Y = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 1, 0, r, dims, "geo")
        for n, m in ((1, 1), (3, 3), (1, 3), (3, 1)):
            if dims[n - 1] != dims[m - 1]:
                continue
            plan, flat, ranks, offs = _splice(X, Y, n, m)
            for b in range(B):
                _check_pair(plan, flat, offs, X, Y, b, n, m, dense=(R == 8))


def test_splice_determinism():
    X, Y = ttgen.config_batch("S1", B=64)
    _, a, _, _ = _splice(X, Y, 1, 1)
    _, b, _, _ = _splice(X, Y, 1, 1)
    assert np.array_equal(a, b)
