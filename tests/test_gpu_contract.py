"""GPU parity for ttc_contract (ladder TT output) against oracle O3 (core by core, same gauge) and against
the dense Eq. 8 definition (gauge invariant), plus exact metadata."""
import itertools

import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
import ttgen
from tests import ref_numpy as ref

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _contract(X, Y, xm, ym):
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    plan = ttc.ttc_contract_plan_create(XD, YD, xm, ym)
    cores, ranks, offs = ttc.ttc_contract(plan, XD, YD)
    torch.cuda.synchronize()
    return plan, cores.cpu().numpy().astype(np.float64), ranks, offs


def _check_pair(plan, flat, offs, X, Y, b, xm, ym, dense=True):
    xc, yc = X.train(b), Y.train(b)
    res = oracle.tt_contract(xc, yc, xm, ym)
    assert list(plan.ranks[b]) == list(res["ranks"])
    seg = flat[offs[b]: offs[b] + res["elems"]]
    assert seg.shape == res["flat"].shape
    # core-wise, same construction (gauge).  Each entry is a short fp32 sum: its rounding error is bounded by
    # a few ulps of the sum of |terms|, which the oracle gives exactly when run on |X|, |Y| (R11).
    bound = oracle.tt_contract([np.abs(c) for c in xc], [np.abs(c) for c in yc], xm, ym)["flat"]
    err = np.abs(seg - res["flat"])
    worst = np.max(err / np.maximum(bound, 1e-30))
    assert worst <= 1e-5, f"pair {b}: core-wise error {worst:.3e} of the |terms| bound"
    if dense and res["order"] > 0:
        cores, pos = [], 0
        for l in range(res["order"]):
            a, i, c = int(res["ranks"][l]), int(res["dims"][l]), int(res["ranks"][l + 1])
            cores.append(seg[pos:pos + a * i * c].reshape((a, i, c), order="F"))
            pos += a * i * c
        got = oracle.to_canonical(ref.dense_from_tt(cores), res["perm"])
        want = ref.tcp(ref.dense_from_tt(xc), ref.dense_from_tt(yc), xm, ym)
        err = np.linalg.norm(got - want) / oracle.normaliser(xc, yc)
        assert err <= 1e-4, f"pair {b}: dense normalised error {err:.3e}"


def test_c3_small_dense_and_corewise():
    c = ttgen.CONFIGS["C3"]
    xm, ym = list(c["x_modes"]), list(c["y_modes"])
    X, Y = ttgen.config_batch("C3", B=5)
    plan, flat, ranks, offs = _contract(X, Y, xm, ym)
    assert plan.total == 5 * 102976
    for b in range(5):
        _check_pair(plan, flat, offs, X, Y, b, xm, ym, dense=(b < 2))


def test_c3_full_size_sampled():
    """BASELINE.json configs[2]: 1024 pairs (the launch bench.py --config C3 times), sampled core-wise."""
    c = ttgen.CONFIGS["C3"]
    xm, ym = list(c["x_modes"]), list(c["y_modes"])
    X, Y = ttgen.config_batch("C3", device=DEV)
    plan, flat, ranks, offs = _contract(X, Y, xm, ym)
    for b in (0, 1, 511, 1000, 1023):
        _check_pair(plan, flat, offs, X, Y, b, xm, ym, dense=False)


def _monotone(N, M, K):
    for a in itertools.combinations(range(1, N + 1), K):
        for b in itertools.combinations(range(1, M + 1), K):
            yield list(a), list(b)


def test_all_pair_sets_small_heterogeneous():
    """Every non-crossing pair set of small trains with per-pair different ranks (ragged layouts)."""
    rng = np.random.default_rng(7)
    cases = 0
    for N, M in [(1, 1), (2, 2), (3, 2), (2, 4), (3, 3), (4, 3)]:
        for K in range(0, min(N, M) + 1):
            for xm, ym in _monotone(N, M, K):
                xd = [int(v) for v in rng.integers(1, 4, N)]
                yd = [int(v) for v in rng.integers(1, 4, M)]
                for a, b in zip(xm, ym):
                    yd[b - 1] = xd[a - 1]
                B = 3
                xr = np.stack([[1] + list(rng.integers(1, 6, N - 1)) + [1] for _ in range(B)]).astype(np.int32)
                yr = np.stack([[1] + list(rng.integers(1, 6, M - 1)) + [1] for _ in range(B)]).astype(np.int32)
                X = ttgen.gaussian_batch(cases, 0, 0, 0, xr, xd, "geo")
                Y = ttgen.gaussian_batch(cases, 0, 1, 0, yr, yd, "geo")
                plan, flat, ranks, offs = _contract(X, Y, xm, ym)
                for b in range(B):
                    if plan.L == 0:
                        want, _ = oracle.tt_inner(X.train(b), Y.train(b))
                        assert abs(flat[b] - want) <= 1e-5 * oracle.normaliser(X.train(b), Y.train(b))
                    else:
                        _check_pair(plan, flat, offs, X, Y, b, xm, ym)
                cases += 1
    assert cases > 40


def test_outer_product_is_bitwise_concatenation():
    X, Y = ttgen.config_batch("C3", B=3)
    plan, flat, ranks, offs = _contract(X, Y, [], [])
    xs = int(X.offsets[1])
    ys = int(Y.offsets[1])
    for b in range(3):
        seg = flat[offs[b]: offs[b] + xs + ys]
        want = np.concatenate([X.cores[b * xs:(b + 1) * xs].numpy(), Y.cores[b * ys:(b + 1) * ys].numpy()])
        assert np.array_equal(seg, want.astype(np.float64))


def test_contract_determinism():
    c = ttgen.CONFIGS["C3"]
    X, Y = ttgen.config_batch("C3", B=16)
    _, a, _, _ = _contract(X, Y, list(c["x_modes"]), list(c["y_modes"]))
    _, b, _, _ = _contract(X, Y, list(c["x_modes"]), list(c["y_modes"]))
    assert np.array_equal(a, b)
