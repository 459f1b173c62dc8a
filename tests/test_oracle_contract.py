"""Pins for oracle O3 (ladder tt_contract) and its metadata: the dense definition (Eq. 8 after Alg. 2's
final permutation), exact counts of the K step and the hand-derived C3 values."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import ttgen
from tests import ref_numpy as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _dense(res):
    if res["order"] == 0:
        return np.asarray(res["cores"][0])
    return oracle.to_canonical(ref.dense_from_tt(res["cores"]), res["perm"])


def _monotone_pairs(N, M, K):
    for xm in itertools.combinations(range(1, N + 1), K):
        for ym in itertools.combinations(range(1, M + 1), K):
            yield list(xm), list(ym)


def test_ladder_equals_dense_tcp_exhaustive():
    """O3 reconstructed and permuted by out_perm == Eq. 8 (numpy tensordot and oracle O1) for every
    non-crossing pair set of small trains."""
    rng = np.random.default_rng(20)
    cases = 0
    for N, M in [(1, 1), (1, 3), (2, 2), (3, 2), (3, 3), (4, 3), (2, 4)]:
        for K in range(0, min(N, M) + 1):
            for xm, ym in _monotone_pairs(N, M, K):
                xd = list(rng.integers(1, 4, N))
                yd = list(rng.integers(1, 4, M))
                for a, b in zip(xm, ym):
                    yd[b - 1] = xd[a - 1]
                xr = [1] + list(rng.integers(1, 4, N - 1)) + [1]
                yr = [1] + list(rng.integers(1, 4, M - 1)) + [1]
                X, Y = ref.random_train(rng, xd, xr), ref.random_train(rng, yd, yr)
                res = oracle.tt_contract(X, Y, xm, ym)
                want = ref.tcp(ref.dense_from_tt(X), ref.dense_from_tt(Y), xm, ym)
                got = _dense(res)
                assert got.shape == want.shape
                np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-12)
                z1, _ = oracle.tcp(oracle.tt_reconstruct(X), oracle.tt_reconstruct(Y), xm, ym)
                np.testing.assert_allclose(got, z1, rtol=1e-11, atol=1e-12)
                assert res["order"] == N + M - 2 * K
                # bond ranks are products R_a * P_b of bonds of the operands
                assert all(int(r) >= 1 for r in res["ranks"])
                cases += 1
    assert cases > 60


def test_outer_product_is_concatenation_bitwise():
    """K = 0: the result is the two trains one after the other, values copied exactly."""
    rng = np.random.default_rng(21)
    X = ref.random_train(rng, [2, 3], [1, 2, 1])
    Y = ref.random_train(rng, [4, 2, 2], [1, 3, 2, 1])
    res = oracle.tt_contract(X, Y, [], [])
    assert res["order"] == 5
    for got, want in zip(res["cores"], X + Y):
        assert got.shape == want.shape and np.array_equal(got, want)
    assert list(res["src"]) == [1, 2, -1, -2, -3] and list(res["perm"]) == [1, 2, 3, 4, 5]


def test_all_modes_is_inner_product():
    rng = np.random.default_rng(22)
    dims = [3, 2, 4]
    X = ref.random_train(rng, dims, [1, 2, 3, 1])
    Y = ref.random_train(rng, dims, [1, 3, 2, 1])
    res = oracle.tt_contract(X, Y, [1, 2, 3], [1, 2, 3])
    assert res["order"] == 0
    assert abs(res["cores"][0] - oracle.tt_inner(X, Y)[0]) < 1e-12


@pytest.mark.parametrize("I,R,want", [(1000, 5, 25000), (1000, 2, 4000), (20, 20, 8000)])
def test_k_step_count_pins(I, R, want):
    """PAPER.md:442 (25000, 4000) and SPEC.md:346 (8000): the K = A_x^T A_y step costs R_1 I_n P_1 MACs.
    Order-5 trains contracted x_1^1: the oracle counts exactly those MACs forming the transfer."""
    rng = np.random.default_rng(23)
    dims = [I, 3, 2, 2, 3]
    ranks = [1, R, 2, 2, 2, 1]
    X, Y = ref.random_train(rng, dims, ranks), ref.random_train(rng, dims, ranks)
    res = oracle.tt_contract(X, Y, [1], [1])
    assert res["t_macs"] == want
    # and the transfer is Eq. 12's K = A_x^T A_y (R_1 x P_1): absorbed into the next core (X_2 (x) I_{P_1}),
    # core 1 of the output is sum_r K[r, p] X_2[r, i, r'] at bond index r' + R_2 p (R9, R10)
    assert res["order"] == 8
    K_mat = X[0][0].T @ Y[0][0]
    X2 = X[1]
    R2 = X2.shape[2]
    want = np.einsum("rp,ris->isp", K_mat, X2).reshape(1, dims[1], R2 * R, order="F")
    np.testing.assert_allclose(res["cores"][0], want, rtol=1e-12, atol=1e-12 * np.max(np.abs(want)))


def test_single_leading_pair_transfer_is_eq12():
    """Pair (1,1): T_1 = A_x^T A_y (Eq. 12) is absorbed into X_2 (x) I_{P_1}; check core 1 directly."""
    rng = np.random.default_rng(24)
    X = ref.random_train(rng, [4, 3, 2], [1, 2, 3, 1])
    Y = ref.random_train(rng, [4, 2], [1, 3, 1])
    res = oracle.tt_contract(X, Y, [1], [1])
    K = X[0][0].T @ Y[0][0]                               # R_1 x P_1
    R1, P1 = K.shape
    X2 = X[1]                                             # R_1 x I_2 x R_2
    want = np.zeros((1, 3, X2.shape[2] * P1))
    for i in range(3):
        for rr in range(X2.shape[2]):
            for p in range(P1):
                want[0, i, rr + X2.shape[2] * p] = sum(K[r, p] * X2[r, i, rr] for r in range(R1))
    np.testing.assert_allclose(res["cores"][0], want, rtol=1e-13, atol=1e-14)


def test_eq10_example_shape_and_perm():
    """Example 1: X (order 4) x_3^2 Y (order 3) -> Z in R^{I1 x I2 x I4 x J1 x J3}."""
    rng = np.random.default_rng(25)
    xd, yd = [2, 3, 4, 5], [6, 4, 7]
    X = ref.random_train(rng, xd, [1, 2, 3, 2, 1])
    Y = ref.random_train(rng, yd, [1, 2, 2, 1])
    res = oracle.tt_contract(X, Y, [3], [2])
    got = _dense(res)
    assert got.shape == (2, 3, 5, 6, 7)
    np.testing.assert_allclose(got, ref.tcp(ref.dense_from_tt(X), ref.dense_from_tt(Y), [3], [2]), rtol=1e-11,
                               atol=1e-12)


def test_c3_metadata_hand_values():
    g = json.load(open(os.path.join(GOLD, "c3_ladder_meta.json")))
    rng = np.random.default_rng(26)
    X = ref.random_train(rng, [g["I"]] * g["N"], [1] + [g["R"]] * (g["N"] - 1) + [1])
    Y = ref.random_train(rng, [g["I"]] * g["M"], [1] + [g["P"]] * (g["M"] - 1) + [1])
    res = oracle.tt_contract(X, Y, g["x_modes"], g["y_modes"])
    assert res["order"] == g["order"]
    assert list(res["dims"]) == g["dims"]
    assert list(res["ranks"]) == g["ranks"]
    assert list(res["src"]) == g["src"]
    assert list(res["perm"]) == g["perm"]
    assert res["elems"] == g["elems"]
    assert res["t_macs"] == g["transfer_macs"]


@pytest.mark.slow
def test_c3_dense_check_two_pairs():
    """C3 (BASELINE.json configs[2]): dense Eq. 8 (8^9 MACs) vs the reconstructed ladder TT, 2 pairs."""
    c = ttgen.CONFIGS["C3"]
    X, Y = ttgen.config_batch("C3", B=2)
    for b in range(2):
        xc, yc = X.train(b), Y.train(b)
        res = oracle.tt_contract(xc, yc, list(c["x_modes"]), list(c["y_modes"]))
        z, macs = oracle.tcp(oracle.tt_reconstruct(xc), oracle.tt_reconstruct(yc), list(c["x_modes"]),
                             list(c["y_modes"]))
        assert macs == 8 ** 9
        got = _dense(res)
        scale = oracle.normaliser(xc, yc)
        assert np.max(np.abs(got - z)) <= 1e-12 * scale


def test_mode_errors():
    rng = np.random.default_rng(27)
    X = ref.random_train(rng, [2, 3], [1, 2, 1])
    Y = ref.random_train(rng, [3, 2], [1, 2, 1])
    with pytest.raises(oracle.OracleError):
        oracle.tt_contract(X, Y, [1, 2], [2, 1])   # crossing pairs are not a ladder
    with pytest.raises(oracle.OracleError):
        oracle.tt_contract(X, Y, [1], [1])         # I_1 = 2 != J_1 = 3


def test_batch_wrappers_equal_single_pair_calls():
    """oracle_tt_contract_batch / oracle_tt_splice_batch (the C3 / S1 cpu_baseline legs) return, pair by pair at
    the caller's offsets, exactly what the single-pair O3 / O5 return (same loops, so bitwise), including a
    sub-range (first, count) and more threads than pairs."""
    for cfg in ("C3", "S1"):
        c = ttgen.CONFIGS[cfg]
        B = 5
        X, Y = ttgen.config_batch(cfg, B=B)
        singles = []
        for b in range(B):
            if cfg == "C3":
                singles.append(oracle.tt_contract(X.train(b), Y.train(b), list(c["x_modes"]), list(c["y_modes"])))
            else:
                singles.append(oracle.tt_splice(X.train(b), Y.train(b), c["x_mode"], c["y_mode"]))
        per = singles[0]["elems"]
        for first, count, nth in ((0, B, 1), (0, B, 8), (2, 3, 2)):
            gap = 7   # non-packed output layout: trains 7 floats apart, in reverse order
            offs = np.array([(count - 1 - j) * (per + gap) for j in range(count)], np.int64)
            total = count * (per + gap)
            if cfg == "C3":
                out = oracle.tt_contract_batch(X, Y, list(c["x_modes"]), list(c["y_modes"]), offs, total, nth, first,
                                               count)
            else:
                out = oracle.tt_splice_batch(X, Y, c["x_mode"], c["y_mode"], offs, total, nth, first, count)
            for j in range(count):
                seg = out[offs[j]: offs[j] + per]
                assert np.array_equal(seg, singles[first + j]["flat"]), (cfg, first, j)
                assert not np.any(out[offs[j] + per: offs[j] + per + gap])   # nothing written in the gaps
