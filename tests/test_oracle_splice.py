"""Pins for oracle O5 (the paper's TTCP splice of end modes, Alg. 2 steps 4-5 on TT operands): the dense
definition (Eq. 8 after the final permutation of step 6), Eq. 12's K, the rank law (R and P, no Kronecker
bonds), the (N, 1) case against the ladder (O3, bitwise) and Example 1's shape law."""
import numpy as np
import pytest

import oracle
from tests import ref_numpy as ref


def _dense(res):
    if res["order"] == 0:
        return np.asarray(res["cores"][0])
    return oracle.to_canonical(ref.dense_from_tt(res["cores"]), res["perm"])


def _case(rng, N, M, n, m, dmax=4, rmax=4):
    xd = list(rng.integers(1, dmax, N))
    yd = list(rng.integers(1, dmax, M))
    yd[m - 1] = xd[n - 1]
    xr = [1] + list(rng.integers(1, rmax, N - 1)) + [1]
    yr = [1] + list(rng.integers(1, rmax, M - 1)) + [1]
    return ref.random_train(rng, xd, xr), ref.random_train(rng, yd, yr), xr, yr


@pytest.mark.parametrize("N,M", [(1, 1), (1, 2), (2, 1), (2, 2), (3, 2), (2, 4), (4, 3), (5, 5)])
def test_splice_equals_dense_tcp(N, M):
    """O5 reconstructed and permuted by out_perm == Eq. 8 (numpy and oracle O1) for all four end-mode choices."""
    rng = np.random.default_rng(100 + 7 * N + M)
    for n in sorted({1, N}):
        for m in sorted({1, M}):
            for _ in range(3):
                X, Y, xr, yr = _case(rng, N, M, n, m)
                res = oracle.tt_splice(X, Y, n, m)
                want = ref.tcp(ref.dense_from_tt(X), ref.dense_from_tt(Y), [n], [m])
                got = _dense(res)
                assert got.shape == want.shape
                np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-12)
                z1, _ = oracle.tcp(oracle.tt_reconstruct(X), oracle.tt_reconstruct(Y), [n], [m])
                np.testing.assert_allclose(got, z1, rtol=1e-11, atol=1e-12)
                assert res["order"] == N + M - 2


def test_splice_rank_law_and_order():
    """Ranks are the operands' own bonds (Alg. 2 step 5: no Kronecker products): for n = m = 1 the chain is
    X_N^T .. X_2^T, K absorbed into Y_2, Y_3 .. Y_M, so the bonds are R_{N-1} .. R_1, P_2 .. P_{M-1}."""
    rng = np.random.default_rng(7)
    X, Y, xr, yr = _case(rng, 4, 4, 1, 1, dmax=3, rmax=5)
    res = oracle.tt_splice(X, Y, 1, 1)
    assert list(res["ranks"]) == [1, xr[3], xr[2], xr[1], yr[2], yr[3], 1]
    assert list(res["src"]) == [4, 3, 2, -2, -3, -4]
    # canonical order x2, x3, x4, y2, y3, y4 -> ladder positions
    assert list(res["perm"]) == [3, 2, 1, 4, 5, 6]
    # n = N, m = M: X_1 .. X_{N-1}, K, Y_{M-1}^T .. Y_1^T
    X, Y, xr, yr = _case(rng, 4, 4, 4, 4, dmax=3, rmax=5)
    res = oracle.tt_splice(X, Y, 4, 4)
    assert list(res["src"]) == [1, 2, 3, -3, -2, -1]
    assert list(res["ranks"]) == [1, xr[1], xr[2], xr[3], yr[2], yr[1], 1]


def test_splice_K_is_eq12():
    """N = 1 and M = 2, n = m = 1: the output's single core is K Y_2 with K = A_x^T A_y (Eq. 12)."""
    rng = np.random.default_rng(8)
    X, Y, xr, yr = _case(rng, 1, 2, 1, 1, dmax=5, rmax=4)
    res = oracle.tt_splice(X, Y, 1, 1)
    Ax = X[0][0, :, :]            # I x R_1 (R_1 = 1 here: N = 1)
    Ay = Y[0][0, :, :]            # I x P_1
    K = Ax.T @ Ay
    want = np.einsum("rp,pjq->rjq", K, Y[1])
    np.testing.assert_allclose(res["cores"][0], want, rtol=1e-13, atol=1e-14)


def test_splice_last_first_equals_ladder_bitwise():
    """n = N, m = 1: the splice chain X_1 .. X_{N-1}, K, Y_2 .. Y_M is exactly the ladder of the same pair."""
    rng = np.random.default_rng(9)
    for N, M in [(3, 3), (2, 4), (4, 2)]:
        X, Y, xr, yr = _case(rng, N, M, N, 1)
        a = oracle.tt_splice(X, Y, N, 1)
        b = oracle.tt_contract(X, Y, [N], [1])
        assert list(a["ranks"]) == list(b["ranks"]) and list(a["perm"]) == list(b["perm"])
        assert np.array_equal(a["flat"], b["flat"])


def test_splice_example1_shape():
    """Example 1 / Eq. 10: X of order 4, Y of order 3, contracted mode permuted to the front
    (Z^rho in R^{I4 x I2 x I1 x J1 x J3}); here with the modes already first: output dims (I4, I3, I2, J2, J3)
    in ladder order and (I2, I3, I4, J2, J3) after out_perm."""
    rng = np.random.default_rng(10)
    xd, yd = [3, 2, 4, 5], [3, 6, 2]
    X = ref.random_train(rng, xd, [1, 2, 3, 2, 1])
    Y = ref.random_train(rng, yd, [1, 2, 2, 1])
    res = oracle.tt_splice(X, Y, 1, 1)
    assert list(res["dims"]) == [5, 4, 2, 6, 2]
    assert _dense(res).shape == (2, 4, 5, 6, 2)


def test_splice_rejects_interior_modes():
    rng = np.random.default_rng(11)
    X, Y, _, _ = _case(rng, 3, 3, 1, 1)
    with pytest.raises(oracle.OracleError):
        oracle.tt_splice(X, Y, 2, 1)
