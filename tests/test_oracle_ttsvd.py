"""Pins for oracle O6 (TT-SVD, Alg. 1, and the dense-input TTCP pipeline, Alg. 2): exact reconstruction at eps = 0,
Alg. 1's error guarantee ||X - TT(X)|| <= eps ||X||, the minimality of every delta-truncated rank (checked on the
singular values directly), recovery of the ranks of a tensor built from a low-rank train, left-orthonormal cores,
the rank bound R_n <= min(R_{n-1} I_n, prod_{k>n} I_k), and Alg. 2 == Eq. 8 (O1b / numpy)."""
import numpy as np
import pytest

import oracle
from oracle import ttsvd
from tests import ref_numpy as ref


def _dense(cores):
    return ref.dense_from_tt(cores)


@pytest.mark.parametrize("dims", [(5,), (4, 6), (3, 4, 5), (20, 20, 20), (2, 3, 4, 3, 2), (6, 1, 5)])
def test_exact_at_eps_zero(dims):
    X = np.random.default_rng(sum(dims)).standard_normal(dims)
    cores = ttsvd.tt_svd(X, 0.0)
    np.testing.assert_allclose(_dense(cores), X, rtol=1e-10, atol=1e-10)
    # left-orthonormal cores, rank bound, boundary ranks
    R = [c.shape[0] for c in cores] + [1]
    assert R[0] == 1 and R[-1] == 1
    for n, c in enumerate(cores[:-1]):
        U = c.reshape(-1, c.shape[2], order="F")
        np.testing.assert_allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-10)
        assert R[n + 1] <= min(R[n] * dims[n], int(np.prod(dims[n + 1:])))


@pytest.mark.parametrize("eps", [0.05, 0.2, 0.5])
def test_error_guarantee_and_minimal_ranks(eps):
    """Alg. 1 guarantees ||X - TT||_F <= eps ||X||_F; every truncation keeps the fewest singular values allowed."""
    rng = np.random.default_rng(int(eps * 100))
    X = rng.standard_normal((6, 7, 5, 4))
    cores = ttsvd.tt_svd(X, eps)
    err = np.linalg.norm(_dense(cores) - X)
    assert err <= eps * np.linalg.norm(X) * (1 + 1e-12)
    # replay the unfoldings and check minimality at each step
    delta = eps / np.sqrt(3) * np.linalg.norm(X)
    Z = X.reshape(6, -1, order="F")
    for n in range(3):
        s = np.linalg.svd(Z, compute_uv=False)
        Rn = cores[n].shape[2]
        assert np.sum(s[Rn:] ** 2) <= delta ** 2 * (1 + 1e-12)
        if Rn > 1:
            assert np.sum(s[Rn - 1:] ** 2) > delta ** 2
        U = cores[n].reshape(-1, Rn, order="F")
        Z = (U.T @ Z).reshape(Rn * X.shape[n + 1], -1, order="F") if n < 2 else U.T @ Z


def test_recovers_ranks_of_a_low_rank_train():
    rng = np.random.default_rng(3)
    dims, ranks = (6, 5, 7, 4), [1, 3, 4, 2, 1]
    X = _dense(ref.random_train(rng, dims, ranks))
    cores = ttsvd.tt_svd(X, 1e-9)
    assert [c.shape[0] for c in cores] + [1] == ranks
    np.testing.assert_allclose(_dense(cores), X, rtol=1e-9, atol=1e-9)


def test_sign_convention():
    """R24: the largest-magnitude entry of every left singular vector is positive."""
    X = np.random.default_rng(4).standard_normal((5, 6, 7))
    for c in ttsvd.tt_svd(X, 0.0)[:-1]:
        U = c.reshape(-1, c.shape[2], order="F")
        for j in range(U.shape[1]):
            assert U[np.argmax(np.abs(U[:, j])), j] > 0


@pytest.mark.parametrize("shape_x,shape_y,n,m", [((20, 20, 20), (20, 20, 20), 1, 1), ((4, 5, 6), (6, 3), 3, 1),
                                                 ((3, 4), (5, 4, 2), 2, 2), ((4, 3, 5, 2), (2, 5, 3), 3, 2)])
def test_alg2_equals_eq8(shape_x, shape_y, n, m):
    """Alg. 2 (permutation, TT-SVD, K, splice, reconstruction, permutation) == Eq. 8 at eps = 0; within the
    truncation bound (2 eps + eps^2) ||X|| ||Y|| at eps > 0 (Example 2's x_1^1 on 20 x 20 x 20 included)."""
    rng = np.random.default_rng(sum(shape_x) + n)
    X, Y = rng.standard_normal(shape_x), rng.standard_normal(shape_y)
    want = ref.tcp(X, Y, [n], [m])
    got = ttsvd.ttcp_dense(X, Y, n, m, 0.0)
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9)
    z1, _ = oracle.tcp(X, Y, [n], [m])
    np.testing.assert_allclose(got, z1, rtol=1e-9, atol=1e-9)
    for eps in (0.1, 0.3):
        got = ttsvd.ttcp_dense(X, Y, n, m, eps)
        assert np.linalg.norm(got - want) <= (2 * eps + eps ** 2) * np.linalg.norm(X) * np.linalg.norm(Y)


@pytest.mark.parametrize("spectrum,want", [((1.0, 1e-5, 1e-9), 2), ((1.0, 3e-7, 3e-8), 2), ((1.0, 0.5, 2e-7), 3)])
def test_sigma_floor_on_constructed_spectra(spectrum, want):
    """R25 pinned on spectra that straddle the floor: singular values of the first unfolding above 1e-7 sigma_max
    are kept at eps = 0 (1e-5, 3e-7, 2e-7), those below it are dropped (1e-9, 3e-8) -- on the fp64 tensor and on
    its fp32 rounding (what a GPU caller passes: the rounding adds singular values near 1e-8, below the floor).
    The kept part reconstructs the tensor to the dropped singular value (Eckart-Young: ||X - X_R|| = s_R)."""
    rng = np.random.default_rng(int(1e3 * spectrum[1]) + len(spectrum))
    X = ref.tensor_with_unfolding_spectrum(rng, (20, 20, 20), spectrum)
    s = np.linalg.svd(X.reshape(20, -1, order="F"), compute_uv=False)
    np.testing.assert_allclose(s[:3], spectrum, rtol=1e-6, atol=1e-15)
    for Xin in (X, X.astype(np.float32).astype(np.float64)):
        cores = ttsvd.tt_svd(Xin, 0.0)
        assert cores[0].shape[2] == want
        dropped = spectrum[want] if want < len(spectrum) else 0.0
        err = np.linalg.norm(_dense(cores) - Xin)
        assert err <= dropped + 1e-7 * np.linalg.norm(Xin)


def test_sigma_floor_is_fp32_input_resolution():
    """R25's floor is the resolution of fp32 input data: rounding a tensor to fp32 moves its singular values by at
    most ||X - fl32(X)||_2 <= ||X - fl32(X)||_F <= 2^-24 ||X||_F (Weyl), and for a rank-1 unfolding sigma_max =
    ||X||_F, so 2^-24 = 6e-8 < 1e-7: spurious singular values created by the rounding never pass the floor."""
    rng = np.random.default_rng(9)
    for dims in ((20, 20, 20), (8, 50, 20), (40, 10, 20)):
        X = ref.tensor_with_unfolding_spectrum(rng, dims, (1.0,))
        X32 = X.astype(np.float32).astype(np.float64)
        assert np.linalg.norm(X - X32) <= 2.0 ** -24 * np.linalg.norm(X)
        s = np.linalg.svd(X32.reshape(dims[0], -1, order="F"), compute_uv=False)
        assert s[1] < ttsvd.SIGMA_FLOOR * s[0]
        assert [c.shape[2] for c in ttsvd.tt_svd(X32, 0.0)[:1]] == [1]
