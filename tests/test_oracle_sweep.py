"""Pins for oracle O2 (TT sweep) and O2' (explicit transfers): brute force through the dense definition,
closed forms and invariants (SURVEY.md §8c 'What pins each part')."""
import itertools

import numpy as np
import pytest

import oracle
import ttgen
from oracle import complexity as cx
from tests import ref_numpy as ref


def _rand_pair(rng, N, I_max=3, R_max=3):
    dims = list(rng.integers(1, I_max + 1, N))
    xr = [1] + list(rng.integers(1, R_max + 1, N - 1)) + [1]
    yr = [1] + list(rng.integers(1, R_max + 1, N - 1)) + [1]
    return dims, ref.random_train(rng, dims, xr), ref.random_train(rng, dims, yr)


def test_sweep_equals_dense_definition_exhaustive_tiny():
    """O2 == full contraction (Fig. 1b) of the Eq. 9 reconstructions, N <= 4, I <= 3, R, P <= 3."""
    rng = np.random.default_rng(10)
    n = 0
    for N in range(1, 5):
        for _ in range(40):
            dims, X, Y = _rand_pair(rng, N)
            v, macs = oracle.tt_inner(X, Y)
            dx, dy = ref.dense_from_tt(X), ref.dense_from_tt(Y)
            want = float(np.sum(dx * dy))
            assert abs(v - want) <= 1e-12 * max(1.0, np.linalg.norm(dx) * np.linalg.norm(dy))
            # and via the oracle's own dense path (O1)
            modes = list(range(1, N + 1))
            z, _ = oracle.tcp(oracle.tt_reconstruct(X), oracle.tt_reconstruct(Y), modes, modes)
            assert abs(v - float(z)) <= 1e-12 * max(1.0, np.linalg.norm(dx) * np.linalg.norm(dy))
            xr = [c.shape[0] for c in X] + [1]
            yr = [c.shape[0] for c in Y] + [1]
            assert macs == cx.sweep_macs(dims, xr, yr)
            n += 1
    assert n == 160


def test_c1_against_dense_reconstruction_and_tcp():
    """BASELINE.json configs[0] (C1): N=5, I=10, R=4 -- O2 against the 10^5-element dense contraction."""
    X, Y = ttgen.config_batch("C1")
    xc, yc = X.train(0), Y.train(0)
    v, macs = oracle.tt_inner(xc, yc)
    dx, dy = oracle.tt_reconstruct(xc), oracle.tt_reconstruct(yc)
    assert dx.size == 10 ** 5
    modes = [1, 2, 3, 4, 5]
    z, dmacs = oracle.tcp(dx, dy, modes, modes)
    assert dmacs == 10 ** 5
    assert abs(v - float(z)) <= 1e-12 * np.linalg.norm(dx) * np.linalg.norm(dy)
    np.testing.assert_allclose(dx, ref.dense_from_tt(xc), rtol=1e-12, atol=1e-15)
    assert macs == 4240  # SURVEY.md §8a closed form for C1


def test_z1_is_eq12_kernel():
    """Z_1 = A_x^T A_y (Eq. 12) with A_x = X_1 as I_1 x R_1."""
    rng = np.random.default_rng(11)
    dims, X, Y = _rand_pair(rng, 4, I_max=5, R_max=4)
    Z1 = oracle.tt_inner_partial(X, Y, 1)
    Ax, Ay = X[0][0], Y[0][0]
    np.testing.assert_allclose(Z1, Ax.T @ Ay, rtol=1e-13, atol=1e-14)


def test_inner_self_is_squared_frobenius_norm():
    rng = np.random.default_rng(12)
    for N in (1, 2, 3, 5):
        dims, X, _ = _rand_pair(rng, N, I_max=4, R_max=4)
        v, _ = oracle.tt_inner(X, X)
        d = ref.dense_from_tt(X)
        assert abs(v - float(np.sum(d * d))) <= 1e-12 * float(np.sum(d * d))


def test_symmetry_and_transfer_agreement():
    rng = np.random.default_rng(13)
    for N in (1, 2, 4, 7):
        dims, X, Y = _rand_pair(rng, N, I_max=4, R_max=5)
        a, _ = oracle.tt_inner(X, Y)
        b, _ = oracle.tt_inner(Y, X)
        c = oracle.tt_inner_transfer(X, Y)
        scale = np.sqrt(oracle.tt_inner(X, X)[0] * oracle.tt_inner(Y, Y)[0])
        assert abs(a - b) <= 1e-13 * scale
        assert abs(a - c) <= 1e-13 * scale


def test_rank1_closed_form():
    """Rank-1 trains: <X, Y> = prod_n <x_n, y_n>."""
    rng = np.random.default_rng(14)
    for N in (1, 3, 6):
        xs = [rng.standard_normal(3) for _ in range(N)]
        ys = [rng.standard_normal(3) for _ in range(N)]
        v, _ = oracle.tt_inner([x.reshape(1, -1, 1) for x in xs], [y.reshape(1, -1, 1) for y in ys])
        want = np.prod([x @ y for x, y in zip(xs, ys)])
        assert abs(v - want) <= 1e-13 * max(1.0, abs(want))


def test_rank1_embedded_in_full_rank_storage():
    """ttgen 'rank1' kind: only [0, i, 0] nonzero in R x I x R cores -> same closed form."""
    X, Y = ttgen.make_pair("rank1", 1, 2, 0, ttgen.uniform_ranks(3, 5, 4), (3,) * 5)
    for b in range(3):
        xc, yc = X.train(b), Y.train(b)
        want = np.prod([xc[n][0, :, 0] @ yc[n][0, :, 0] for n in range(5)])
        v, _ = oracle.tt_inner(xc, yc)
        assert abs(v - want) <= 1e-13 * max(1e-3, abs(want))


def test_tagged_pairs_give_their_index():
    X, Y = ttgen.make_pair("tagged", 1, 2, 5, ttgen.uniform_ranks(4, 6, 3), (2,) * 6)
    for b in range(4):
        assert oracle.tt_inner(X.train(b), Y.train(b))[0] == 5 + b


def test_orthogonal_first_cores_give_zero():
    """columns of A_x orthogonal to those of A_y -> K = 0 -> <X,Y> = 0 exactly."""
    rng = np.random.default_rng(15)
    dims, X, Y = _rand_pair(rng, 4, I_max=3, R_max=3)
    dims[0] = 4
    X[0] = np.zeros((1, 4, X[0].shape[2])); X[0][0, :2, :] = rng.standard_normal((2, X[0].shape[2]))
    Y[0] = np.zeros((1, 4, Y[0].shape[2])); Y[0][0, 2:, :] = rng.standard_normal((2, Y[0].shape[2]))
    assert oracle.tt_inner(X, Y)[0] == 0.0


def test_reversal_invariance():
    """Reversing both trains (core n -> N+1-n, rank modes swapped) reverses the modes of both tensors,
    which leaves the full contraction unchanged."""
    rng = np.random.default_rng(16)
    dims, X, Y = _rand_pair(rng, 5, I_max=3, R_max=4)
    rev = lambda T: [np.transpose(c, (2, 1, 0)) for c in T[::-1]]
    a, _ = oracle.tt_inner(X, Y)
    b, _ = oracle.tt_inner(rev(X), rev(Y))
    assert abs(a - b) <= 1e-13 * np.sqrt(oracle.tt_inner(X, X)[0] * oracle.tt_inner(Y, Y)[0])


def test_core_scaling_is_exact():
    rng = np.random.default_rng(17)
    dims, X, Y = _rand_pair(rng, 4, I_max=3, R_max=3)
    a, _ = oracle.tt_inner(X, Y)
    X2 = [c.copy() for c in X]
    X2[2] = X2[2] * 2.0
    assert oracle.tt_inner(X2, Y)[0] == 2.0 * a


def test_batch_matches_single_and_widening_is_exact():
    X, Y = ttgen.config_batch("C5", B=3)
    out = oracle.tt_inner_batch(X, Y, nthreads=2)
    for b in range(3):
        assert out[b] == oracle.tt_inner(X.train(b), Y.train(b))[0]


def test_sweep_macs_closed_forms():
    """C2 795,136 and C4 29,393,408 MACs per pair (uniform ranks: W-first == min order)."""
    for cfg, want in (("C1", 4240), ("C2", 795136), ("C4", 29393408)):
        c = ttgen.CONFIGS[cfg]
        r = [1] + [c["R"]] * (c["N"] - 1) + [1]
        assert cx.sweep_macs([c["I"]] * c["N"], r, r) == want
