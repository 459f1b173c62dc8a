"""Pins for oracle O1 (dense Eq. 9 reconstruction, dense Eq. 8 TCP) and the exact op-count model.

Every check compares the oracle with something other than itself: the paper's printed counts, SPEC.md's
worked examples, brute-force python loops, or numpy tensordot (tests/ref_numpy.py).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from oracle import complexity as cx
from tests import ref_numpy as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_eq2_linear_index_spec_example():
    """(3,2,4) in [3,4,5] -> 42.  Storage = Eq. 2 order; contracting with a one-hot tensor over
    all modes (Fig. 1b 'contraction along all modes') reads exactly one stored element."""
    g = _gold("spec_examples.json")
    for key in ("linear_index", "linear_index_2"):
        e = g[key]
        shape = tuple(e["shape"])
        x = np.arange(1, np.prod(shape) + 1, dtype=np.float64).reshape(shape, order="F")  # value = 1-based position
        sel = np.zeros(shape)
        sel[tuple(i - 1 for i in e["multi"])] = 1.0
        modes = list(range(1, len(shape) + 1))
        z, macs = oracle.tcp(x, sel, modes, modes)
        assert float(z) == e["value"]
        assert macs == np.prod(shape)


def test_tcp_matrices_is_matmul_and_vectors_is_dot():
    """SPEC.md:115-116 / Fig. 1b: x_2^1 of matrices is the matrix product; vectors: dot."""
    rng = np.random.default_rng(1)
    A, B = rng.standard_normal((3, 4)), rng.standard_normal((4, 5))
    z, macs = oracle.tcp(A, B, [2], [1])
    np.testing.assert_allclose(z, A @ B, rtol=1e-13, atol=1e-13)
    assert macs == 3 * 4 * 5
    u, v = rng.standard_normal(7), rng.standard_normal(7)
    z, macs = oracle.tcp(u, v, [1], [1])
    assert z.shape == () and abs(float(z) - float(u @ v)) < 1e-13 and macs == 7


def test_tcp_spec_shape_example_vs_bruteforce():
    """x in R^{2x3x4}, y in R^{3x5}, (n,m)=(2,1) -> shape (2,4,5), checked against explicit loops."""
    e = _gold("spec_examples.json")["tcp_shape"]
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(e["x_shape"]), rng.standard_normal(e["y_shape"])
    z, _ = oracle.tcp(x, y, [e["n"]], [e["m"]])
    assert list(z.shape) == e["z_shape"]
    for a, c, d in itertools.product(range(2), range(4), range(5)):
        s = sum(x[a, k, c] * y[k, d] for k in range(3))
        assert abs(z[a, c, d] - s) < 1e-13


def test_tcp_eq10_shape_law():
    """PAPER.md:294-296 (Eq. 10): X x_3^2 Y in R^{I1 x I2 x I4 x J1 x J3}."""
    e = _gold("spec_examples.json")["eq10_shape"]
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(e["x_shape"]), rng.standard_normal(e["y_shape"])
    z, _ = oracle.tcp(x, y, [e["n"]], [e["m"]])
    assert list(z.shape) == e["z_shape"]
    np.testing.assert_allclose(z, ref.tcp(x, y, [3], [2]), rtol=1e-12, atol=1e-12)


def _shapes(max_order=3, max_dim=3):
    for N in range(1, max_order + 1):
        for dims in itertools.product(range(1, max_dim + 1), repeat=N):
            yield dims


@pytest.mark.parametrize("seed", [0, 1])
def test_tcp_vs_numpy_all_pair_sets(seed):
    """Eq. 8 extended to K disjoint pairs, every mode-pair set of small X, Y, against numpy tensordot."""
    rng = np.random.default_rng(seed)
    cases = 0
    for N, M in [(1, 1), (1, 2), (2, 2), (2, 3), (3, 2), (3, 3), (4, 3), (3, 4)]:
        xd = tuple(rng.integers(1, 4, N))
        for K in range(0, min(N, M) + 1):
            for xm in itertools.combinations(range(1, N + 1), K):
                for ym in itertools.permutations(range(1, M + 1), K):
                    yd = [int(rng.integers(1, 4)) for _ in range(M)]
                    for a, b in zip(xm, ym):
                        yd[b - 1] = xd[a - 1]
                    x, y = rng.standard_normal(xd), rng.standard_normal(yd)
                    z, macs = oracle.tcp(x, y, list(xm), list(ym))
                    np.testing.assert_allclose(z, ref.tcp(x, y, xm, ym), rtol=1e-12, atol=1e-12)
                    assert macs == int(np.prod(z.shape, dtype=np.int64)) * int(np.prod([xd[a - 1] for a in xm]))
                    cases += 1
    assert cases > 200


def test_tcp_shape_errors():
    x, y = np.zeros((2, 3)), np.zeros((4, 5))
    with pytest.raises(oracle.OracleError):
        oracle.tcp(x, y, [2], [1])          # I_2 = 3 != J_1 = 4


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_reconstruct_vs_numpy(seed):
    """O1a (Eq. 9) against numpy tensordot chains on random tiny trains."""
    rng = np.random.default_rng(seed)
    for N in range(1, 5):
        for _ in range(6):
            dims = list(rng.integers(1, 4, N))
            ranks = [1] + list(rng.integers(1, 4, N - 1)) + [1]
            cores = ref.random_train(rng, dims, ranks)
            np.testing.assert_allclose(oracle.tt_reconstruct(cores), ref.dense_from_tt(cores), rtol=1e-12, atol=1e-12)


def test_reconstruct_rank1_is_outer_product():
    """Closed form: a rank-1 TT is the outer product of its mode vectors."""
    rng = np.random.default_rng(5)
    vs = [rng.standard_normal(d) for d in (3, 2, 4)]
    cores = [v.reshape(1, -1, 1) for v in vs]
    np.testing.assert_allclose(oracle.tt_reconstruct(cores), np.einsum("a,b,c->abc", *vs), rtol=1e-14)


def test_paper_counts_exact():
    """PAPER.md:63, 442, 459 printed counts, as exact integers (complexity model)."""
    g = _gold("paper_counts.json")
    assert cx.tcp_ops_uniform(10, 5) == g["tcp_order5_I10"]["value"]
    assert cx.tcp_ops((10,) * 5, (10,) * 5, 1, 1) == g["tcp_order5_I10"]["value"]
    assert cx.tcp_ops_uniform(1000, 5) == int(g["tcp_order5_I1000"]["value"])
    assert cx.ttcp_ops(1000, 5, 5) == g["ttcp_I1000_R5"]["value"]
    assert cx.ttcp_ops(1000, 2, 2) == g["ttcp_I1000_R2"]["value"]
    assert cx.speedup_ratio(1000, 5, 5) == int(g["speedup_I1000_N5_R5"]["value"])
    assert cx.ttd_ops(1000, 5, 5) == g["ttd_I1000_N5_R5"]["value"]


@pytest.mark.slow
def test_paper_tcp_count_by_running_the_loops():
    """the dense x_n^m of two order-5, I=10 tensors runs 10^9 multiply-adds -- counted by
    executing the oracle's Eq. 8 loop nest (count-only mode, no arithmetic)."""
    x = np.zeros((10,) * 5)
    _, macs = oracle.tcp(x, x, [3], [1], count_only=True)
    assert macs == _gold("paper_counts.json")["tcp_order5_I10"]["value"]
