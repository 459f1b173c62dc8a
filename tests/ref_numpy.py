"""Independent numpy float64 cross-checks of the oracle -- test infrastructure.

Uses numpy's own multi-index semantics (tensordot/einsum), never the oracle's index arithmetic, so a
wrong stride, sign or transposed operand in oracle/ttc_oracle.c shows up as a mismatch here.
"""
import numpy as np


def dense_from_tt(cores):
    """Eq. 9: G1 x G2 x ... contracted over consecutive rank modes."""
    T = np.asarray(cores[0], dtype=np.float64)          # (1, I1, R1)
    for c in cores[1:]:
        T = np.tensordot(T, np.asarray(c, dtype=np.float64), axes=([-1], [0]))
    return T.reshape(T.shape[1:-1])                     # drop R_0 = R_N = 1


def tcp(x, y, x_modes, y_modes):
    """Eq. 8 over disjoint 1-based mode pairs; output X free then Y free modes."""
    return np.tensordot(np.asarray(x, np.float64), np.asarray(y, np.float64),
                        axes=([m - 1 for m in x_modes], [m - 1 for m in y_modes]))


def random_train(rng, dims, ranks, scale=1.0):
    return [rng.standard_normal((ranks[n], dims[n], ranks[n + 1])) * scale for n in range(len(dims))]


def tensor_with_unfolding_spectrum(rng, dims, s):
    """A dense tensor (Eq. 2 order) whose mode-1 unfolding X_(1) (I_1 x prod_{k>1} I_k) has exactly the singular
    values s: X_(1) = U diag(s) V^T with U, V orthonormal columns from QR of Gaussian matrices."""
    s = np.asarray(s, dtype=np.float64)
    m, n = dims[0], int(np.prod(dims[1:]))
    U, _ = np.linalg.qr(rng.standard_normal((m, s.size)))
    V, _ = np.linalg.qr(rng.standard_normal((n, s.size)))
    return (U @ np.diag(s) @ V.T).reshape(dims, order="F")
