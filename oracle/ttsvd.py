"""O6 -- TT-SVD (Alg. 1) and the dense-input TTCP pipeline (Alg. 2 steps 1-6)
in plain numpy fp64.  TEST INFRASTRUCTURE ONLY (same rules as oracle/ttc_oracle.c: only tests/, smoke() and
bench.py's CPU legs use it; it shares nothing with the CUDA product).

Alg. 1, step by step in the paper's order and notation:
    delta = eps / sqrt(N - 1) * ||X||_F
    Z <- X_(1)                                    (mode-1 unfolding; little-endian)
    for n = 1 .. N-1:
        delta-truncated SVD  Z = U S V^T + E,  ||E||_F <= delta,  U in R^{R_{n-1} I_n x R_n}
        G^(n) <- reshape(U, [R_{n-1}, I_n, R_n])
        Z <- reshape(S V^T, [R_n I_{n+1}, I_{n+2} ... I_N])
    G^(N) <- Z
Readings: "USV" is U S V^T (R22); R_n is the SMALLEST rank whose discarded singular values satisfy
sum_{j > R_n} s_j^2 <= delta^2 (R23); singular vectors carry a sign convention -- the entry of largest magnitude
of every column of U is positive, the corresponding row of S V^T flipped with it (R24: the TT-SVD is unique only
up to these signs); singular values at or below 1e-7 of the largest count as zero (R25: the resolution of the
input data -- operands arrive in fp32, and rounding a tensor to fp32 moves its singular values by up to
||X - fl32(X)||_2 <= 2^-24 ||X||_F ~ 6e-8 ||X||_F (Weyl), so smaller ones are not determined by the input; pinned on
constructed spectra in tests/test_oracle_ttsvd.py), so eps = 0 returns the numerical TT ranks.
"""
import numpy as np

import oracle

SIGMA_FLOOR = 1e-7    # R25: relative to the largest singular value of the unfolding


def delta_rank(s, delta):
    """Smallest R with sum_{j >= R} s_j^2 <= delta^2 (s descending), ignoring s_j <= SIGMA_FLOOR * s_0 (R23, R25)."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0 or s[0] == 0.0:
        return 1
    keep = int(np.sum(s > SIGMA_FLOOR * s[0]))
    tail = np.concatenate([np.cumsum((s[::-1] ** 2))[::-1], [0.0]])   # tail[R] = sum_{j >= R} s_j^2
    R = keep
    while R > 1 and tail[R - 1] <= delta * delta:
        R -= 1
    return max(R, 1)


def tt_svd(X, eps: float):
    """Alg. 1: cores G^(1..N) of X (order N, dims X.shape) with ||X - TT||_F <= eps ||X||_F."""
    X = np.asarray(X, dtype=np.float64)
    dims = X.shape
    N = len(dims)
    if N == 1:
        return [X.reshape(1, dims[0], 1).copy()]
    delta = eps / np.sqrt(N - 1) * np.linalg.norm(X)
    Z = X.reshape(dims[0], -1, order="F")
    cores, R = [], 1
    for n in range(N - 1):
        U, s, Vt = np.linalg.svd(Z, full_matrices=False)
        Rn = delta_rank(s, delta)
        U, s, Vt = U[:, :Rn], s[:Rn], Vt[:Rn, :]
        for j in range(Rn):   # R24: largest-magnitude entry of every column of U positive
            k = int(np.argmax(np.abs(U[:, j])))
            if U[k, j] < 0:
                U[:, j] = -U[:, j]
                Vt[j, :] = -Vt[j, :]
        cores.append(U.reshape(R, dims[n], Rn, order="F"))
        SV = s[:, None] * Vt
        if n + 1 < N - 1:
            Z = SV.reshape(Rn * dims[n + 1], -1, order="F")
        else:
            Z = SV.reshape(Rn, dims[n + 1], order="F")
        R = Rn
    cores.append(Z.reshape(R, dims[N - 1], 1, order="F"))
    return cores


def ttcp_dense(X, Y, n: int, m: int, eps: float):
    """Alg. 2 with the TT-SVD of Alg. 1: permute the contracted modes to the front (step 1), decompose (steps 2-3),
    K = A_x^T A_y and the spliced chain (steps 4-5, oracle O5), reconstruct and permute to Eq. 8's order (steps
    5-6).  Returns Z = X x_n^m Y (approximately, within the truncation error)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    px = [n - 1] + [k for k in range(X.ndim) if k != n - 1]
    py = [m - 1] + [k for k in range(Y.ndim) if k != m - 1]
    Xr, Yr = np.transpose(X, px), np.transpose(Y, py)
    cx, cy = tt_svd(Xr, eps), tt_svd(Yr, eps)
    res = oracle.tt_splice(cx, cy, 1, 1)
    if res["order"] == 0:
        return np.asarray(res["cores"][0])
    return oracle.to_canonical(oracle.tt_reconstruct(res["cores"]), res["perm"])
