"""Exact operation-count models of §IV -- TEST INFRASTRUCTURE ONLY.

MAC = 1 operation (Fig. 4's 25000 = R*I*P).  Python ints: 10^27 does not fit
in 64 bits.  The sweep count is the full tt_inner cost (W-first association, the order oracle O2 runs),
which the paper does not cost (it costs the K step only; reading R18).
"""
from __future__ import annotations

from math import prod


def tcp_ops(x_shape, y_shape, n: int, m: int) -> int:
    """Dense x_n^m: I_1..I_N (all of X) times the non-contracted J's."""
    if x_shape[n - 1] != y_shape[m - 1]:
        raise ValueError(f"contracted dimension mismatch: I_{n}={x_shape[n - 1]} vs J_{m}={y_shape[m - 1]}")
    return prod(int(d) for d in x_shape) * prod(int(d) for k, d in enumerate(y_shape) if k != m - 1)


def tcp_ops_uniform(I: int, N: int) -> int:
    """O(I^{2N-1})."""
    return I ** (2 * N - 1)


def ttcp_ops(I_n: int, R1: int, P1: int) -> int:
    """The K = A_x^T A_y step, R_1 I_n P_1 MACs (Alg. 2 step 4)."""
    return R1 * I_n * P1


def ttd_ops(I: int, N: int, R: int) -> int:
    """TT-SVD extra cost O(I^{N-1} R^2) (Remark 3)."""
    return I ** (N - 1) * R * R


def speedup_ratio(I: int, N: int, R: int) -> int:
    """I^{2N-1} / (I R^2) as an integer quotient (Remark 3)."""
    return tcp_ops_uniform(I, N) // ttcp_ops(I, R, R)


def sweep_macs(dims, xr, yr) -> int:
    """MACs of the O2 sweep: sum_n R_{n-1}P_{n-1}I_nP_n + R_{n-1}I_nR_nP_n."""
    return sum(xr[n] * yr[n] * dims[n] * yr[n + 1] + xr[n] * dims[n] * xr[n + 1] * yr[n + 1] for n in range(len(dims)))
