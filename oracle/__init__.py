"""fp64 CPU oracle for the TT contraction hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package.  The product (paper_2109_00626_b200/) never imports it and shares no code with it.

Pinned (tests/test_oracle_*.py) against: the paper's worked counts, SPEC.md's
worked examples, numpy einsum on every tiny shape, brute force, closed forms (rank-1 trains) and
invariants (<X,X> = ||X||_F^2, symmetry, reversal, O2 == O2').  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import complexity  # noqa: F401  (exact integer op counts)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "ttc_oracle.c")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        c_int, c_dp, c_i64pp = ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        L.oracle_tt_reconstruct.argtypes = [c_int, _i32p, _i32p, _f64p, _f64p]
        L.oracle_tcp.argtypes = [c_int, _i32p, ctypes.c_void_p, c_int, _i32p, ctypes.c_void_p, c_int, _i32p, _i32p,
                                 ctypes.c_void_p, c_i64pp]
        L.oracle_tt_inner.argtypes = [c_int, _i32p, _i32p, _f64p, _i32p, _f64p, c_dp, c_i64pp]
        L.oracle_tt_inner_partial.argtypes = [c_int, _i32p, _i32p, _f64p, _i32p, _f64p, c_int, _f64p]
        L.oracle_tt_inner_transfer.argtypes = [c_int, _i32p, _i32p, _f64p, _i32p, _f64p, c_dp]
        L.oracle_tt_contract.argtypes = [c_int, _i32p, _i32p, _f64p, c_int, _i32p, _i32p, _f64p, c_int, _i32p, _i32p,
                                         ctypes.POINTER(ctypes.c_int32), _i32p, _i32p, _i32p, _i32p, c_i64pp,
                                         ctypes.c_void_p, c_i64pp, c_i64pp]
        L.oracle_tt_splice.argtypes = [c_int, _i32p, _i32p, _f64p, c_int, _i32p, _i32p, _f64p, c_int, c_int,
                                       ctypes.POINTER(ctypes.c_int32), _i32p, _i32p, _i32p, _i32p, c_i64pp,
                                       ctypes.c_void_p]
        L.oracle_tt_inner_batch.argtypes = [c_int, c_int, _i32p, _i32p, _i64p, _f32p, _i32p, _i64p, _f32p, _f64p,
                                            c_int]
        L.oracle_tt_contract_batch.argtypes = [c_int, c_int, _i32p, _i32p, _i64p, _f32p, c_int, _i32p, _i32p, _i64p,
                                               _f32p, c_int, _i32p, _i32p, _i64p, _f64p, c_int]
        L.oracle_tt_splice_batch.argtypes = [c_int, c_int, _i32p, _i32p, _i64p, _f32p, c_int, _i32p, _i32p, _i64p,
                                             _f32p, c_int, c_int, _i64p, _f64p, c_int]
        L.oracle_max_threads.restype = c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _chk(rc):
    if rc != 0:
        raise OracleError({1: "bad argument", 2: "shape mismatch", 3: "bad modes", 4: "out of memory"}.get(rc, rc))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _train(cores):
    """list of (R_{n-1}, I_n, R_n) arrays -> (dims, ranks, flat fp64 in Eq. 2 order)."""
    dims = _i32([c.shape[1] for c in cores])
    ranks = _i32([cores[0].shape[0]] + [c.shape[2] for c in cores])
    flat = np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1, order="F") for c in cores])
    return dims, ranks, np.ascontiguousarray(flat)


def tt_reconstruct(cores) -> np.ndarray:
    """O1a: the dense tensor of a train by Eq. 9 (returned with Fortran order so that flat = Eq. 2 order)."""
    dims, ranks, flat = _train(cores)
    out = np.empty(int(np.prod(dims.astype(np.int64))), dtype=np.float64)
    _chk(lib().oracle_tt_reconstruct(len(dims), dims, ranks, flat, out))
    return out.reshape(tuple(dims), order="F")


def tcp(x: np.ndarray, y: np.ndarray, x_modes, y_modes, count_only: bool = False):
    """O1b: Eq. 8 over the disjoint 1-based mode pairs (x_modes[k], y_modes[k]); returns (Z, macs).

    Z's modes are in Eq. 8 order (X free ascending, then Y free ascending); a 0-d array when every mode is
    contracted.  count_only runs the loop nest without arithmetic (for the paper's 10^9 count)."""
    xd, yd = _i32(x.shape), _i32(y.shape)
    K = len(x_modes)
    xm, ym = _i32(list(x_modes) or [0]), _i32(list(y_modes) or [0])
    macs = ctypes.c_int64(0)
    freex = [d for n, d in enumerate(x.shape) if (n + 1) not in x_modes]
    freey = [d for m, d in enumerate(y.shape) if (m + 1) not in y_modes]
    zshape = tuple(freex + freey)
    if count_only:
        _chk(lib().oracle_tcp(len(xd), xd, None, len(yd), yd, None, K, xm, ym, None, ctypes.byref(macs)))
        return None, macs.value
    xf = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, order="F"))
    yf = np.ascontiguousarray(np.asarray(y, dtype=np.float64).reshape(-1, order="F"))
    z = np.empty(int(np.prod(zshape, dtype=np.int64)), dtype=np.float64)
    _chk(lib().oracle_tcp(len(xd), xd, xf.ctypes.data, len(yd), yd, yf.ctypes.data, K, xm, ym, z.ctypes.data,
                          ctypes.byref(macs)))
    return z.reshape(zshape, order="F"), macs.value


def tt_inner(xcores, ycores):
    """O2: <X, Y> by the core-by-core sweep; returns (value, macs)."""
    dims, xr, xf = _train(xcores)
    dims2, yr, yf = _train(ycores)
    if not np.array_equal(dims, dims2):
        raise OracleError("shape mismatch")
    v, macs = ctypes.c_double(0.0), ctypes.c_int64(0)
    _chk(lib().oracle_tt_inner(len(dims), dims, xr, xf, yr, yf, ctypes.byref(v), ctypes.byref(macs)))
    return v.value, macs.value


def tt_inner_partial(xcores, ycores, steps: int) -> np.ndarray:
    """O2 stopped after `steps` cores: Z_steps as an R_steps x P_steps matrix (Z_1 = A_x^T A_y, Eq. 12)."""
    dims, xr, xf = _train(xcores)
    _, yr, yf = _train(ycores)
    z = np.empty(int(xr[steps]) * int(yr[steps]), dtype=np.float64)
    _chk(lib().oracle_tt_inner_partial(len(dims), dims, xr, xf, yr, yf, steps, z))
    return z.reshape((int(xr[steps]), int(yr[steps])), order="F")


def tt_inner_transfer(xcores, ycores) -> float:
    """O2': <X, Y> by explicit transfer matrices E_n (a different association from O2)."""
    dims, xr, xf = _train(xcores)
    _, yr, yf = _train(ycores)
    v = ctypes.c_double(0.0)
    _chk(lib().oracle_tt_inner_transfer(len(dims), dims, xr, xf, yr, yf, ctypes.byref(v)))
    return v.value


def tt_contract(xcores, ycores, x_modes, y_modes, with_cores: bool = True):
    """O3: X x_{pairs} Y as a TT (ladder).  Returns dict(order, dims, ranks, src, perm, elems, cores, t_macs, a_macs)

    src[l] = +n (X mode n) / -m (Y mode m), 1-based; perm[c] = 1-based ladder position of canonical mode c;
    cores = list of (R_{l-1}, I_l, R_l) arrays (or [scalar] when every mode is contracted)."""
    xd, xr, xf = _train(xcores)
    yd, yr, yf = _train(ycores)
    K = len(x_modes)
    xm, ym = _i32(list(x_modes) or [0]), _i32(list(y_modes) or [0])
    Lmax = len(xd) + len(yd)
    L = ctypes.c_int32(0)
    od, ork, osrc, operm = (np.zeros(Lmax + 1, np.int32) for _ in range(4))
    ne, tm, am = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    lb = lib()
    _chk(lb.oracle_tt_contract(len(xd), xd, xr, xf, len(yd), yd, yr, yf, K, xm, ym, ctypes.byref(L), od, ork, osrc,
                               operm, ctypes.byref(ne), None, None, None))
    res = dict(order=L.value, dims=od[:L.value].copy(), ranks=ork[:L.value + 1].copy(), src=osrc[:L.value].copy(),
               perm=operm[:L.value].copy(), elems=ne.value)
    if with_cores:
        buf = np.zeros(ne.value, dtype=np.float64)
        _chk(lb.oracle_tt_contract(len(xd), xd, xr, xf, len(yd), yd, yr, yf, K, xm, ym, ctypes.byref(L), od, ork,
                                   osrc, operm, ctypes.byref(ne), buf.ctypes.data, ctypes.byref(tm),
                                   ctypes.byref(am)))
        cores, pos = [], 0
        if L.value == 0:
            cores = [buf[0]]
        for l in range(L.value):
            a, i, b = int(ork[l]), int(od[l]), int(ork[l + 1])
            cores.append(buf[pos:pos + a * i * b].reshape((a, i, b), order="F"))
            pos += a * i * b
        res.update(cores=cores, flat=buf, t_macs=tm.value, a_macs=am.value)
    return res


def tt_splice(xcores, ycores, n: int, m: int, with_cores: bool = True):
    """O5: X x_n^m Y for end modes (n in {1, N}, m in {1, M}, 1-based) as the paper's TTCP splice (Alg. 2 steps
    4-5).  Same result dict as tt_contract (order, dims, ranks, src, perm, elems, cores, flat)."""
    xd, xr, xf = _train(xcores)
    yd, yr, yf = _train(ycores)
    Lmax = len(xd) + len(yd)
    L = ctypes.c_int32(0)
    od, ork, osrc, operm = (np.zeros(Lmax + 1, np.int32) for _ in range(4))
    ne = ctypes.c_int64(0)
    lb = lib()
    _chk(lb.oracle_tt_splice(len(xd), xd, xr, xf, len(yd), yd, yr, yf, int(n), int(m), ctypes.byref(L), od, ork,
                             osrc, operm, ctypes.byref(ne), None))
    res = dict(order=L.value, dims=od[:L.value].copy(), ranks=ork[:L.value + 1].copy(), src=osrc[:L.value].copy(),
               perm=operm[:L.value].copy(), elems=ne.value)
    if with_cores:
        buf = np.zeros(ne.value, dtype=np.float64)
        _chk(lb.oracle_tt_splice(len(xd), xd, xr, xf, len(yd), yd, yr, yf, int(n), int(m), ctypes.byref(L), od, ork,
                                 osrc, operm, ctypes.byref(ne), buf.ctypes.data))
        cores, pos = [], 0
        if L.value == 0:
            cores = [buf[0]]
        for l in range(L.value):
            a, i, b = int(ork[l]), int(od[l]), int(ork[l + 1])
            cores.append(buf[pos:pos + a * i * b].reshape((a, i, b), order="F"))
            pos += a * i * b
        res.update(cores=cores, flat=buf)
    return res


def to_canonical(dense_ladder: np.ndarray, perm) -> np.ndarray:
    """Alg. 2 step 6: ladder-ordered dense Z -> Eq. 8 order (perm 1-based)."""
    return np.transpose(dense_ladder, [int(p) - 1 for p in perm])


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def tt_inner_batch(X, Y, nthreads: int = 0, first: int = 0, count: int = None) -> np.ndarray:
    """O2 over pairs first..first+count-1 of two ttgen.TTBatch objects (host fp32 cores, widened exactly)."""
    count = X.B - first if count is None else count
    xc = np.ascontiguousarray(X.cores.detach().cpu().numpy(), dtype=np.float32)
    yc = np.ascontiguousarray(Y.cores.detach().cpu().numpy(), dtype=np.float32)
    return tt_inner_batch_np(xc, yc, X, Y, nthreads, first, count)


def tt_inner_batch_np(xc, yc, X, Y, nthreads: int = 0, first: int = 0, count: int = None) -> np.ndarray:
    count = X.B - first if count is None else count
    out = np.zeros(count, dtype=np.float64)
    xr = np.ascontiguousarray(X.ranks[first:first + count], dtype=np.int32)
    yr = np.ascontiguousarray(Y.ranks[first:first + count], dtype=np.int32)
    xo = np.ascontiguousarray(X.offsets[first:first + count], dtype=np.int64)
    yo = np.ascontiguousarray(Y.offsets[first:first + count], dtype=np.int64)
    _chk(lib().oracle_tt_inner_batch(count, X.N, _i32(X.dims), xr, xo, xc, yr, yo, yc, out, nthreads))
    return out


def tt_contract_batch(X, Y, x_modes, y_modes, out_offsets, total, nthreads: int = 0, first: int = 0,
                      count: int = None) -> np.ndarray:
    """O3 over a batch; out_offsets[b] (relative to the returned buffer) from the caller's layout."""
    count = X.B - first if count is None else count
    xc = np.ascontiguousarray(X.cores.detach().cpu().numpy(), dtype=np.float32)
    yc = np.ascontiguousarray(Y.cores.detach().cpu().numpy(), dtype=np.float32)
    out = np.zeros(int(total), dtype=np.float64)
    _chk(lib().oracle_tt_contract_batch(
        count, X.N, _i32(X.dims), np.ascontiguousarray(X.ranks[first:first + count], np.int32),
        np.ascontiguousarray(X.offsets[first:first + count], np.int64), xc,
        Y.N, _i32(Y.dims), np.ascontiguousarray(Y.ranks[first:first + count], np.int32),
        np.ascontiguousarray(Y.offsets[first:first + count], np.int64), yc,
        len(x_modes), _i32(x_modes), _i32(y_modes), np.ascontiguousarray(out_offsets, np.int64), out, nthreads))
    return out


def tt_splice_batch(X, Y, n: int, m: int, out_offsets, total, nthreads: int = 0, first: int = 0,
                    count: int = None) -> np.ndarray:
    """O5 over a batch; out_offsets[b] (relative to the returned buffer) from the caller's layout."""
    count = X.B - first if count is None else count
    xc = np.ascontiguousarray(X.cores.detach().cpu().numpy(), dtype=np.float32)
    yc = np.ascontiguousarray(Y.cores.detach().cpu().numpy(), dtype=np.float32)
    out = np.zeros(int(total), dtype=np.float64)
    _chk(lib().oracle_tt_splice_batch(
        count, X.N, _i32(X.dims), np.ascontiguousarray(X.ranks[first:first + count], np.int32),
        np.ascontiguousarray(X.offsets[first:first + count], np.int64), xc,
        Y.N, _i32(Y.dims), np.ascontiguousarray(Y.ranks[first:first + count], np.int32),
        np.ascontiguousarray(Y.offsets[first:first + count], np.int64), yc,
        int(n), int(m), np.ascontiguousarray(out_offsets, np.int64), out, nthreads))
    return out


def normaliser(xcores, ycores) -> float:
    """||X||_F ||Y||_F with ||X||_F = sqrt(O2(X, X)) (SURVEY.md §8c error measure)."""
    return float(np.sqrt(max(tt_inner(xcores, xcores)[0], 0.0) * max(tt_inner(ycores, ycores)[0], 0.0)))
