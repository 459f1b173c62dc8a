"""Seeded synthetic Tensor-Train inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no contraction, no sweep, no transfer): it only draws
TT cores and rank profiles and lays them out in the storage convention both sides agree on.

Storage convention (Def. 2 / Eq. 2, little-endian: first index fastest):
  core n of a train is an order-3 array R_{n-1} x I_n x R_n (Def. 7 / Eq. 9, PAPER.md:158-165,
  boundary ranks R_0 = R_N = 1) whose element [r, i, s] lives at r + R_{n-1}*(i + I_n*s);
  a train is its N cores concatenated in core order; a batch is B trains, train b starting at offsets[b].

Workload recipe: the paper's only experiment draws zero-mean Gaussian
tensors (Example 2); BASELINE.json's configs are Gaussian TT cores.  Variances:
  uniform configs      sigma_n^2 = 1 / (I * R)                (BASELINE.json configs[0..3])
  heterogeneous ranks  sigma_n^2 = 1 / (I_n * sqrt(R_{n-1} R_n))  (SURVEY.md §8c Q13 reading)
Validation kinds that make the 1e-4 criterion non-vacuous:
  iid, self (Y := X), corr (Y_n = X_n + 0.1 * noise), int (cores in {-1,0,1}), rank1 (only [0,i,0]
  nonzero: closed form), tagged (rank-1 embedded, <X_b, Y_b> = b exactly).
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional, Sequence

import numpy as np
import torch

# BASELINE.json "configs", labelled C1..C5 as in SURVEY.md §0.
CONFIGS = {
    "C1": dict(op="inner", B=1, N=5, I=10, R=4),
    "C2": dict(op="inner", B=4096, N=8, I=16, R=16),
    "C3": dict(op="contract", B=1024, N=6, M=6, I=8, R=8, P=8, x_modes=(2, 4, 6), y_modes=(1, 3, 5)),
    "C4": dict(op="inner", B=8192, N=16, I=4, R=64),
    "C5": dict(op="inner", B=65536, N=64, I=2, rank_choices=(8, 16, 24, 32)),
    # SURVEY.md §8f NEXT-1 (not a BASELINE.json config): the paper's TTCP splice of end modes on C3's operands,
    # contracting X mode 1 with Y mode 1 (Example 2's x_1^1, on TT operands)
    "S1": dict(op="splice", B=16384, N=6, M=6, I=8, R=8, P=8, x_mode=1, y_mode=1),
    # SURVEY.md §8f NEXT-2 (not a BASELINE.json config): dense reconstruction (Alg. 2 steps 5-6) of Example 2's
    # TTCP output -- x_1^1 of two 20 x 20 x 20 tensors in TT format with ranks 20 is an order-4 train with
    # I = 20 and bonds 20 -- 160,000 floats per train
    "R1": dict(op="reconstruct", B=1024, N=4, I=20, R=20),
    # the whole dense-input TTCP of Alg. 2 on Example 2 case (i): pairs of
    # zero-mean unit-variance Gaussian 20 x 20 x 20 tensors, x_1^1, TT-SVD at eps = 0 (full ranks 20)
    "A2": dict(op="alg2", B=1024, N=3, I=20, shape=(20, 20, 20), x_mode=1, y_mode=1, eps=0.0),
    # Example 2 cases (ii) and (iii): 20 x 20 x 20 x 5 and 20 x 20 x 20 x 5 x 4 (full TT ranks [1, 20, 100, 5, 1]
    # and [1, 20, 400, 20, 4, 1]; TTCP outputs of 4,000,000 and 64,000,000 entries per pair)
    "A2ii": dict(op="alg2", B=64, N=4, I=20, shape=(20, 20, 20, 5), x_mode=1, y_mode=1, eps=0.0),
    "A2iii": dict(op="alg2", B=8, N=5, I=20, shape=(20, 20, 20, 5, 4), x_mode=1, y_mode=1, eps=0.0),
}
CFG_ID = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "S1": 6, "R1": 7, "A2": 8, "A2ii": 9, "A2iii": 10}


def alg2_shape(cfg: str):
    """Dense operand shape of an "alg2" workload."""
    c = CONFIGS[cfg]
    return tuple(c.get("shape", (c["I"],) * c["N"]))

DEFAULT_SEED = 20210901  # arXiv 2109.00626 submission month; recorded in every bench line
SIDE_X, SIDE_Y = 0, 1


@dataclasses.dataclass
class TTBatch:
    """B tensor trains of a common order N and mode sizes dims, possibly different ranks per train."""
    cores: torch.Tensor          # float32, flat, device or host
    ranks: np.ndarray            # int32 [B, N+1], row b = R_0..R_N (R_0 = R_N = 1)
    offsets: np.ndarray          # int64 [B], element offset of train b in `cores`
    dims: tuple                  # (I_1..I_N)

    @property
    def B(self) -> int:
        return int(self.ranks.shape[0])

    @property
    def N(self) -> int:
        return len(self.dims)

    def uniform_rank(self) -> Optional[int]:
        """Interior rank if every train has ranks (1, R, ..., R, 1), else None."""
        if self.B == 0:
            return None
        r = self.ranks
        if self.N == 1:
            return 1
        inner = r[:, 1:-1]
        v = int(inner.flat[0])
        return v if bool(np.all(inner == v)) else None

    def train(self, b: int):
        """Host float64 cores of train b as a list of (R_{n-1}, I_n, R_n) arrays in Eq. 2 order."""
        flat = self.cores[int(self.offsets[b]): int(self.offsets[b]) + train_elems(self.ranks[b], self.dims)]
        flat = flat.detach().to("cpu").numpy().astype(np.float64)
        out, pos = [], 0
        for n, I in enumerate(self.dims):
            r0, r1 = int(self.ranks[b, n]), int(self.ranks[b, n + 1])
            sz = r0 * I * r1
            out.append(flat[pos:pos + sz].reshape((r0, I, r1), order="F"))
            pos += sz
        return out

    def to(self, device) -> "TTBatch":
        return TTBatch(self.cores.to(device), self.ranks, self.offsets, self.dims)


def core_sizes(ranks_row, dims) -> list:
    return [int(ranks_row[n]) * int(dims[n]) * int(ranks_row[n + 1]) for n in range(len(dims))]


def train_elems(ranks_row, dims) -> int:
    return int(sum(core_sizes(ranks_row, dims)))


def packed_offsets(ranks: np.ndarray, dims) -> tuple:
    """Offsets of B packed trains (train b right after train b-1) and the total element count."""
    dims_a = np.asarray(dims, dtype=np.int64)
    r = ranks.astype(np.int64)
    sizes = (r[:, :-1] * dims_a[None, :] * r[:, 1:]).sum(axis=1) if r.shape[0] else np.zeros(0, np.int64)
    offs = np.zeros(r.shape[0], dtype=np.int64)
    if r.shape[0] > 1:
        offs[1:] = np.cumsum(sizes)[:-1]
    return offs, int(sizes.sum())


def uniform_ranks(B: int, N: int, R: int) -> np.ndarray:
    r = np.full((B, N + 1), R, dtype=np.int32)
    r[:, 0] = 1
    r[:, N] = 1
    return r


def _seed(*parts) -> int:
    h = hashlib.sha256(",".join(str(int(p)) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def random_ranks(seed: int, cfg_id: int, side: int, b0: int, B: int, N: int, choices: Sequence[int]) -> np.ndarray:
    """Per pair, per operand, per bond iid uniform draw from `choices`; R_0 = R_N = 1."""
    out = np.empty((B, N + 1), dtype=np.int32)
    ch = np.asarray(choices, dtype=np.int32)
    for j in range(B):
        rng = np.random.default_rng(np.random.SeedSequence([seed, cfg_id, b0 + j, side, 1]))
        out[j, 1:N] = ch[rng.integers(0, len(ch), size=N - 1)]
    out[:, 0] = 1
    out[:, N] = 1
    return out


def _scales(ranks: np.ndarray, dims, rule: str) -> np.ndarray:
    """Per (train, core) standard deviation of the Gaussian entries."""
    dims_a = np.asarray(dims, dtype=np.float64)[None, :]
    r = ranks.astype(np.float64)
    if rule == "uniform":  # 1/(I*R) with R the interior rank (max of the two bonds)
        R = np.maximum(r[:, :-1], r[:, 1:])
        return 1.0 / np.sqrt(dims_a * R)
    if rule == "geo":      # 1/(I_n sqrt(R_{n-1} R_n))
        return 1.0 / np.sqrt(dims_a * np.sqrt(r[:, :-1] * r[:, 1:]))
    if rule == "unit":
        return np.ones_like(r[:, :-1] * dims_a)
    raise ValueError(rule)


def gaussian_batch(seed: int, cfg_id: int, side: int, b0: int, ranks: np.ndarray, dims, rule: str = "uniform",
                   device="cpu") -> TTBatch:
    """iid Gaussian cores for pairs b0..b0+B-1 (ranks row j belongs to pair b0+j), generated on `device`.

    Pair b's values depend only on (seed, cfg_id, side, b, its rank row), so every shard of a batch
    regenerates exactly the data the unsharded batch holds for those pairs."""
    B = ranks.shape[0]
    offs, total = packed_offsets(ranks, dims)
    cores = torch.empty(total, dtype=torch.float32, device=device)
    if B == 0:
        return TTBatch(cores, ranks.copy(), offs, tuple(int(d) for d in dims))
    dims_l = [int(d) for d in dims]
    sizes = (ranks[:, :-1].astype(np.int64) * np.asarray(dims_l, np.int64)[None, :] * ranks[:, 1:])
    scl = _scales(ranks, dims_l, rule)
    for j in range(B):
        gp = torch.Generator(device=device)
        gp.manual_seed(_seed(seed, cfg_id, side, b0 + j))
        n_el = int(sizes[j].sum())
        cores[int(offs[j]): int(offs[j]) + n_el] = torch.randn(n_el, generator=gp, dtype=torch.float32, device=device)
    # per-element scale: one vectorised pass per chunk of pairs
    CH = 4096
    for j0 in range(0, B, CH):
        j1 = min(B, j0 + CH)
        s = torch.as_tensor(scl[j0:j1].reshape(-1), dtype=torch.float32, device=device)
        rep = torch.as_tensor(sizes[j0:j1].reshape(-1), dtype=torch.int64, device=device)
        lo = int(offs[j0])
        hi = int(offs[j1 - 1] + sizes[j1 - 1].sum())
        cores[lo:hi] *= torch.repeat_interleave(s, rep)
    return TTBatch(cores, ranks.copy(), offs, tuple(dims_l))


def make_pair(kind: str, seed: int, cfg_id: int, b0: int, xranks: np.ndarray, dims, yranks: np.ndarray = None,
              rule: str = "uniform", device="cpu", density: float = 0.25):
    """(X, Y) batches of one validation kind (module docstring).  yranks defaults to xranks."""
    if yranks is None:
        yranks = xranks
    dims_l = tuple(int(d) for d in dims)
    if kind == "iid":
        return (gaussian_batch(seed, cfg_id, SIDE_X, b0, xranks, dims_l, rule, device),
                gaussian_batch(seed, cfg_id, SIDE_Y, b0, yranks, dims_l, rule, device))
    if kind == "self":
        X = gaussian_batch(seed, cfg_id, SIDE_X, b0, xranks, dims_l, rule, device)
        return X, TTBatch(X.cores.clone(), X.ranks.copy(), X.offsets.copy(), dims_l)
    if kind == "corr":
        X = gaussian_batch(seed, cfg_id, SIDE_X, b0, xranks, dims_l, rule, device)
        Nz = gaussian_batch(seed, cfg_id, SIDE_Y, b0, xranks, dims_l, rule, device)
        return X, TTBatch(X.cores + 0.1 * Nz.cores, X.ranks.copy(), X.offsets.copy(), dims_l)
    if kind == "int":
        out = []
        for side, rk in ((SIDE_X, xranks), (SIDE_Y, yranks)):
            offs, total = packed_offsets(rk, dims_l)
            g = torch.Generator(device="cpu")
            g.manual_seed(_seed(seed, cfg_id, side, b0, 7))
            v = torch.randint(-1, 2, (total,), generator=g).float()
            keep = torch.rand(total, generator=g) < density
            out.append(TTBatch((v * keep).to(device), rk.copy(), offs, dims_l))
        return tuple(out)
    if kind in ("rank1", "tagged"):
        out = []
        for side, rk in ((SIDE_X, xranks), (SIDE_Y, yranks)):
            offs, total = packed_offsets(rk, dims_l)
            host = torch.zeros(total, dtype=torch.float32)
            g = torch.Generator(device="cpu")
            g.manual_seed(_seed(seed, cfg_id, side, b0, 11))
            for j in range(rk.shape[0]):
                pos = int(offs[j])
                for n, I in enumerate(dims_l):
                    r0, r1 = int(rk[j, n]), int(rk[j, n + 1])
                    # element [0, i, 0] sits at 0 + r0*(i + I*0) = r0*i
                    if kind == "rank1":
                        vals = torch.randn(I, generator=g) / float(np.sqrt(I))
                    else:
                        vals = torch.zeros(I)
                        vals[0] = float(b0 + j) if (side == SIDE_X and n == 0) else 1.0
                    host[pos + r0 * torch.arange(I)] = vals
                    pos += r0 * I * r1
            out.append(TTBatch(host.to(device), rk.copy(), offs, dims_l))
        return tuple(out)
    raise ValueError(kind)


def config_batch(cfg: str, kind: str = "iid", b0: int = 0, B: Optional[int] = None, seed: int = DEFAULT_SEED,
                 device="cpu"):
    """(X, Y) for pairs b0..b0+B-1 of BASELINE.json config `cfg` (default: the whole batch)."""
    c = CONFIGS[cfg]
    B = c["B"] if B is None else B
    cid = CFG_ID[cfg]
    if cfg == "C5":
        N = c["N"]
        xr = random_ranks(seed, cid, SIDE_X, b0, B, N, c["rank_choices"])
        yr = random_ranks(seed, cid, SIDE_Y, b0, B, N, c["rank_choices"])
        if kind in ("self", "corr"):
            yr = xr
        return make_pair(kind, seed, cid, b0, xr, (c["I"],) * N, yr, rule="geo", device=device)
    if cfg in ("C3", "S1"):
        xr = uniform_ranks(B, c["N"], c["R"])
        yr = uniform_ranks(B, c["M"], c["P"])
        X = gaussian_batch(seed, cid, SIDE_X, b0, xr, (c["I"],) * c["N"], "uniform", device)
        Y = gaussian_batch(seed, cid, SIDE_Y, b0, yr, (c["I"],) * c["M"], "uniform", device)
        return X, Y
    xr = uniform_ranks(B, c["N"], c["R"])
    return make_pair(kind, seed, cid, b0, xr, (c["I"],) * c["N"], None, rule="uniform", device=device)


def dense_pairs(cfg: str, b0: int = 0, B: Optional[int] = None, seed: int = DEFAULT_SEED, device="cpu"):
    """(X, Y) dense float32 [B * I^N] batches of an "alg2" workload: N(0, 1) values, seeded per pair and side
    (Example 2: zero-mean, unit-variance Gaussian tensors)."""
    c = CONFIGS[cfg]
    B = c["B"] if B is None else B
    n_el = int(np.prod(alg2_shape(cfg)))
    out = []
    for side in (SIDE_X, SIDE_Y):
        host = torch.empty(B * n_el, dtype=torch.float32)
        for b in range(B):
            g = torch.Generator().manual_seed(_seed(seed, CFG_ID[cfg], side, b0 + b))
            host[b * n_el:(b + 1) * n_el] = torch.randn(n_el, generator=g, dtype=torch.float64).float()
        out.append(host.to(device))
    return tuple(out)
