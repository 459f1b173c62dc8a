"""GPU parity for ttc_reconstruct (dense tensors of trains, Alg. 2 steps 5-6) against the
oracle's Eq. 9 reconstruction (O1a, pinned in test_oracle_dense.py) and numpy's transpose for the permutation;
end to end, contraction / splice on the GPU followed by reconstruction equals the dense Eq. 8 definition."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
import ttgen
from tests import ref_numpy as ref

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _recon(T, perm=None):
    TD = ttc.TTDevice.from_batch(T, DEV)
    out = ttc.ttc_reconstruct(TD, perm)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _want(cores, perm):
    d = oracle.tt_reconstruct(cores)
    return d if perm is None else np.transpose(d, [p - 1 for p in perm])


def _check(T, got, perm=None, tol=2e-6):
    n_el = int(np.prod(T.dims))
    for b in range(T.B):
        cores = T.train(b)
        want = _want(cores, perm)
        seg = got[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        # fp32 sums of R_k products: bound by the reconstruction of |cores| (the exact sum of |terms|)
        bound = oracle.tt_reconstruct([np.abs(c) for c in cores])
        if perm is not None:
            bound = np.transpose(bound, [p - 1 for p in perm])
        assert np.max(np.abs(seg - want) / np.maximum(bound, 1e-30)) <= tol, f"train {b}"


@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("case", range(7))
def test_random_trains(case, big, monkeypatch):
    """Orders 1..6, odd mode sizes, heterogeneous per-train ranks, with and without a permutation; through the
    one-launch shared-memory kernel and (TTC_RECON_BIG=1) the workspace GEMM chain of reconstruct_big.cu."""
    if big:
        monkeypatch.setenv("TTC_RECON_BIG", "1")
    rng = np.random.default_rng(40 + case)
    dims = [(7,), (3, 5), (4, 1, 6), (2, 3, 4, 5), (5, 4, 3, 2, 3), (3, 2, 3, 2, 3, 2), (20, 20, 20, 20)][case]
    N = len(dims)
    B = 5
    r = np.stack([[1] + list(rng.integers(1, 9, N - 1)) + [1] for _ in range(B)]).astype(np.int32)
    T = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, r, dims, "geo")
    _check(T, _recon(T))
    perm = list(rng.permutation(N) + 1)
    _check(T, _recon(T, perm), perm)


def test_r1_sampled_and_uniform():
    """The R1 workload bench.py --config R1 times (Example 2's TTCP output, order 4, I = 20, ranks 20)."""
    T, _ = ttgen.config_batch("R1", B=64)
    got = _recon(T)
    n_el = 20 ** 4
    for b in (0, 63):
        want = oracle.tt_reconstruct(T.train(b))
        seg = got[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        bound = oracle.tt_reconstruct([np.abs(c) for c in T.train(b)])
        assert np.max(np.abs(seg - want) / bound) <= 2e-6


def test_contract_then_reconstruct_is_eq8():
    """Alg. 2 steps 4-6 end to end on the GPU: ladder contraction (C3's mode pairs on smaller operands), then the
    dense reconstruction in Eq. 8 order (perm = the plan's out_perm) == tensordot of the dense operands."""
    rng = np.random.default_rng(5)
    dims, xm, ym = (3,) * 6, [2, 4, 6], [1, 3, 5]
    B = 3
    r = np.tile(np.array([1, 3, 3, 3, 3, 3, 1], np.int32), (B, 1))
    X = ttgen.gaussian_batch(11, 0, 0, 0, r, dims, "geo")
    Y = ttgen.gaussian_batch(12, 0, 1, 0, r, dims, "geo")
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    plan = ttc.ttc_contract_plan_create(XD, YD, xm, ym)
    cores, ranks, offs = ttc.ttc_contract(plan, XD, YD)
    Z = ttc.TTDevice(cores, plan.dims, ranks=ranks, offsets=offs)
    dense = ttc.ttc_reconstruct(Z, plan.perm).cpu().numpy().astype(np.float64)
    n_el = 3 ** 6
    for b in range(B):
        want = ref.tcp(ref.dense_from_tt(X.train(b)), ref.dense_from_tt(Y.train(b)), xm, ym)
        got = dense[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        err = np.linalg.norm(got - want) / oracle.normaliser(X.train(b), Y.train(b))
        assert err <= 1e-5


def test_splice_then_reconstruct_is_eq8():
    """The paper's own pipeline on TT operands: splice x_1^1 (Alg. 2 steps 4-5), reconstruct + permute (steps
    5-6) == Eq. 8 (Example 2's shape: two order-3 tensors, 20 x 20 x 20, TT ranks 6)."""
    dims = (20, 20, 20)
    B = 2
    r = np.tile(np.array([1, 6, 6, 1], np.int32), (B, 1))
    X = ttgen.gaussian_batch(13, 0, 0, 0, r, dims, "geo")
    Y = ttgen.gaussian_batch(14, 0, 1, 0, r, dims, "geo")
    XD, YD = ttc.TTDevice.from_batch(X, DEV), ttc.TTDevice.from_batch(Y, DEV)
    plan = ttc.ttc_splice_plan_create(XD, YD, 1, 1)
    cores, ranks, offs = ttc.ttc_contract(plan, XD, YD)
    Z = ttc.TTDevice(cores, plan.dims, ranks=ranks, offsets=offs)
    dense = ttc.ttc_reconstruct(Z, plan.perm).cpu().numpy().astype(np.float64)
    n_el = 20 ** 4
    for b in range(B):
        want = ref.tcp(ref.dense_from_tt(X.train(b)), ref.dense_from_tt(Y.train(b)), [1], [1])
        got = dense[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        err = np.linalg.norm(got - want) / oracle.normaliser(X.train(b), Y.train(b))
        assert err <= 1e-5


@pytest.mark.parametrize("dims,rk", [((20, 20, 5, 20, 20, 5), (1, 5, 100, 20, 100, 5, 1)),
                                     ((5, 20, 20, 20, 5), (1, 5, 100, 100, 5, 1)),
                                     ((7, 2000, 9), (1, 7, 9, 1))])
def test_beyond_shared_memory(dims, rk):
    """Trains whose partial products fit no shared-memory split (Example 2 case (ii)'s TTCP output, 4,000,000
    entries with ranks 100; an order-5 one with two rank-100 bonds; a long middle mode): the workspace path,
    heterogeneous per-train ranks, identity and random permutations."""
    rng = np.random.default_rng(sum(dims))
    B = 2
    r = np.tile(np.array(rk, np.int32), (B, 1))
    r[1, 1:-1] = np.maximum(1, r[1, 1:-1] - 1)
    T = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, r, dims, "geo")
    TD = ttc.TTDevice.from_batch(T, DEV)
    assert ttc.ttc_reconstruct_workspace(TD) > 0
    with pytest.raises(ttc.TTCError) as e:   # the workspace-free entry point names the size it needs
        ttc._check(ttc._lib.ttc_reconstruct(ctypes.byref(TD.c), None, ttc._ptr(torch.empty(1, device=DEV)), None, None))
    assert e.value.status == ttc.TTC_ERR_ARG and "workspace" in str(e.value)
    _check(T, _recon(T))
    perm = list(rng.permutation(len(dims)) + 1)
    _check(T, _recon(T, perm), perm)


def test_reconstruct_errors():
    T, _ = ttgen.config_batch("R1", B=2)
    TD = ttc.TTDevice.from_batch(T, DEV)
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_reconstruct(TD, [1, 1, 2, 3])
    assert e.value.status == ttc.TTC_ERR_MODES


@pytest.mark.parametrize("N,perm_first", [(4, 2), (4, 1), (5, 3), (6, 3), (3, 2)])
def test_output_stride_one_mode_placement(N, perm_first):
    """The output's stride-1 mode is the left block's first mode (little-endian rows), its last mode k (rows
    enumerated big-endian, 16-byte stores) or elsewhere (scalar stores): all three give Eq. 9 + permutation."""
    rng = np.random.default_rng(100 + 10 * N + perm_first)
    dims = tuple(int(x) for x in rng.integers(3, 9, size=N))
    r = np.stack([[1] + [int(x) for x in rng.choice([4, 8, 5], size=N - 1)] + [1] for _ in range(3)]).astype(np.int32)
    T = ttgen.gaussian_batch(int(rng.integers(1 << 30)), 0, 0, 0, r, dims, "geo")
    rest = [k for k in range(1, N + 1) if k != perm_first]
    perm = [perm_first] + list(rng.permutation(rest))
    _check(T, _recon(T, perm), perm)


@pytest.mark.parametrize("big", [False, True])
def test_out_offsets(big, monkeypatch):
    """Caller-given output offsets (out_offsets_dev: trains in reverse order with gaps): every train's dense tensor
    lands at its offset, bitwise equal to the packed call, and nothing is written in the gaps."""
    if big:
        monkeypatch.setenv("TTC_RECON_BIG", "1")
    rng = np.random.default_rng(8)
    dims, B = (5, 4, 3, 6), 4
    r = np.stack([[1] + list(rng.integers(1, 6, 3)) + [1] for _ in range(B)]).astype(np.int32)
    T = ttgen.gaussian_batch(3, 0, 0, 0, r, dims, "geo")
    TD = ttc.TTDevice.from_batch(T, DEV)
    packed = ttc.ttc_reconstruct(TD, [2, 1, 4, 3]).cpu().numpy()
    n_el = int(np.prod(dims))
    gap = 37
    offs = np.array([(B - 1 - b) * (n_el + gap) + gap for b in range(B)], np.int64)
    out = torch.full((B * (n_el + gap) + gap,), float("nan"), dtype=torch.float32, device=DEV)
    ttc.ttc_reconstruct(TD, [2, 1, 4, 3], out=out, out_offsets=torch.from_numpy(offs).to(DEV))
    got = out.cpu().numpy()
    written = np.zeros(got.size, bool)
    for b in range(B):
        seg = got[offs[b]: offs[b] + n_el]
        assert np.array_equal(seg.view(np.uint32), packed[b * n_el:(b + 1) * n_el].view(np.uint32)), f"train {b}"
        written[offs[b]: offs[b] + n_el] = True
    assert np.all(np.isnan(got[~written])), "wrote into a gap"
