"""GPU parity for the batched TT-SVD (ttc_tt_svd; Alg. 1) against oracle O6, and the whole dense-input TTCP
pipeline of Alg. 2 on the GPU (TT-SVD of X^rho and Y^rho, splice, reconstruction + permutation) against Eq. 8
(SURVEY.md §8f NEXT-3)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2109_00626_b200 as ttc
from oracle import ttsvd
from tests import ref_numpy as ref

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _dense_batch(Xs):
    return torch.from_numpy(np.concatenate([x.reshape(-1, order="F") for x in Xs]).astype(np.float32)).to(DEV)


def _trains(T):
    cores = T.cores.cpu().numpy().astype(np.float64)
    out = []
    rows = T.rank_rows()
    offs = T.offsets_np if T.offsets_np is not None else T._packed_offsets()
    for b in range(T.B):
        r = rows[b]
        pos, cs = int(offs[b]), []
        for n in range(T.N):
            a, i, c = int(r[n]), int(T.dims_np[n]), int(r[n + 1])
            cs.append(cores[pos:pos + a * i * c].reshape((a, i, c), order="F"))
            pos += a * i * c
        out.append(cs)
    return out


@pytest.mark.parametrize("dims", [(5,), (4, 6), (3, 4, 5), (20, 20, 20), (2, 3, 4, 3, 2), (6, 1, 5), (8, 8, 8, 8)])
def test_full_rank_reconstruction_and_ranks(dims):
    rng = np.random.default_rng(sum(dims))
    Xs = [rng.standard_normal(dims) for _ in range(3)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 0.0)
    for b, cs in enumerate(_trains(T)):
        want_cores = ttsvd.tt_svd(Xs[b], 0.0)
        assert [c.shape for c in cs] == [c.shape for c in want_cores]
        err = np.linalg.norm(ref.dense_from_tt(cs) - Xs[b]) / np.linalg.norm(Xs[b])
        assert err <= 2e-5, f"tensor {b}: relative reconstruction error {err:.3e}"
        for c in cs[:-1]:   # left-orthonormal cores
            U = c.reshape(-1, c.shape[2], order="F")
            np.testing.assert_allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-4)


def test_low_rank_ranks_and_cores_match_oracle():
    """A tensor built from a generic low-rank train (well separated singular values): the eps-truncation finds
    the construction's ranks, and the cores agree with O6 entry by entry (same sign convention, R24)."""
    rng = np.random.default_rng(3)
    dims, ranks = (6, 5, 7, 4), [1, 3, 4, 2, 1]
    Xs = [ref.dense_from_tt(ref.random_train(rng, dims, ranks)) for _ in range(4)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 1e-5)
    for b, cs in enumerate(_trains(T)):
        want = ttsvd.tt_svd(Xs[b], 1e-5)
        assert [c.shape[0] for c in cs] + [1] == ranks
        for c, w in zip(cs, want):
            assert np.max(np.abs(c - w)) <= 1e-3 * np.max(np.abs(w)), "core mismatch"


@pytest.mark.parametrize("eps", [0.05, 0.2, 0.5])
def test_error_guarantee(eps):
    rng = np.random.default_rng(int(100 * eps))
    dims = (6, 7, 5, 4)
    Xs = [rng.standard_normal(dims) for _ in range(4)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, eps)
    for b, cs in enumerate(_trains(T)):
        err = np.linalg.norm(ref.dense_from_tt(cs) - Xs[b])
        assert err <= eps * np.linalg.norm(Xs[b]) * (1 + 1e-4)
        # same ranks as the oracle (random spectra: decisions far from the threshold are robust; allow a
        # difference of one only where the discarded energy is within 1e-4 of delta^2)
        want = ttsvd.tt_svd(Xs[b], eps)
        assert all(abs(c.shape[2] - w.shape[2]) <= 1 for c, w in zip(cs[:-1], want[:-1]))


def test_permuted_decomposition():
    """perm (Alg. 2 step 1): the TT of X^rho equals the TT-SVD of numpy's transpose."""
    rng = np.random.default_rng(9)
    dims, perm = (4, 5, 6), [3, 1, 2]
    Xs = [rng.standard_normal(dims) for _ in range(2)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 0.0, perm=perm)
    for b, cs in enumerate(_trains(T)):
        want = np.transpose(Xs[b], [p - 1 for p in perm])
        np.testing.assert_allclose(ref.dense_from_tt(cs), want, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("shape_x,shape_y,n,m", [((20, 20, 20), (20, 20, 20), 1, 1), ((4, 5, 6), (6, 3), 3, 1),
                                                 ((3, 4), (5, 4, 2), 2, 2), ((4, 3, 5, 2), (2, 5, 3), 3, 2)])
def test_alg2_pipeline_on_gpu(shape_x, shape_y, n, m):
    """Alg. 2 end to end on the GPU == Eq. 8 (Example 2's x_1^1 on 20 x 20 x 20 included), eps = 0."""
    rng = np.random.default_rng(sum(shape_x) + m)
    B = 2
    Xs = [rng.standard_normal(shape_x) for _ in range(B)]
    Ys = [rng.standard_normal(shape_y) for _ in range(B)]
    px = [n] + [k for k in range(1, len(shape_x) + 1) if k != n]
    py = [m] + [k for k in range(1, len(shape_y) + 1) if k != m]
    TX = ttc.ttc_tt_svd(_dense_batch(Xs), shape_x, 0.0, perm=px)
    TY = ttc.ttc_tt_svd(_dense_batch(Ys), shape_y, 0.0, perm=py)
    plan = ttc.ttc_splice_plan_create(TX, TY, 1, 1)
    cores, ranks, offs = ttc.ttc_contract(plan, TX, TY)
    Z = ttc.TTDevice(cores, plan.dims, ranks=ranks, offsets=offs)
    dense = ttc.ttc_reconstruct(Z, plan.perm).cpu().numpy().astype(np.float64)
    n_el = int(np.prod([d for k, d in enumerate(shape_x) if k != n - 1])) * \
        int(np.prod([d for k, d in enumerate(shape_y) if k != m - 1]))
    for b in range(B):
        want = ref.tcp(Xs[b], Ys[b], [n], [m])
        got = dense[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        err = np.linalg.norm(got - want) / (np.linalg.norm(Xs[b]) * np.linalg.norm(Ys[b]))
        assert err <= 1e-5, f"pair {b}: {err:.3e}"
        np.testing.assert_allclose(got, ttsvd.ttcp_dense(Xs[b], Ys[b], n, m, 0.0), rtol=1e-3, atol=1e-3)


def test_ttsvd_errors():
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_tt_svd_capacity((2000, 2000))           # unfolding side 2000 > 1024
    assert e.value.status == ttc.TTC_ERR_UNSUPPORTED
    with pytest.raises(ttc.TTCError) as e:
        ttc.ttc_tt_svd_capacity((4, 5), perm=[1, 1])
    assert e.value.status == ttc.TTC_ERR_MODES


@pytest.mark.parametrize("dims,eps", [((3, 4, 5), 0.0), ((20, 20, 20), 0.0), ((6, 5, 7, 4), 0.2), ((2, 3, 4, 3, 2), 0.1)])
@pytest.mark.parametrize("other", ["TTC_TTSVD_FUSED", "TTC_TTSVD_BIG"])
def test_pipeline_matches_fused_kernel(dims, eps, other, monkeypatch):
    """The launch pipeline (one-warp Jacobi per eigenproblem, Gram sides <= 32), the fused one-CTA-per-tensor
    kernel (TTC_TTSVD_FUSED=1) and the one-sided Jacobi kernel of the large path (TTC_TTSVD_BIG=1) implement the
    same Alg. 1 with the same readings: equal ranks, cores equal to fp32 rounding (rotation orders differ)."""
    rng = np.random.default_rng(len(dims) + int(10 * eps))
    Xs = [rng.standard_normal(dims) for _ in range(5)]
    dense = _dense_batch(Xs)
    T_pipe = ttc.ttc_tt_svd(dense, dims, eps)
    monkeypatch.setenv(other, "1")        # the fused kernel, or the workspace one-sided Jacobi kernel
    T_fused = ttc.ttc_tt_svd(dense, dims, eps)
    monkeypatch.delenv(other)
    for b, (cp, cf) in enumerate(zip(_trains(T_pipe), _trains(T_fused))):
        assert [c.shape for c in cp] == [c.shape for c in cf], f"tensor {b}: ranks differ"
        scale = np.linalg.norm(Xs[b])
        for p, f in zip(cp, cf):
            assert np.max(np.abs(p - f)) <= 1e-4 * max(1.0, scale), f"tensor {b}: cores differ"
        err = np.linalg.norm(ref.dense_from_tt(cp) - Xs[b]) / scale
        assert err <= max(eps, 2e-5) * (1 + 1e-4)


@pytest.mark.parametrize("spectrum,want", [((1.0, 1e-5, 1e-9), 2), ((1.0, 3e-7, 3e-8), 2), ((1.0, 0.5, 2e-7), 3)])
def test_sigma_floor_on_constructed_spectra(spectrum, want):
    """R25 on the GPU: first-unfolding singular values straddling the 1e-7 sigma_max floor (tests/
    test_oracle_ttsvd.py pins the oracle on the same tensors).  A Gram eigenproblem solved in fp32, or a floor
    other than the oracle's, would drop 1e-5 / 3e-7 / 2e-7 or keep 1e-9 / 3e-8 and fail the rank check."""
    rng = np.random.default_rng(int(1e3 * spectrum[1]) + len(spectrum))
    X = ref.tensor_with_unfolding_spectrum(rng, (20, 20, 20), spectrum)
    X32 = X.astype(np.float32).astype(np.float64)
    T = ttc.ttc_tt_svd(_dense_batch([X32, X32]), (20, 20, 20), 0.0)
    want_cores = ttsvd.tt_svd(X32, 0.0)
    assert want_cores[0].shape[2] == want
    for cs in _trains(T):
        assert [c.shape for c in cs] == [c.shape for c in want_cores]
        err = np.linalg.norm(ref.dense_from_tt(cs) - X32) / np.linalg.norm(X32)
        assert err <= 2e-5


EXAMPLE2 = [(20, 20, 20, 5), (20, 20, 20, 5, 4)]   # PAPER.md:406-412, cases (ii) and (iii)


@pytest.mark.parametrize("dims", EXAMPLE2)
def test_example2_sizes_match_oracle(dims):
    """Example 2's order-4 and order-5 Gaussian tensors (40,000 / 160,000 elements; unfoldings up to 400 x 100 and
    400 x 400) through the workspace kernel: the ranks of O6 (full: [1, 20, 100, 5, 1] / [1, 20, 400, 20, 4, 1]),
    cores entry by entry (R24 signs), reconstruction and left-orthonormality."""
    rng = np.random.default_rng(len(dims))
    Xs = [rng.standard_normal(dims).astype(np.float32).astype(np.float64) for _ in range(2)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 0.0)
    for b, cs in enumerate(_trains(T)):
        want = ttsvd.tt_svd(Xs[b], 0.0)
        assert [c.shape for c in cs] == [w.shape for w in want], f"tensor {b}: ranks differ"
        for n, (c, w) in enumerate(zip(cs, want)):
            d = np.max(np.abs(c - w))
            assert d <= 1e-5 * max(1.0, np.max(np.abs(w))), f"tensor {b} core {n + 1}: max |diff| {d:.3e}"
        err = np.linalg.norm(ref.dense_from_tt(cs) - Xs[b]) / np.linalg.norm(Xs[b])
        assert err <= 2e-6, f"tensor {b}: relative reconstruction error {err:.3e}"
        for c in cs[:-1]:
            U = c.reshape(-1, c.shape[2], order="F")
            np.testing.assert_allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-5)


@pytest.mark.parametrize("dims,ranks", [((20, 20, 20, 5), [1, 7, 30, 5, 1]), ((20, 20, 20, 5, 4), [1, 9, 60, 11, 3, 1]),
                                        ((5, 20, 20, 20), [1, 5, 70, 20, 1])])
def test_example2_sizes_low_rank(dims, ranks):
    """Trains of known ranks at Example 2's sizes: eps = 1e-5 recovers the construction's ranks and O6's cores."""
    rng = np.random.default_rng(sum(ranks))
    Xs = [ref.dense_from_tt(ref.random_train(rng, dims, ranks)) for _ in range(3)]
    Xs = [x.astype(np.float32).astype(np.float64) for x in Xs]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 1e-5)
    for b, cs in enumerate(_trains(T)):
        want = ttsvd.tt_svd(Xs[b], 1e-5)
        assert [c.shape[0] for c in cs] + [1] == ranks
        assert [c.shape for c in cs] == [w.shape for w in want]
        for c, w in zip(cs, want):
            assert np.max(np.abs(c - w)) <= 1e-4 * np.max(np.abs(w)), "core mismatch"


@pytest.mark.parametrize("eps", [0.1, 0.3])
def test_example2_error_guarantee(eps):
    """||X - TT(X)|| <= eps ||X|| (Alg. 1's guarantee) on case (iii), ranks within one of O6's."""
    dims = EXAMPLE2[1]
    rng = np.random.default_rng(int(100 * eps))
    Xs = [rng.standard_normal(dims).astype(np.float32).astype(np.float64) for _ in range(2)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, eps)
    for b, cs in enumerate(_trains(T)):
        err = np.linalg.norm(ref.dense_from_tt(cs) - Xs[b])
        assert err <= eps * np.linalg.norm(Xs[b]) * (1 + 1e-4)
        want = ttsvd.tt_svd(Xs[b], eps)
        assert all(abs(c.shape[2] - w.shape[2]) <= 1 for c, w in zip(cs[:-1], want[:-1]))


@pytest.mark.parametrize("case", [0, 1])
def test_example2_alg2_on_gpu(case):
    """Example 2 cases (ii) and (iii) end to end on the GPU: X x_1^1 Y of two 20 x 20 x 20 x 5 (x 4) Gaussian
    tensors through TT-SVD (workspace kernel), splice (ranks up to 400 in case (iii)), reconstruction (workspace
    GEMM chain; 4,000,000 / 64,000,000 entries per pair) == Eq. 8 (eps = 0: exact up to rounding)."""
    dims = EXAMPLE2[case]
    rng = np.random.default_rng(11 + case)
    B = 2 - case
    Xs = [rng.standard_normal(dims).astype(np.float32).astype(np.float64) for _ in range(B)]
    Ys = [rng.standard_normal(dims).astype(np.float32).astype(np.float64) for _ in range(B)]
    TX = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 0.0)
    TY = ttc.ttc_tt_svd(_dense_batch(Ys), dims, 0.0)
    plan = ttc.ttc_splice_plan_create(TX, TY, 1, 1)
    cores, ranks, offs = ttc.ttc_contract(plan, TX, TY)
    Z = ttc.TTDevice(cores, plan.dims, ranks=ranks, offsets=offs)
    dense = ttc.ttc_reconstruct(Z, plan.perm).cpu().numpy().astype(np.float64)
    n_el = int(np.prod(dims[1:])) ** 2
    for b in range(B):
        want = ref.tcp(Xs[b], Ys[b], [1], [1])
        got = dense[b * n_el:(b + 1) * n_el].reshape(want.shape, order="F")
        err = np.linalg.norm(got - want) / (np.linalg.norm(Xs[b]) * np.linalg.norm(Ys[b]))
        assert err <= 1e-5, f"pair {b}: {err:.3e}"


def test_big_path_in_chunks_matches_fused_kernel(monkeypatch):
    """More tensors than co-resident CTAs (200 > 148): the workspace kernel runs in several cooperative launches
    of whole groups; ranks and cores equal the fused shared-memory kernel's to fp32 rounding."""
    dims, B = (12, 10, 9), 200
    rng = np.random.default_rng(77)
    Xs = [rng.standard_normal(dims) for _ in range(B)]
    dense = _dense_batch(Xs)
    monkeypatch.setenv("TTC_TTSVD_FUSED", "1")
    T_f = ttc.ttc_tt_svd(dense, dims, 0.05)
    monkeypatch.delenv("TTC_TTSVD_FUSED")
    monkeypatch.setenv("TTC_TTSVD_BIG", "1")
    T_b = ttc.ttc_tt_svd(dense, dims, 0.05)
    monkeypatch.delenv("TTC_TTSVD_BIG")
    assert np.array_equal(T_f.rank_rows(), T_b.rank_rows())
    for b, (cf, cb) in enumerate(zip(_trains(T_f), _trains(T_b))):
        scale = np.linalg.norm(Xs[b])
        for f, g in zip(cf, cb):
            assert np.max(np.abs(f - g)) <= 1e-4 * max(1.0, scale), f"tensor {b}: cores differ"


def test_example2_permuted_big_operand():
    """Alg. 2 step 1's permutation folded into the workspace kernel's read: the TT of X^rho (X of shape
    5 x 20 x 20 x 20, rho = (2, 3, 4, 1): 20 x 20 x 20 x 5) equals O6's TT-SVD of numpy's transpose."""
    rng = np.random.default_rng(21)
    dims, perm = (5, 20, 20, 20), [2, 3, 4, 1]
    Xs = [rng.standard_normal(dims).astype(np.float32).astype(np.float64) for _ in range(2)]
    T = ttc.ttc_tt_svd(_dense_batch(Xs), dims, 0.0, perm=perm)
    for b, cs in enumerate(_trains(T)):
        Xr = np.transpose(Xs[b], [p - 1 for p in perm])
        want = ttsvd.tt_svd(Xr, 0.0)
        assert [c.shape for c in cs] == [w.shape for w in want]
        for c, w in zip(cs, want):
            assert np.max(np.abs(c - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))


@pytest.mark.parametrize("dims", [(20000,), (1, 20000), (20000, 1), (3, 1, 7000), (130, 130)])
def test_big_path_degenerate_shapes(dims):
    """The workspace kernel on its degenerate cases: order 1 (the train is the tensor), unit modes (one-column
    unfoldings: no rotation), a zero tensor (every rank 1, the train's product zero), against O6."""
    rng = np.random.default_rng(len(dims))
    X = rng.standard_normal(dims).astype(np.float32).astype(np.float64)
    Z0 = np.zeros(dims)
    T = ttc.ttc_tt_svd(_dense_batch([X, Z0]), dims, 0.0)
    got = _trains(T)
    want = ttsvd.tt_svd(X, 0.0)
    assert [c.shape for c in got[0]] == [w.shape for w in want]
    for c, w in zip(got[0], want):
        assert np.max(np.abs(c - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))
    # zero tensor: every rank 1 (R23 with s_0 = 0), a train whose product is exactly zero
    assert all(c.shape[0] == 1 and c.shape[2] == 1 for c in got[1])
    assert np.all(ref.dense_from_tt(got[1]) == 0)


@pytest.mark.parametrize("dims", [(900, 40), (40, 900), (1000, 300)])
def test_big_path_narrow_blocks(dims):
    """Long columns (L > 768) put the block one-sided Jacobi on 8- or 4-column blocks; cores against O6."""
    rng = np.random.default_rng(sum(dims))
    X = rng.standard_normal(dims).astype(np.float32).astype(np.float64)
    T = ttc.ttc_tt_svd(_dense_batch([X]), dims, 0.0)
    got, want = _trains(T)[0], ttsvd.tt_svd(X, 0.0)
    assert [c.shape for c in got] == [w.shape for w in want]
    for c, w in zip(got, want):
        assert np.max(np.abs(c - w)) <= 1e-5 * max(1.0, np.max(np.abs(w)))


def test_big_paths_capture_in_a_cuda_graph():
    """The workspace TT-SVD (cooperative launches + a stream-ordered reset of its barrier counters) and the
    workspace reconstruction captured in a CUDA graph on a side stream: replays reproduce the direct calls bitwise."""
    dims, B = (20, 20, 20, 5), 3
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(B * 40000).astype(np.float32)).to(DEV)
    ref = ttc.ttc_tt_svd(x, dims, 0.0)
    cap = ttc.ttc_tt_svd_capacity(dims)
    cores = torch.zeros(B * cap, device=DEV)
    ranks = torch.zeros((B, len(dims) + 1), dtype=torch.int32, device=DEV)
    ws = torch.empty(ttc.ttc_tt_svd_workspace(B, dims), dtype=torch.uint8, device=DEV)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ttc.ttc_tt_svd_into(x, dims, 0.0, cores, ranks, workspace=ws)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(cores, ref.cores) and np.array_equal(ranks.cpu().numpy(), ref.rank_rows())
    # the spliced result of two of them, reconstructed through the workspace path inside a graph
    plan = ttc.ttc_splice_plan_create(ref, ref, 1, 1)
    zc, zr, zo = ttc.ttc_contract(plan, ref, ref)
    Z = ttc.TTDevice(zc, plan.dims, ranks=zr, offsets=zo)
    want = ttc.ttc_reconstruct(Z, plan.perm)
    nb = ttc.ttc_reconstruct_workspace(Z, plan.perm)
    assert nb > 0
    rws = torch.empty(nb, dtype=torch.uint8, device=DEV)
    out = torch.empty_like(want)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        ttc.ttc_reconstruct(Z, plan.perm, out=out, workspace=rws, stream=s)
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)
