"""paper_2109_00626_b200 -- batched Tensor-Train contraction (TTCP, arXiv 2109.00626) on B200.

Thin Python binding over the C ABI of libttc.so (include/ttc.h): the functions here carry the C names and
only marshal arguments (torch tensors -> device pointers, numpy -> host pointers, torch stream -> handle).
Every step of the computation runs in the CUDA kernels of libttc.so; there is no CPU fallback, and
importing this package without the built library raises.

    X = TTDevice(cores, dims, ranks=None or int32[B, N+1], offsets=None or int64[B])
    out = ttc_inner(X, Y)                                  # <X_b, Y_b>, float32 [B] on the device
    plan = ttc_contract_plan_create(X, Y, [2, 4, 6], [1, 3, 5])
    order, dims, src, perm, total, max_rank = ttc_contract_plan_query(plan)
    cores, ranks, offsets = ttc_contract(plan, X, Y)       # output TTs (ladder order; perm -> Eq. 8 order)
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTC_LIB_PATH") or os.path.join(_HERE, "libttc.so")   # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "there is no fallback implementation")

_lib = ctypes.CDLL(LIB_PATH)

TTC_OK, TTC_ERR_NULL, TTC_ERR_SHAPE, TTC_ERR_RANK, TTC_ERR_MODES = 0, 1, 2, 3, 4
TTC_ERR_ALIGN, TTC_ERR_OVERFLOW, TTC_ERR_UNSUPPORTED, TTC_ERR_CUDA, TTC_ERR_ARG = 5, 6, 7, 8, 9
TTC_MAX_ORDER, TTC_MAX_CONTRACT_ORDER, TTC_MAX_RANK, TTC_MAX_SPLICE_RANK = 256, 64, 128, 1024

EXPORTED = ("ttc_inner", "ttc_inner_ordered", "ttc_contract_plan_create", "ttc_splice_plan_create", "ttc_contract_plan_query",
            "ttc_contract_plan_layout", "ttc_reconstruct", "ttc_reconstruct_workspace", "ttc_reconstruct_ws",
            "ttc_tt_svd", "ttc_tt_svd_capacity", "ttc_tt_svd_workspace", "ttc_contract", "ttc_contract_plan_destroy", "ttc_pair_cost", "ttc_partition", "ttc_status_string",
            "ttc_last_error", "ttc_version")


class ttc_tt_batch(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("order", ctypes.c_int32), ("dims", ctypes.c_void_p),
                ("ranks_host", ctypes.c_void_p), ("ranks_dev", ctypes.c_void_p), ("uniform_rank", ctypes.c_int32),
                ("offsets_host", ctypes.c_void_p), ("offsets_dev", ctypes.c_void_p), ("cores", ctypes.c_void_p),
                ("n_elems", ctypes.c_int64)]


_P = ctypes.POINTER
_lib.ttc_inner.argtypes = [_P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_inner_ordered.argtypes = [_P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_contract_plan_create.argtypes = [_P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_void_p, _P(ctypes.c_void_p)]
_lib.ttc_splice_plan_create.argtypes = [_P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_void_p]
_lib.ttc_contract_plan_query.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 6
_lib.ttc_contract_plan_layout.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_contract.argtypes = [ctypes.c_void_p, _P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p]
_lib.ttc_contract_plan_destroy.argtypes = [ctypes.c_void_p]
_lib.ttc_contract_plan_destroy.restype = None
_lib.ttc_pair_cost.argtypes = [_P(ttc_tt_batch), _P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_partition.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
_lib.ttc_status_string.restype = ctypes.c_char_p
_lib.ttc_status_string.argtypes = [ctypes.c_int]
_lib.ttc_last_error.restype = ctypes.c_char_p
_lib.ttc_version.restype = ctypes.c_int32
_lib.ttc_reconstruct.argtypes = [_P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_reconstruct_workspace.argtypes = [_P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_reconstruct_ws.argtypes = [_P(ttc_tt_batch), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
_lib.ttc_tt_svd_capacity.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.ttc_tt_svd_workspace.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]
_lib.ttc_tt_svd.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_void_p]
for _f in ("ttc_inner", "ttc_inner_ordered", "ttc_contract_plan_create", "ttc_splice_plan_create", "ttc_contract_plan_query",
           "ttc_contract_plan_layout", "ttc_reconstruct", "ttc_reconstruct_workspace", "ttc_reconstruct_ws",
           "ttc_tt_svd", "ttc_tt_svd_capacity", "ttc_tt_svd_workspace", "ttc_contract", "ttc_pair_cost", "ttc_partition"):
    getattr(_lib, _f).restype = ctypes.c_int


class TTCError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{ttc_status_string(status)}: {detail}")


def ttc_status_string(status: int) -> str:
    return _lib.ttc_status_string(int(status)).decode()


def ttc_last_error() -> str:
    return _lib.ttc_last_error().decode()


def ttc_version() -> int:
    return int(_lib.ttc_version())


def _check(rc: int):
    if rc != TTC_OK:
        raise TTCError(rc, ttc_last_error())


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.data_ptr()
    return a.ctypes.data


class TTDevice:
    """A batch of B trains as the C ABI sees it (ttc_tt_batch), with the host arrays it needs kept alive.

    cores: float32 torch tensor (flat, on the GPU for compute calls); dims: (I_1..I_N);
    ranks: int32 [B, N+1] (row b = R_0..R_N) or None with uniform_rank; offsets: int64 [B] or None (packed).
    Ranks that are the same for every train are passed as uniform (the C ABI's fast path)."""

    def __init__(self, cores: torch.Tensor, dims: Sequence[int], ranks=None, offsets=None, uniform_rank: int = None,
                 batch: int = None):
        if cores.dtype != torch.float32:
            raise TypeError("cores must be float32")
        if not cores.is_contiguous():
            raise ValueError("cores must be contiguous")
        self.cores = cores
        self.dims_np = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
        N = int(self.dims_np.shape[0])
        self.ranks_np = None
        self.uniform_rank = 1
        if ranks is not None:
            r = np.ascontiguousarray(np.asarray(ranks, dtype=np.int32))
            if r.ndim != 2 or r.shape[1] != N + 1:
                raise ValueError(f"ranks must be [B, N+1] = [*, {N + 1}], got {r.shape}")
            B = r.shape[0]
            inner = r[:, 1:N]
            uni = B > 0 and N > 1 and bool(np.all(inner == inner.flat[0])) and bool(np.all(r[:, 0] == 1)) \
                and bool(np.all(r[:, N] == 1))
            if B > 0 and N == 1 and bool(np.all(r == 1)):
                uni, self.uniform_rank = True, 1
            elif uni:
                self.uniform_rank = int(inner.flat[0])
            if not uni:
                self.ranks_np = r
        else:
            if batch is None:
                raise ValueError("batch is required with uniform ranks")
            B = int(batch)
            self.uniform_rank = int(uniform_rank if uniform_rank is not None else 1)
        self.B = int(B)
        self.N = N
        self.offsets_np = None
        if offsets is not None:
            o = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
            if o.shape != (B,):
                raise ValueError(f"offsets must be [B] = [{B}], got {o.shape}")
            packed = self._packed_offsets()
            if packed is None or not np.array_equal(o, packed):
                self.offsets_np = o
        dev = cores.device
        self.ranks_dev = torch.from_numpy(self.ranks_np).to(dev) if self.ranks_np is not None else None
        self.offsets_dev = torch.from_numpy(self.offsets_np).to(dev) if self.offsets_np is not None else None
        if self.ranks_np is not None and self.offsets_np is None and self.B > 1:
            self.offsets_np = self._packed_offsets()
            self.offsets_dev = torch.from_numpy(self.offsets_np).to(dev)
        self.c = ttc_tt_batch(self.B, self.N, _ptr(self.dims_np), _ptr(self.ranks_np), _ptr(self.ranks_dev),
                              self.uniform_rank, _ptr(self.offsets_np), _ptr(self.offsets_dev),
                              cores.data_ptr() if cores.numel() else None, int(cores.numel()))

    def _packed_offsets(self):
        if self.ranks_np is None:
            return None if self.B == 0 else np.arange(self.B, dtype=np.int64) * self._uniform_train_elems()
        r = self.ranks_np.astype(np.int64)
        sizes = (r[:, :-1] * self.dims_np[None, :].astype(np.int64) * r[:, 1:]).sum(axis=1)
        offs = np.zeros(self.B, np.int64)
        if self.B > 1:
            offs[1:] = np.cumsum(sizes)[:-1]
        return offs

    def _uniform_train_elems(self):
        r = [1] + [self.uniform_rank] * (self.N - 1) + [1]
        return int(sum(r[n] * int(self.dims_np[n]) * r[n + 1] for n in range(self.N)))

    @classmethod
    def from_batch(cls, b, device=None):
        """From any object with .cores, .dims, .ranks, .offsets (e.g. ttgen.TTBatch)."""
        cores = b.cores if device is None else b.cores.to(device)
        return cls(cores.contiguous(), b.dims, ranks=b.ranks, offsets=b.offsets)

    def rank_rows(self) -> np.ndarray:
        if self.ranks_np is not None:
            return self.ranks_np
        r = np.full((self.B, self.N + 1), self.uniform_rank, np.int32)
        r[:, 0] = 1
        r[:, self.N] = 1
        return r


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class CostOrder:
    """A processing order for ttc_inner_ordered: pairs by descending ttc_pair_cost (MACs), host + device copy."""

    def __init__(self, x: "TTDevice", y: "TTDevice"):
        mac, _ = ttc_pair_cost(x, y)
        self.host = np.ascontiguousarray(np.argsort(-mac, kind="stable").astype(np.int32))
        self.dev = torch.from_numpy(self.host).to(x.cores.device)


def ttc_cost_order(x: "TTDevice", y: "TTDevice") -> CostOrder:
    return CostOrder(x, y)


def ttc_inner(x: TTDevice, y: TTDevice, out: torch.Tensor = None, stream=None, order: CostOrder = None) -> torch.Tensor:
    """out[b] = <X_b, Y_b> (ttc.h: ttc_inner; with `order`, ttc_inner_ordered: same values, pairs started in
    that order).  Asynchronous on `stream` (default: torch's current stream)."""
    if out is None:
        out = torch.empty(x.B, dtype=torch.float32, device=x.cores.device)
        _keep_alive(stream, out.device, out)
    if order is None:
        _check(_lib.ttc_inner(ctypes.byref(x.c), ctypes.byref(y.c), _ptr(out) if out.numel() else None,
                              _stream_handle(stream)))
    else:
        _check(_lib.ttc_inner_ordered(ctypes.byref(x.c), ctypes.byref(y.c), _ptr(order.host), _ptr(order.dev),
                                      _ptr(out) if out.numel() else None, _stream_handle(stream)))
    return out


class ContractPlan:
    """Owns a ttc_contract_plan* (host-only)."""

    def __init__(self, handle: int, x: TTDevice, y: TTDevice):
        self.handle = handle
        order = ctypes.c_int32(0)
        total = ctypes.c_int64(0)
        mr = ctypes.c_int32(0)
        L = x.N + y.N
        dims, src, perm = (np.zeros(max(L, 1), np.int32) for _ in range(3))
        _check(_lib.ttc_contract_plan_query(handle, ctypes.byref(order), _ptr(dims), _ptr(src), _ptr(perm),
                                            ctypes.byref(total), ctypes.byref(mr)))
        self.L = order.value
        self.dims, self.src, self.perm = dims[:self.L].copy(), src[:self.L].copy(), perm[:self.L].copy()
        self.total = total.value
        self.max_rank = mr.value
        self.B = x.B
        self.ranks = np.zeros((x.B, self.L + 1), np.int32)
        self.offsets = np.zeros(x.B, np.int64)
        _check(_lib.ttc_contract_plan_layout(handle, _ptr(self.ranks) if x.B else None,
                                             _ptr(self.offsets) if x.B else None))
        self._offsets_dev = None
        self._uniform_out = None

    # bound at class creation: module globals may already be None when a plan is collected at interpreter exit
    _destroy = _lib.ttc_contract_plan_destroy

    def __del__(self):
        if getattr(self, "handle", None):
            type(self)._destroy(self.handle)
            self.handle = None


def ttc_contract_plan_create(x: TTDevice, y: TTDevice, x_modes: Sequence[int], y_modes: Sequence[int]) -> ContractPlan:
    xm = np.ascontiguousarray(np.asarray(list(x_modes), dtype=np.int32))
    ym = np.ascontiguousarray(np.asarray(list(y_modes), dtype=np.int32))
    h = ctypes.c_void_p(0)
    _check(_lib.ttc_contract_plan_create(ctypes.byref(x.c), ctypes.byref(y.c), len(xm), _ptr(xm) if len(xm) else None,
                                         _ptr(ym) if len(ym) else None, ctypes.byref(h)))
    return ContractPlan(h.value, x, y)


def ttc_splice_plan_create(x: TTDevice, y: TTDevice, x_mode: int, y_mode: int) -> ContractPlan:
    """The paper's TTCP splice of one pair of end modes (ttc.h: ttc_splice_plan_create); use the plan like a
    contraction plan (query / layout / ttc_contract)."""
    h = ctypes.c_void_p(0)
    _check(_lib.ttc_splice_plan_create(ctypes.byref(x.c), ctypes.byref(y.c), int(x_mode), int(y_mode), ctypes.byref(h)))
    return ContractPlan(h.value, x, y)


def ttc_contract_plan_query(plan: ContractPlan):
    return plan.L, plan.dims, plan.src, plan.perm, plan.total, plan.max_rank


def ttc_contract_plan_layout(plan: ContractPlan):
    return plan.ranks, plan.offsets


def ttc_contract_plan_destroy(plan: ContractPlan):
    plan.__del__()


def ttc_contract(plan: ContractPlan, x: TTDevice, y: TTDevice, out: torch.Tensor = None, stream=None):
    """Output cores of every pair (ttc.h: ttc_contract) -> (cores float32 [total], ranks [B, L+1], offsets [B])."""
    if out is None:
        out = torch.empty(max(plan.total, 0), dtype=torch.float32, device=x.cores.device)
    if plan._uniform_out is None:
        plan._uniform_out = plan.B <= 1 or bool(np.all(plan.ranks == plan.ranks[0:1]))
    uniform_out = plan._uniform_out
    offs_dev = None
    if not uniform_out:
        if plan._offsets_dev is None or plan._offsets_dev.device != out.device:
            plan._offsets_dev = torch.from_numpy(plan.offsets).to(out.device)
        offs_dev = plan._offsets_dev
    _check(_lib.ttc_contract(plan.handle, ctypes.byref(x.c), ctypes.byref(y.c), _ptr(out) if out.numel() else None,
                             _ptr(offs_dev), _stream_handle(stream)))
    return out, plan.ranks, plan.offsets


def ttc_reconstruct_workspace(t: TTDevice, perm=None) -> int:
    """Bytes of device workspace ttc_reconstruct_ws needs (0: the one-launch shared-memory kernel runs)."""
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    nb = ctypes.c_int64(0)
    _check(_lib.ttc_reconstruct_workspace(ctypes.byref(t.c), _ptr(pm), ctypes.byref(nb)))
    return nb.value


def ttc_reconstruct(t: TTDevice, perm=None, out: torch.Tensor = None, out_offsets=None, stream=None,
                    workspace: torch.Tensor = None) -> torch.Tensor:
    """Dense tensor of every train (ttc.h: ttc_reconstruct / ttc_reconstruct_ws), Eq. 2 order after the optional
    mode permutation perm (1-based; e.g. a contraction plan's perm gives Eq. 8's order).  Returns float32
    [B * prod(dims)] (packed).  workspace: uint8 device scratch of ttc_reconstruct_workspace bytes for trains
    beyond shared memory (allocated here from torch's caching allocator when None and needed)."""
    n_el = int(np.prod(t.dims_np.astype(np.int64))) if t.N else 1
    if out is None:
        out = torch.empty(max(t.B * n_el, 0), dtype=torch.float32, device=t.cores.device)
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    ws = workspace
    if ws is None:
        nb = ttc_reconstruct_workspace(t, pm)
        ws = torch.empty(nb, dtype=torch.uint8, device=t.cores.device) if nb else None
    _check(_lib.ttc_reconstruct_ws(ctypes.byref(t.c), _ptr(pm), _ptr(out) if out.numel() else None, _ptr(out_offsets),
                                   _ptr(ws) if ws is not None else None, int(ws.numel()) if ws is not None else 0,
                                   _stream_handle(stream)))
    if workspace is None:
        _keep_alive(stream, t.cores.device, ws)
    return out


def ttc_tt_svd_capacity(dims, perm=None) -> int:
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    cap = ctypes.c_int64(0)
    _check(_lib.ttc_tt_svd_capacity(int(d.size), _ptr(d), _ptr(pm), ctypes.byref(cap)))
    return cap.value


def ttc_tt_svd_workspace(B: int, dims, perm=None) -> int:
    """Bytes of device workspace ttc_tt_svd's launch pipeline needs for B tensors (0: the fused launch is used)."""
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    nb = ctypes.c_int64(0)
    _check(_lib.ttc_tt_svd_workspace(int(B), int(d.size), _ptr(d), _ptr(pm), ctypes.byref(nb)))
    return nb.value


def _svd_workspace(B, d, pm, device, workspace):
    if workspace is not None:
        return workspace
    nb = ttc_tt_svd_workspace(B, d, pm)
    return torch.empty(max(nb, 16), dtype=torch.uint8, device=device) if nb else None


def _torch_stream(stream, device):
    """The torch.cuda.Stream the call is enqueued on (the current stream when None)."""
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream), device=device)


def _keep_alive(stream, device, *tensors):
    """Tensors allocated here and used by kernels on `stream`: tell torch's caching allocator, so that their memory
    is not handed to another allocation before the kernels on `stream` are done with it."""
    if not torch.cuda.is_available():
        return
    ts = _torch_stream(stream, device)
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(ts)


def ttc_tt_svd_into(dense: torch.Tensor, dims, eps: float, cores: torch.Tensor, ranks: torch.Tensor, perm=None,
                    stream=None, workspace: torch.Tensor = None) -> None:
    """ttc_tt_svd into caller-owned device buffers (no host synchronisation): cores float32 [B * capacity],
    ranks int32 [B, N + 1]; workspace: uint8 device scratch of ttc_tt_svd_workspace bytes (allocated here from
    torch's caching allocator when None)."""
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    n_el = int(np.prod(d.astype(np.int64)))
    B = dense.numel() // max(n_el, 1)
    ws = _svd_workspace(B, d, pm, dense.device, workspace)
    _check(_lib.ttc_tt_svd(int(B), int(d.size), _ptr(d), _ptr(dense) if dense.numel() else None, _ptr(pm),
                           float(eps), _ptr(cores), _ptr(ranks), _ptr(ws) if ws is not None else None,
                           int(ws.numel()) if ws is not None else 0, _stream_handle(stream)))
    if workspace is None:
        _keep_alive(stream, dense.device, ws)


def ttc_tt_svd(dense: torch.Tensor, dims, eps: float, perm=None, stream=None) -> "TTDevice":
    """TT-SVD of B dense tensors (ttc.h: ttc_tt_svd; Alg. 1, optionally of the permuted X^rho of Alg. 2 step 1).
    dense: float32 [B * prod(dims)] on the device.  Returns the trains as a TTDevice (ranks read back to the host,
    trains at b * capacity)."""
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int32))
    pm = None if perm is None else np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    n_el = int(np.prod(d.astype(np.int64)))
    B = dense.numel() // max(n_el, 1)
    cap = ttc_tt_svd_capacity(d, pm)
    cores = torch.zeros(max(B * cap, 1), dtype=torch.float32, device=dense.device)
    ranks = torch.zeros((max(B, 1), d.size + 1), dtype=torch.int32, device=dense.device)
    ws = _svd_workspace(B, d, pm, dense.device, None)
    _check(_lib.ttc_tt_svd(int(B), int(d.size), _ptr(d), _ptr(dense) if dense.numel() else None, _ptr(pm),
                           float(eps), _ptr(cores), _ptr(ranks), _ptr(ws) if ws is not None else None,
                           int(ws.numel()) if ws is not None else 0, _stream_handle(stream)))
    _keep_alive(stream, dense.device, ws, cores, ranks)
    rdims = d if pm is None else d[pm - 1]
    if B and torch.cuda.is_available():
        _torch_stream(stream, dense.device).synchronize()   # the ranks are written by kernels on `stream`
    r = ranks[:B].cpu().numpy()
    return TTDevice(cores, rdims, ranks=r, offsets=np.arange(B, dtype=np.int64) * cap)


def ttc_pair_cost(x: TTDevice, y: TTDevice):
    """Host cost model (ttc.h): per pair sweep MACs and algorithmic HBM bytes."""
    mac = np.zeros(x.B, np.float64)
    by = np.zeros(x.B, np.float64)
    _check(_lib.ttc_pair_cost(ctypes.byref(x.c), ctypes.byref(y.c), _ptr(mac) if x.B else None,
                              _ptr(by) if x.B else None))
    return mac, by


def ttc_partition(cost, k: int) -> np.ndarray:
    """Contiguous k-way split of the batch minimising the largest part cost (ttc.h)."""
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    bounds = np.zeros(k + 1, np.int32)
    _check(_lib.ttc_partition(_ptr(c) if c.size else None, int(c.size), int(k), _ptr(bounds)))
    return bounds
