"""Multi-GPU sharding of a batch of independent TT pairs.

One process per GPU (torchrun), torch.distributed for the plumbing.  Pairs are independent, so the batch is
split into contiguous, cost-balanced ranges with `ttc_partition` (identical on every rank: a pure function of
the host cost vector); each rank runs `ttc_inner` on its range only.  The only exchange step is optional: the
north star's gather of the per-pair results (4 bytes per pair) with one `all_gather_into_tensor` padded to the
largest shard, then compacted by the bounds.  No data-path collective is involved in the computation itself.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import TTDevice, _keep_alive, ttc_inner, ttc_pair_cost, ttc_partition


def shard_bounds(cost: Sequence[float], world: int) -> np.ndarray:
    """Contiguous k-way split of the batch minimising the largest shard cost (ttc_partition)."""
    return ttc_partition(np.asarray(cost, dtype=np.float64), int(world))


def shard_view(t: TTDevice, lo: int, hi: int) -> TTDevice:
    """Pairs [lo, hi) of a batch as a TTDevice over the same core buffer (no copy)."""
    ranks = t.rank_rows()[lo:hi]
    offs = (t.offsets_np if t.offsets_np is not None else t._packed_offsets())
    offs = offs[lo:hi] if offs is not None else None
    return TTDevice(t.cores, t.dims_np, ranks=ranks, offsets=offs)


def gather_results(local: torch.Tensor, bounds: np.ndarray, group=None) -> torch.Tensor:
    """All-gather per-rank result vectors of (possibly) different lengths, padded to the largest shard,
    compacted into pair order.  Works on NCCL (device tensors) and gloo (host tensors)."""
    world = dist.get_world_size(group)
    sizes = np.diff(np.asarray(bounds, dtype=np.int64))
    S = int(sizes.max()) if sizes.size else 0
    pad = torch.zeros(S, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    full = torch.empty(world * S, dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, pad, group=group)
    else:
        parts = list(full.split(S))
        dist.all_gather(parts, pad, group=group)
    keep = [full[r * S: r * S + int(sizes[r])] for r in range(world)]
    return torch.cat(keep) if keep else full[:0]


def sharded_inner(x: TTDevice, y: TTDevice, group=None, gather: bool = True, cost: Optional[np.ndarray] = None,
                  stream=None):
    """<X_b, Y_b> of the whole batch with this rank computing its cost-balanced range.

    Returns (result, bounds): the gathered float32 [B] results in pair order (gather=True), or this rank's
    shard results."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if cost is None:
        cost, _ = ttc_pair_cost(x, y)
    bounds = shard_bounds(cost, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    xs, ys = shard_view(x, lo, hi), shard_view(y, lo, hi)
    out = ttc_inner(xs, ys, stream=stream)
    # the shard views' device rank / offset tables are freed when this function returns, possibly while the
    # kernel on `stream` still reads them: hand them to the caching allocator's stream tracking
    _keep_alive(stream, x.cores.device, xs.ranks_dev, xs.offsets_dev, ys.ranks_dev, ys.offsets_dev)
    if not gather:
        return out, bounds
    return gather_results(out, bounds, group), bounds
