"""Query sharding across GPUs (one process per GPU, torch.distributed).

The path shards by query: every rank holds the full data set (replicated
from rank 0 with one broadcast over NCCL/NVLink) and interpolates a
contiguous slice of the queries.  The only other exchange is a 4-double
all-reduce that gives every rank the global bbox(data ∪ all queries), so all
ranks build the identical grid and use the same area / snap tolerance —
which makes results bit-identical for any number of GPUs.  Works with the
nccl backend (CUDA tensors) and gloo (CPU tensors, used by the tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n_total items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad world/rank {world}/{rank}")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_bbox(local_box, dist, device=None):
    """All-reduce per-rank (min_x, min_y, max_x, max_y) into the union box."""
    import torch
    t = torch.tensor([local_box[0], local_box[1], -local_box[2], -local_box[3]],
                     dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    v = t.tolist()
    return np.array([v[0], v[1], -v[2], -v[3]])


def replicate(tensor, dist, src: int = 0):
    """Broadcast rank `src`'s data tensor (3 x m FP64: x, y, z) in place."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(tensor, src=src)
    return tensor


def gather_results(local, n_total: int, dist, device=None):
    """Assemble per-rank result slices (FP64) into the full array on every
    rank (all_gather of equal-size padded slices); used for verification."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    size = -(-n_total // world)
    pad = torch.zeros(size, dtype=torch.float64, device=device)
    pad[: local.numel()] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    out = []
    for r in range(world):
        lo, hi = shard_range(n_total, world, r)
        out.append(parts[r][: hi - lo])
    return torch.cat(out)
