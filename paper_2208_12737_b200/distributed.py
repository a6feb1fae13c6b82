"""Multi-GPU plumbing: pose sharding.

Poses are independent units (the reference guarantees ray and pose
independence, ``SPEC.md:237,407``), so the path shards over a batch of poses
with NO collective inside the render loop:

1. the CT is broadcast once from rank 0 (``broadcast_volume``; NCCL over
   NVLink on the GPU box, gloo in the CPU tests);
2. each rank renders its contiguous block of poses (``shard_range``);
3. images / per-pose gradients are gathered only when one rank needs them
   (``gather_rows``, padded all-gather for uneven shards);
4. a shared batched-registration loss is the only all-reduce
   (``allreduce_sum``: a few floats).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Balanced contiguous block [start, stop) of n items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(int(n), world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def broadcast_volume(vol: torch.Tensor | None, shape, device, dtype=torch.float32, src: int = 0,
                     group=None) -> torch.Tensor:
    """Every rank gets rank `src`'s volume (one collective, before any render)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return vol.to(device=device, dtype=dtype)
    if dist.get_rank(group) == src:
        buf = vol.to(device=device, dtype=dtype).contiguous()
    else:
        buf = torch.empty(tuple(shape), device=device, dtype=dtype)
    dist.broadcast(buf, src=src, group=group)
    return buf


def gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather per-pose rows (images (b, H, W) or gradients (b, k)) from
    uneven contiguous shards back into global order (n_total, ...)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rows = [shard_range(n_total, r, world) for r in range(world)]
    cap = max(stop - start for start, stop in rows)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:stop - start] for b, (start, stop) in zip(bufs, rows)], dim=0)


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """Shared-loss reduction for batched registration (a few floats)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def max_over_ranks(value: float, device, group=None) -> float:
    """Timing rule: report the slowest rank."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
