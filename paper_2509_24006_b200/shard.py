"""(batch x head) sharding of SLA problems across ranks -- one process per GPU.

The path shards with no data-path collective: every (batch, head) unit is independent in the
forward and the backward (the reference has no cross-head state), so rank r simply
runs its contiguous range of units.  The only collective is the optional VALIDATION gather of
outputs / gradients to rank 0 (NCCL over NVLink on GPUs, gloo in the CPU tests), which never
sits inside a timed region.  W is per head and shared by the batch, so when the batch dimension
is split the per-head dW partials are summed with one d x d all-reduce (off the hot path).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int   # first unit (flattened b * H + h)
    count: int   # units on this rank

    @property
    def units(self) -> range:
        return range(self.first, self.first + self.count)


def partition_units(n_units: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split: the first n_units % world ranks take one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("partition_units: bad rank / world")
    base, extra = divmod(n_units, world)
    first = rank * base + min(rank, extra)
    return Shard(rank, world, first, base + (1 if rank < extra else 0))


def batch_slices(batch: int, heads: int, shard: Shard):
    """(b, h) pairs of a shard, in unit order."""
    return [(u // heads, u % heads) for u in shard.units]


def gather_units(local: torch.Tensor, shard: Shard, n_units: int, group=None) -> torch.Tensor | None:
    """Validation gather of per-unit results [count, ...] to rank 0 as [n_units, ...].

    Works for uneven shards (pads to the largest shard, then trims).  Returns None on ranks
    other than 0."""
    world = shard.world
    if world == 1:
        return local
    if local.is_cuda and dist.get_backend(group) == "gloo":  # gloo moves host tensors
        out = gather_units(local.cpu(), shard, n_units, group)
        return None if out is None else out.to(local.device)
    biggest = -(-n_units // world)
    pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if shard.rank != 0:
        return None
    parts = []
    for r in range(world):
        s = partition_units(n_units, world, r)
        parts.append(bufs[r][: s.count])
    return torch.cat(parts, 0)


def allreduce_dw(dw: torch.Tensor, group=None) -> torch.Tensor:
    """Sum per-head dW partials when the batch of one head is split across ranks."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dw, group=group)
    return dw
