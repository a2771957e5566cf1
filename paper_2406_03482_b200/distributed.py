"""Multi-GPU layout of the decode path: one process per GPU, units sharded.

A unit (one (batch, kv-head) pair) is independent of every other unit on the
hot path, so the cache is partitioned into contiguous unit blocks, one per
rank; each GPU quantizes, stores and decodes only its own units and no
collective touches the data path.  The only exchange is the
optional gather of the per-unit decode outputs (a few hundred KB per step) for
callers that want the full [units, G, d] result on every rank -- an
all_gather over NCCL (NVLink/NVSwitch) on GPUs, gloo in CPU tests.

The reference is single-process; this module has no reference
counterpart beyond the unit independence it relies on (kvcache.py:189-196).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class UnitShard:
    """Contiguous block [start, start + count) of the global unit range."""

    rank: int
    world: int
    total: int
    start: int
    count: int

    @property
    def stop(self) -> int:
        return self.start + self.count


def shard_units(total_units: int, world: int, rank: int) -> UnitShard:
    """Balanced contiguous split: the first (total % world) ranks get one extra unit."""
    if total_units < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard request: total={total_units} world={world} rank={rank}")
    base, extra = divmod(total_units, world)
    start = rank * base + min(rank, extra)
    return UnitShard(rank, world, total_units, start, base + (1 if rank < extra else 0))


def shard_of(total_units: int) -> UnitShard:
    """This process's shard under the current default process group (1 rank if none)."""
    if dist.is_available() and dist.is_initialized():
        return shard_units(total_units, dist.get_world_size(), dist.get_rank())
    return shard_units(total_units, 1, 0)


def gather_units(local: torch.Tensor, shard: UnitShard, group=None) -> torch.Tensor:
    """All-gather per-unit results [count, ...] of every rank into [total, ...].

    Uneven shards are padded to the largest shard for the collective and then
    compacted, so the result is the exact concatenation in unit order.
    """
    if shard.world == 1:
        return local
    max_count = -(-shard.total // shard.world)
    pad = torch.zeros((max_count,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: shard.count] = local
    out = torch.empty((shard.world * max_count,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = []
    for r in range(shard.world):
        s = shard_units(shard.total, shard.world, r)
        parts.append(out[r * max_count: r * max_count + s.count])
    return torch.cat(parts, dim=0)
