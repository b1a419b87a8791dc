"""Multi-GPU sharding (one process per GPU, torch.distributed over NCCL).

The hot path partitions naturally (independent grid points / schedules), so ranks
share no data until the single final exchange: one all_reduce(MIN) over int64
packed keys, which is an allgather + argmin in one collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import api


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def sweep(grid, *, cand=False, group=None, stream=None, bounds=None, shard_fn=None, blocked=True):
    """cp_sweep(grid) = one shard per rank + all_reduce(MIN) of the int64 keys.

    Default: blocked ownership (cp_sweep_shard_rank; every rank evaluates its slice of every (p, m)
    block, so all ranks carry the same mix of work).  `bounds` (or blocked=False) selects contiguous
    point ranges instead (cp_sweep_partition's cost-balanced cuts).  Returns (keys [n_points] on
    every rank, cand_ms of the local shard or None).  `shard_fn` (grid, lo, hi) -> (keys, cand_ms)
    replaces the CUDA shard (tests drive the host logic on CPU; contiguous ranges)."""
    rank, ws = world()
    cg = api.to_cp_grid(grid)
    if shard_fn is None and bounds is None and blocked:
        keys, cm = api.sweep_shard_rank(grid, rank, ws, cand=cand, stream=stream, cgrid=cg)
    else:
        if bounds is None:
            bounds = api.sweep_partition(grid, ws, cgrid=cg)
        lo, hi = bounds[rank], bounds[rank + 1]
        if shard_fn is None:
            keys, cm = api.sweep_shard(grid, lo, hi, cand=cand, stream=stream, cgrid=cg)
        else:
            keys, cm = shard_fn(grid, lo, hi)
    if ws > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    return keys, cm


def shard_range(n: int, rank: int, ws: int):
    """Contiguous equal split of n uniform-cost items (schedules / instances)."""
    return n * rank // ws, n * (rank + 1) // ws


def best_schedule(best_key: torch.Tensor, group=None):
    """all_reduce(MIN) of the (makespan << 32 | index) key of each rank's best schedule."""
    if world()[1] > 1:
        dist.all_reduce(best_key, op=dist.ReduceOp.MIN, group=group)
    return best_key
