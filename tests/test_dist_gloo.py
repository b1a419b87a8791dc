"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path: cost-balanced
sweep partition + one all_reduce(MIN) over int64 packed keys, and the best-schedule
reduction.  Per-shard keys come from the oracle here (no GPU); the GPU shards are covered
by tests/test_parity_gpu.py::test_sweep_config5_sample_and_shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import configs as K
from workloads.core import Grid

KEY_NONE = 2**63 - 1


def small_grid():
    base = K.tiny(0, 0)
    r = np.array([0, 50, 100, 200])
    return Grid(base=base, n_dc=2, pp_vals=[2, 4], mb_vals=[3, 8], lat=r, bw=r, mlim_x1000=np.array([1000, 2000]),
                tdp=np.array([0]), cand_mask=0b11111)


def oracle_shard(grid, lo, hi):
    from oracle import oracle as O
    keys = torch.full((grid.n_points,), KEY_NONE, dtype=torch.int64)
    G, keep = O.to_or_grid(grid)
    for k in range(lo, hi):
        key, _ = O.sweep_point(grid, k, G=G)
        keys[k] = KEY_NONE if key == 2**64 - 1 else key
    return keys, None


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_00217_b200 import dist as cpd
        g = small_grid()
        keys, _ = cpd.sweep(g, shard_fn=oracle_shard)
        # best-schedule reduction: each rank contributes its local best (makespan << 32 | id)
        local = torch.tensor([((1000 + 7 * rank) << 32) | (rank * 100 + 3)], dtype=torch.int64)
        cpd.best_schedule(local)
        lo, hi = cpd.shard_range(1000, rank, world)
        q.put((rank, keys.numpy().tolist(), int(local.item()), (lo, hi)))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sweep_allreduce_min_gloo(world, oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    ref, _ = oracle_shard(small_grid(), 0, small_grid().n_points)
    for rank, keys, best, (lo, hi) in out:
        assert keys == ref.numpy().tolist()                 # every rank holds the full argmin table
        assert best == (1000 << 32) | 3                     # global best = rank 0's
    assert [o[3] for o in out] == [(0, 500), (500, 1000)]
    assert all(k != KEY_NONE for k in ref.numpy())          # every point has a feasible candidate
