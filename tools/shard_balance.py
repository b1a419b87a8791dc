"""Time each rank's shard of the config-5 sweep on one GPU (serially) for world sizes 2, 4, 8:
reports per-shard ms, max/mean imbalance and the implied strong-scaling bound."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
g = K.full_sweep_grid()
cg = cp.to_cp_grid(g)
for _ in range(2):
    cp.sweep_shard(g, cgrid=cg)
torch.cuda.synchronize()
def t(lo, hi, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cp.sweep_shard(g, lo, hi, cgrid=cg)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
full = t(0, g.n_points)
print(f"full sweep {full:.3f} ms")
for world in (2, 4, 8):
    b = cp.sweep_partition(g, world, cgrid=cg)
    ts = [t(b[r], b[r + 1]) for r in range(world)]
    print(f"world {world}: shards ms {[round(x, 3) for x in ts]} max/mean {max(ts) / (sum(ts) / world):.2f} "
          f"speedup bound {full / max(ts):.2f}")
    def tr(rk, reps=3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            cp.sweep_shard_rank(g, rk, world, cgrid=cg)
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    tb = [tr(r) for r in range(world)]
    print(f"world {world} (rank-blocked): shards ms {[round(x, 3) for x in tb]} max/mean {max(tb) / (sum(tb) / world):.2f} "
          f"speedup bound {full / max(tb):.2f}")
