"""Per-task durations of the sweep's greedy tasks (debug build -DGREEDY_DBG_ROUNDS=2 writes
globaltimer end - start, 0.1 us units, into cand_ms): one 1/8 rank shard of config 5 vs the
p = 32, m = 128 class alone.  CROSSPIPE_LIB=.../libcrosspipe_dbgt.so python tools/greedy_task_times.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K  # noqa: E402


def show(tag, cand, shape, sel):
    c = cand.cpu().numpy().reshape(shape + (-1,))
    for c_i, ns in ((2, 1), (3, 2), (4, 4)):
        v = c[sel][..., c_i].ravel()
        v = v[v > 0] / 10.0
        print(f"{tag} ns{ns}: n {v.size} mean {v.mean():7.1f} us  max {v.max():7.1f} us")


g = K.full_sweep_grid()
cg = cp.to_cp_grid(g)
for _ in range(3):
    keys, cand = cp.sweep_shard_rank(g, 0, 8, cand=True, cgrid=cg)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
keys, cand = cp.sweep_shard_rank(g, 0, 8, cand=True, cgrid=cg)
t1.record()
torch.cuda.synchronize()
print("shard 0/8: %.3f ms" % t0.elapsed_time(t1))
shape = (len(g.pp_vals), len(g.mb_vals), 1024)
show("shard p=32 m=128", cand, shape, (3, 4, slice(0, 128)))
show("shard p=24 m=128", cand, shape, (2, 4, slice(0, 128)))
show("shard p=32 m=64 ", cand, shape, (3, 3, slice(0, 128)))

g2 = K.full_sweep_grid()
g2.pp_vals, g2.mb_vals = [32], [8, 128]      # two mb blocks: the m = 128 block takes the long-task launches
cg2 = cp.to_cp_grid(g2)
for _ in range(3):
    keys, cand = cp.sweep_shard_rank(g2, 0, 8, cand=True, cgrid=cg2)
torch.cuda.synchronize()
t0.record()
keys, cand = cp.sweep_shard_rank(g2, 0, 8, cand=True, cgrid=cg2)
t1.record()
torch.cuda.synchronize()
print("class p=32 m=128 alone (1/8): %.3f ms" % t0.elapsed_time(t1))
show("alone p=32 m=128", cand, (1, 2, 1024), (0, 1, slice(0, 128)))
