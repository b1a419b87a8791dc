"""Rounds per greedy sweep task (debug build with -DGREEDY_DBG_ROUNDS=1 writes the round count
into cand_ms): python tools/greedy_rounds.py  (CROSSPIPE_LIB=.../libcrosspipe_dbgr.so)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K  # noqa: E402

g = K.full_sweep_grid()
keys, cand = cp.sweep_shard(g, cand=True)
cand = cand.cpu().numpy().reshape(len(g.pp_vals), len(g.mb_vals), -1, cand.shape[-1])
for i, p in enumerate(g.pp_vals):
    for j, m in enumerate(g.mb_vals):
        row = []
        for c, ns in ((2, 1), (3, 2), (4, 4)):
            r = cand[i, j, :, c]
            row.append(f"ns{ns}: mean {r.mean():7.1f} max {r.max():6d} ops/stage {m * (2 + ns)}")
        print(f"p={p:2d} m={m:3d}", " | ".join(row))

# one long task alone on the GPU: per-round latency of a lone warp
b = K.uniform_instance(32, 128, 4, 100, 100, 100, mlim_x1000=4000, lat=300, bw=200, n_sub=4)
inst = cp.Instances(b)
for _ in range(3):
    r = cp.greedy(inst)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    r = cp.greedy(inst)
e1.record()
torch.cuda.synchronize()
print("lone p=32 m=128 n_sub=4 greedy: %.1f us per call, makespan %d" % (e0.elapsed_time(e1) * 100, int(r["makespan"][0])))
