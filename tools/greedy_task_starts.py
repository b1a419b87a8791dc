"""Start (CROSSPIPE_LIB=..._dbgs.so) or end (..._dbge.so) times of the greedy tasks of one 1/8 rank
shard of config 5, relative to the earliest start / per class: python tools/greedy_task_starts.py start|end"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K  # noqa: E402

what = sys.argv[1]
g = K.full_sweep_grid()
cg = cp.to_cp_grid(g)
for _ in range(3):
    keys, cand = cp.sweep_shard_rank(g, 0, 8, cand=True, cgrid=cg)
torch.cuda.synchronize()
c = cand.cpu().numpy().reshape(len(g.pp_vals), len(g.mb_vals), 1024, -1)[:, :, :128, 2:5].astype(np.int64)
base = c[c > 0].min() if what == "start" else None
if what == "end":
    base = int(os.environ.get("T0", "0"))
for i, p in enumerate(g.pp_vals):
    for j, m in enumerate(g.mb_vals):
        v = c[i, j]
        v = v[v > 0] - c[c > 0].min()
        print(f"{what} p={p:2d} m={m:3d}: min {v.min() / 10:7.1f} us  median {np.median(v) / 10:7.1f}  max {v.max() / 10:7.1f}")
