"""The sweep's longest greedy tasks alone (p = 32, m = 128, n_sub = 4; one 1/8 rank slice = 128
tasks, one warp each) for an ncu capture of their round latency: python tools/prof_long.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K  # noqa: E402

g = K.full_sweep_grid()
g.pp_vals, g.mb_vals, g.cand_mask = [32], [8, 128], 0b10000   # the m = 128 block takes the long-task launches
cg = cp.to_cp_grid(g)
for _ in range(2):
    cp.sweep_shard_rank(g, 0, 8, cgrid=cg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cp.sweep_shard_rank(g, 0, 8, cgrid=cg)
e1.record()
torch.cuda.synchronize()
print("p=32 m=8/128 n_sub=4 slice: %.3f ms" % e0.elapsed_time(e1))
