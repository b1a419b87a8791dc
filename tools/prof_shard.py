"""One rank shard of the config-5 sweep (after warm-up) for an ncu launch list:
python tools/prof_shard.py [rank] [world]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K  # noqa: E402

rank = int(sys.argv[1]) if len(sys.argv) > 1 else 0
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = K.full_sweep_grid()
cg = cp.to_cp_grid(g)
for _ in range(3):
    cp.sweep_shard_rank(g, rank, world, cgrid=cg)
torch.cuda.synchronize()
print("done", rank, world)
