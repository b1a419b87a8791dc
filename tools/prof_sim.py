"""Profiling driver: one config-4 cp_simulate launch (after warm-up) for ncu, or a
config-3 greedy / config-2 sweep launch.  usage: python tools/prof_sim.py [sim|simtl|greedy|sweep2] [n]  (simtl: with the full timeline)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K, plans as PL  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "sim"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
if what in ("sim", "simtl"):
    b = K.perturbed_instance()
    inst = cp.Instances(b)
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED)
    for _ in range(3):
        r = cp.simulate(inst, ops, ln, best=True, timeline=what == "simtl")
elif what == "greedy":
    gi = cp.Instances(K.greedy_batch(n))
    for _ in range(3):
        r = cp.greedy(gi)
else:
    g = K.gpt16_grid()
    for _ in range(3):
        r = cp.sweep_shard(g)
torch.cuda.synchronize()
print("done", what, n)
