"""Repeat the generic-greedy ring-overflow fix-up scenario and report any run that differs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
batch = K.random_instances(150, seed=26, max_p=32, max_m=14)
gi = cp.Instances(batch)
ref = cp.greedy(gi, stats=True, timeline=True)
torch.cuda.synchronize()
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    ring = 1 + (it % 3)
    g = cp.greedy(gi, stats=True, timeline=True, ring=ring)
    r2 = cp.greedy(gi, stats=True, timeline=True)
    torch.cuda.synchronize()
    for name, other in (("ring", g), ("default", r2)):
        for k in ("makespan", "status", "peak_mem", "stage_stats", "ops", "len", "t_start"):
            if not torch.equal(other[k], ref[k]):
                d = (other[k] != ref[k])
                while d.dim() > 1: d = d.any(dim=-1)
                items = torch.nonzero(d).flatten().tolist()[:5]
                print(f"iter {it} ring {ring} {name}: {k} differs at items {items}", flush=True)
                bad += 1
print("bad", bad)
