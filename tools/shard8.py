import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
g = K.full_sweep_grid(); cg = cp.to_cp_grid(g)
for _ in range(3): cp.sweep_shard(g, cgrid=cg)
torch.cuda.synchronize()
def tr(rk, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); cp.sweep_shard_rank(g, rk, 8, cgrid=cg); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts=[]
for _ in range(5):
    e0.record(); cp.sweep_shard(g, cgrid=cg); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
tb = [tr(r) for r in range(8)]
print(os.environ.get("TAG",""), "full %.3f" % sorted(ts)[2], "shards median-of-5", [round(x, 3) for x in tb], "max %.3f" % max(tb))
