import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, copy
import paper_2507_00217_b200 as cp
from workloads import configs as K
from workloads.core import Grid
g0 = K.full_sweep_grid()
for mb, mem, mask, label in (([128], [4000], 0b10000, "p32 m128 x4 greedy4"), ([128], [1000], 0b10000, "p32 m128 x1 greedy4"),
                              ([128], [4000], 0b00010, "p32 m128 1F1B"), ([64], [1500], 0b00100, "p32 m64 x1.5 greedy1")):
    g = Grid(base=g0.base, n_dc=4, pp_vals=[32], mb_vals=mb, lat=g0.lat[:1], bw=g0.bw[:1], mlim_x1000=np.array(mem), tdp=np.array([0]), cand_mask=mask)
    for _ in range(2): cp.sweep_shard(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): cp.sweep_shard(g)
    e1.record(); torch.cuda.synchronize()
    print(label, "single-task sweep ms", round(e0.elapsed_time(e1) / 5, 3))
