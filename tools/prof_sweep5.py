import sys; sys.path.insert(0,'/root/repo')
import torch, paper_2507_00217_b200 as cp
from workloads import configs as K
g = K.full_sweep_grid()
for _ in range(3): cp.sweep_shard(g)
torch.cuda.synchronize()
