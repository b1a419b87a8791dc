import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
b = K.tiny(1.0, 0.5) if len(sys.argv) < 2 else K.random_instances(int(sys.argv[1]), seed=11, max_p=32, max_m=20)
g = cp.greedy(cp.Instances(b))
torch.cuda.synchronize()
print("ok", g["makespan"][:4].tolist())
