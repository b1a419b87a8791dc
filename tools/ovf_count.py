import os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K, plans as PL
b = K.perturbed_instance(); inst = cp.Instances(b)
n = 1_000_000
ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED)
ws = cp.api._workspace(0, inst.desc(), n, ops.device)
r = cp.simulate(inst, ops, ln, best=True, ws=ws)
torch.cuda.synchronize()
print("ovf_count", int(ws[:4].view(torch.int32)[0]))
