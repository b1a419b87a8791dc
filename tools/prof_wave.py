"""One Wave- (or Loop-) pattern cp_simulate launch (bench workload) for ncu: python tools/prof_wave.py [n] [loop]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K, plans as PL
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
loop = len(sys.argv) > 2 and sys.argv[2] == 'loop'
inst = cp.Instances(K.loop_instance() if loop else K.wave_instance())
ops, ln = PL.wave_plans_device(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32, loop=loop)
for _ in range(3):
    r = cp.simulate(inst, ops, ln, best=True, **({'loop': True} if loop else {'wave': True}))
torch.cuda.synchronize()
print("done", n)
