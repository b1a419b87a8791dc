"""Dump the GPU greedy plan rows of regression chunk K, items I... as JSON (for offline comparison)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from tests import greedy_regress_worker as Wk
from workloads import configs as K, unpack_plans
k = int(sys.argv[1]); items = [int(x) for x in sys.argv[2:]]
prm = Wk.chunk_params(k)
batch = K.random_instances(Wk.N_CHUNK, seed=prm["seed"], max_p=prm["max_p"], max_m=prm["max_m"], intra_delay=prm["intra_delay"])
g = cp.greedy(cp.Instances(batch)); torch.cuda.synchronize()
codes, lens = unpack_plans(g["ops"].cpu().numpy().view(np.uint32), g["len"].cpu().numpy().view(np.uint16))
out = {}
for i in items:
    p = int(batch.p[i])
    out[i] = {"rows": ["".join("FBDW"[c] for c in codes[i, s, :lens[i, s]]) for s in range(p)], "makespan": int(g["makespan"][i])}
print(json.dumps(out))
