import sys, json; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2507_00217_b200 as cp
from oracle import oracle as O
from tests.test_parity_gpu import _loop_batch
from tests.gpu_util import plans_to_device, to_host
O.build()
batch, plans, ops, ln = _loop_batch(120, 62, 2, 10)
o, l_ = plans_to_device(ops, ln)
r = to_host(cp.simulate(cp.Instances(batch), o, l_, stats=True, timeline=True, loop=True))
n = 0
for i, pl in enumerate(plans):
    d = batch.item(i); w = O.simulate_loop(d, pl, timeline=True)
    if int(r["makespan"][i]) != w["makespan"]:
        n += 1
        if n > 2: continue
        p = d["p"]
        print("item", i, "p", p, "m", d["m"], "nsub", d["n_sub"], "gpu", int(r["makespan"][i]), "oracle", w["makespan"])
        print(" inst", {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in d.items()})
        for s in range(p):
            L = len(pl[s])
            print("  s", s, "plan", [("FBDW"[x & 3] + str(x >> 2)) for x in pl[s]])
            print("     gpu", list(r["t_start"][i][s, :L]))
            print("     orc", list(w["t_start"][s, :L]))
print("mismatches", n)
