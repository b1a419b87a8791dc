"""Find greedy instances where the GPU differs from the oracle within regression chunks; print details.
usage: python tools/greedy_diff.py CHUNK [CHUNK ...]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from tests import greedy_regress_worker as Wk
from workloads import configs as K, unpack_plans
from oracle import oracle as O
O.build()
for k in map(int, sys.argv[1:]):
    prm = Wk.chunk_params(k)
    batch = K.random_instances(Wk.N_CHUNK, seed=prm["seed"], max_p=prm["max_p"], max_m=prm["max_m"], intra_delay=prm["intra_delay"])
    g = cp.greedy(cp.Instances(batch)); torch.cuda.synchronize()
    codes, lens = unpack_plans(g["ops"].cpu().numpy().view(np.uint32), g["len"].cpu().numpy().view(np.uint16))
    for i in range(len(batch)):
        d = batch.item(i); w = O.greedy(d); p = d["p"]; L = int(w["len"][0])
        gs, gm, gp = int(g["status"][i]), int(g["makespan"][i]), int(g["peak_mem"][i])
        same = gs == w["status"] and gm == w["makespan"] and gp == w["peak_mem"] and np.array_equal(lens[i, :p], w["len"][:p]) and np.array_equal(codes[i, :p, :L], w["codes"][:p, :L])
        if not same:
            print("chunk", k, "item", i, "p", p, "m", d["m"], "nsub", d["n_sub"], "gpu", (gs, gm, gp), "oracle", (w["status"], w["makespan"], w["peak_mem"]))
            for s in range(p):
                a = "".join("FBDW"[c] for c in codes[i, s, :L]); b = "".join("FBDW"[c] for c in w["codes"][s, :L])
                if a != b:
                    j = next(t for t in range(L) if a[t] != b[t])
                    print("  stage", s, "first diff at", j, "gpu", a[max(0,j-6):j+8], "oracle", b[max(0,j-6):j+8])
            print("  inst", json.dumps({kk: (v.tolist() if hasattr(v, "tolist") else v) for kk, v in d.items()})[:1500])
