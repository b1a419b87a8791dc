"""SPEC.md:548 acceptance 5(d) on down-scaled E1 replicas (PAPER.md :497 "The greedy CrossUDSub
schedule matches the solver-based CrossUD in most delay regimes"): 4 stages over 2 DCs (2 + 2),
F = D = W = T_F, 1F1B memory budget, (T_lat/T_F, T_bw/T_F) in {0, 0.5, 1, 2}^2, m microbatches.
Exact CrossUD = cp_exact (the makespan optimum over all whole-block split plans, NEXT 3); greedy
CrossUDSub = the best of cp_greedy with n_sub 1/2/4.  usage: python tools/e1_exact.py M [out.json]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
from workloads.core import InstanceBatch

m = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = sys.argv[2] if len(sys.argv) > 2 else f"profiles/e1_exact_m{m}_r01.json"
f = 100
ratios = [0, 0.5, 1, 2]
pts = [(a, b) for a in ratios for b in ratios]
mk = lambda ns: InstanceBatch.concat([K.uniform_instance(4, m, 2, f, f, f, lat=int(a * f), bw=int(b * f), n_sub=ns)
                                      for (a, b) in pts])
ex_inst = cp.Instances(mk(1))
torch.cuda.synchronize()
# warm start: the greedy's n_sub = 1 makespan (a plan of the enumerated set) seeds the cut
g1 = cp.greedy(ex_inst)["makespan"]
torch.cuda.synchronize()
t0 = time.perf_counter()
ex = cp.exact(ex_inst, max_plans=(1 << 51), upper=g1)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
ems, est = ex["makespan"].cpu().numpy(), ex["status"].cpu().numpy()
g = np.min(np.stack([cp.greedy(cp.Instances(mk(ns)))["makespan"].cpu().numpy() for ns in (1, 2, 4)]), axis=0)
gap = g / np.where(ems > 0, ems, 1) - 1
ok = est == 0
doc = {"workload": f"E1 replica: p=4, 2 DCs (2+2), m={m}, F=D=W={f} ticks, 1F1B budget", "points": pts,
       "exact_makespan": ems.tolist(), "exact_status": est.tolist(), "greedy_best_makespan": g.tolist(),
       "greedy_gap_vs_exact": np.round(gap, 4).tolist(), "exact_search_s": round(dt, 3),
       "summary": {"points solved": int(ok.sum()), "greedy within 5% of exact (SPEC 5(d): >= 80%)":
                   f"{int((gap[ok] <= 0.05).sum())} of {int(ok.sum())}",
                   "greedy == exact": f"{int((gap[ok] == 0).sum())} of {int(ok.sum())}",
                   "max gap": round(float(gap[ok].max()), 4) if ok.any() else None}}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as fh:
    json.dump(doc, fh)
print(json.dumps(doc["summary"]), "exact search", round(dt, 3), "s")
