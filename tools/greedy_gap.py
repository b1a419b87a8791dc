"""Greedy vs exact optimum on random tiny instances (PAPER.md :497 "The greedy CrossUDSub schedule
matches the solver-based CrossUD in most delay regimes").  Random
non-uniform instances (workloads.configs.random_instances: per-stage costs, memory budgets, DP tails,
ZeRO-1, cross-DC and intra-DC delays) with p <= 4, m <= 4, whole blocks (n_sub = 1).  Exact =
cp_exact (optimum over all valid whole-block plans, warm-started by the greedy); greedy = cp_greedy
with n_sub = 1 (same plan space) and the best of n_sub 1/2/4 (CrossUDSub).  Spot-checks instances
against the oracle's exhaustive enumeration.  usage: python tools/greedy_gap.py [n] [out.json]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from workloads import configs as K

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/greedy_gap_r01.json"
b = K.random_instances(n, seed=97, max_p=4, max_m=4, intra_delay=True)
b.n_sub[:n] = 1
inst = cp.Instances(b)
g1 = cp.greedy(inst)
torch.cuda.synchronize()
t0 = time.perf_counter()
ex = cp.exact(inst, upper=g1["makespan"], max_plans=(1 << 51))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
best = g1["makespan"].cpu().numpy().astype(np.int64)
for ns in (2, 4):
    bb = K.random_instances(n, seed=97, max_p=4, max_m=4, intra_delay=True)
    bb.n_sub[:n] = ns
    for fld in ("t_f", "t_d", "t_w"):                 # every sub-block >= 1 tick (Q12)
        getattr(bb, fld)[:n] = np.maximum(getattr(bb, fld)[:n], ns)
    r = cp.greedy(cp.Instances(bb))
    ok = r["status"].cpu().numpy() == 0
    best = np.where(ok, np.minimum(best, r["makespan"].cpu().numpy()), best)
ems, est = ex["makespan"].cpu().numpy(), ex["status"].cpu().numpy()
gs = g1["makespan"].cpu().numpy()
solved = est == 0
gap1 = gs[solved] / ems[solved] - 1
gapb = best[solved] / ems[solved] - 1
from oracle import oracle as O
O.build()
checked = 0
for i in np.random.default_rng(98).choice(np.nonzero(solved)[0], 20, replace=False):
    e = O.enumerate_opt(b.item(int(i)), max_plans=3_000_000)
    if e["evaluated"] >= 0:
        assert e["makespan"] == ems[i], (i, e["makespan"], ems[i])
        checked += 1
q = lambda x: {k: round(float(np.quantile(x, v)), 4) for k, v in (("p50", .5), ("p90", .9), ("p99", .99), ("max", 1.0))}
doc = {"workload": f"{n} random tiny instances (p <= 4, m <= 4, n_sub = 1, random costs / memory / DP / ZeRO-1 / delays)",
       "solved": int(solved.sum()), "exact_search_s": round(dt, 3), "oracle_spot_checked": checked,
       "greedy_n_sub1": {"optimal": f"{int((gap1 == 0).sum())} of {int(solved.sum())}",
                         "within 5%": f"{int((gap1 <= 0.05).sum())} of {int(solved.sum())}", "gap": q(gap1)},
       "crossudsub_best_of_n_sub_1_2_4": {"<= exact": f"{int((gapb <= 0).sum())} of {int(solved.sum())}",
                                          "within 5%": f"{int((gapb <= 0.05).sum())} of {int(solved.sum())}",
                                          "gap": q(gapb)}}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(doc, f)
print(json.dumps(doc, indent=1))
