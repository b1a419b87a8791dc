"""E1 delay-sensitivity table (§5.1, Fig. pre_delay_sensitivity) on the GPU sweep:
4 stages / 2 DCs / 8 microbatches, T_lat/T_F x T_bw/T_F grid, candidates GPipe, 1F1B, greedy
n_sub 1/2/4 (CrossUDSub), ZB-H1.  Slowdown is relative to ZB-H1 at zero delay (the paper's
reference ZBV needs multi-chunk Wave plans, NEXT 1).  Spot-checks points against the oracle.
usage: python tools/e1_grid.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from workloads import configs as K

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/e1_delay_sensitivity_r01.json"
grid = K.e1_grid()
keys, cm = cp.sweep_shard(grid, cand=True)
torch.cuda.synchronize()
cm = cm.cpu().numpy().reshape(len(grid.lat), len(grid.bw), 6)       # point = i_lat * n_bw + i_bw
names = ["GPipe", "1F1B", "CrossUDSub n_sub=1", "CrossUDSub n_sub=2", "CrossUDSub n_sub=4", "ZB-H1"]
ref = float(cm[0, 0, 5])
ratios = (np.asarray(grid.lat) / K.T_F).round(4).tolist()
table = {names[c]: (np.where(cm[:, :, c] >= 0, cm[:, :, c] / ref, np.nan)).round(4).tolist() for c in range(6)}
g = {n: cm[:, :, c] for c, n in enumerate(names)}
best_greedy = np.min(np.stack([g[n] for n in names[2:5]]), axis=0)
summary = {
    "reference": "ZB-H1 at zero delay = %d ticks" % ref,
    "GPipe feasible points": int((cm[:, :, 0] >= 0).sum()),
    "greedy(best n_sub) <= ZB-H1 at": f"{int((best_greedy <= g['ZB-H1']).sum())} of {best_greedy.size} points",
    "greedy(best n_sub) <= 1F1B at": f"{int((best_greedy <= g['1F1B']).sum())} of {best_greedy.size} points",
    "ZB-H1 <= 1F1B at": f"{int((g['ZB-H1'] <= g['1F1B']).sum())} of {best_greedy.size} points",
    "slowdown at max delay (lat=bw=4 T_F)": {n: round(float(cm[-1, -1, c]) / ref, 4) if cm[-1, -1, c] >= 0 else None
                                             for c, n in enumerate(names)},
    "slowdown latency only (lat=4 T_F, bw=0)": {n: round(float(cm[-1, 0, c]) / ref, 4) if cm[-1, 0, c] >= 0 else None
                                                for c, n in enumerate(names)},
    "slowdown bandwidth only (lat=0, bw=4 T_F)": {n: round(float(cm[0, -1, c]) / ref, 4) if cm[0, -1, c] >= 0 else None
                                                  for c, n in enumerate(names)},
}
# oracle spot check of 24 points
from oracle import oracle as O
O.build()
G, keep = O.to_or_grid(grid)
rng = np.random.default_rng(7)
flat = cm.reshape(-1, 6)
checked = 0
for k in rng.choice(grid.n_points, 24, replace=False):
    key, cms = O.sweep_point(grid, int(k), G=G)
    assert list(flat[k]) == cms, (k, list(flat[k]), cms)
    checked += 1
doc = {"workload": "E1: p=4, 2 DCs (2+2), m=8, F=D=W=T_F=38000 ticks, M_L = 1F1B budget, zero DP",
       "axes": {"T_lat/T_F": ratios, "T_bw/T_F": ratios}, "candidates": names,
       "slowdown_vs_zbh1_zero_delay": table, "summary": summary, "oracle_spot_checked_points": checked}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(doc, f)
print(json.dumps(summary, indent=1))
