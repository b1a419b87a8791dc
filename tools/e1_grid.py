"""E1 delay-sensitivity table (§5.1, Fig. pre_delay_sensitivity) on the GPU sweep:
4 stages / 2 DCs / 8 microbatches, T_lat/T_F x T_bw/T_F grid, candidates GPipe, 1F1B, greedy
n_sub 1/2/4 (CrossUDSub), ZB-H1 (sweep), and the two-chunk static schedules ZBV (Wave, reading Q35)
and IV1F1B (Loop, Q34).  Slowdown is relative to ZBV at zero delay, as in the paper (PAPER.md :486,
:491).  Spot-checks points against the oracle.
usage: python tools/e1_grid.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from workloads import configs as K

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/e1_delay_sensitivity_r02.json"
grid = K.e1_grid()
keys, cm = cp.sweep_shard(grid, cand=True)
torch.cuda.synchronize()
cm = cm.cpu().numpy().reshape(len(grid.lat), len(grid.bw), 6)       # point = i_lat * n_bw + i_bw
names = ["GPipe", "1F1B", "CrossUDSub n_sub=1", "CrossUDSub n_sub=2", "CrossUDSub n_sub=4", "ZB-H1"]
# IV1F1B (Loop pattern, reading Q33/Q34) on the same points.  Interleaving splits each stage's layers
# into two chunks, so a chunk block costs T_F/2 (the same model and the same activation messages);
# the wrap link (stage 3 in the second DC back to stage 0) crosses DCs and carries the point's
# (latency, T_bw) like the inner boundary
from workloads.core import InstanceBatch
parts, vparts = [], []
for li in grid.lat:
    for bi in grid.bw:
        b = K.uniform_instance(4, 8, 2, K.T_F // 2, K.T_F // 2, K.T_F // 2, m_f=1, m_d=-1, m_w=0,
                               lat=int(li), bw=int(bi))
        b.lat_f[0, 3], b.bw_f[0, 3], b.lat_b[0, 3], b.bw_b[0, 3] = int(li), int(bi), int(li), int(bi)
        parts.append(b)
        # ZBV (Wave, Q32/Q35): the same half-cost chunks with split W (activation freed by W); budget 2p
        # chunk activations = the 1F1B budget of p full-stage activations; the V never wraps
        vparts.append(K.uniform_instance(4, 8, 2, K.T_F // 2, K.T_F // 2, K.T_F // 2, m_f=1, m_d=0, m_w=-1,
                                         mlim_x1000=2000, lat=int(li), bw=int(bi)))
ib = InstanceBatch.concat(parts)
vb = InstanceBatch.concat(vparts)
vinst = cp.Instances(vb)
vops, vln = cp.build_static("zbv", vinst, stage_stride=4)
vr = cp.simulate(vinst, vops, vln, wave=True)
iinst = cp.Instances(ib)
io = torch.arange(len(ib), dtype=torch.int32, device="cuda")
iops, iln = cp.build_static("iv1f1b", iinst, stage_stride=4)
ir = cp.simulate(iinst, iops, iln, loop=True)
torch.cuda.synchronize()
iv = ir["makespan"].cpu().numpy().reshape(len(grid.lat), len(grid.bw))
ivst = ir["status"].cpu().numpy()
zv = vr["makespan"].cpu().numpy().reshape(len(grid.lat), len(grid.bw))
assert (vr["status"].cpu().numpy() == 0).all()
ref = float(zv[0, 0])
ratios = (np.asarray(grid.lat) / K.T_F).round(4).tolist()
table = {names[c]: (np.where(cm[:, :, c] >= 0, cm[:, :, c] / ref, np.nan)).round(4).tolist() for c in range(6)}
g = {n: cm[:, :, c] for c, n in enumerate(names)}
best_greedy = np.min(np.stack([g[n] for n in names[2:5]]), axis=0)
summary = {
    "reference": "ZBV at zero delay = %d ticks" % ref,
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
table["IV1F1B (Loop)"] = (iv / ref).round(4).tolist()
g["IV1F1B (Loop)"] = iv
summary["IV1F1B (Loop) status"] = ("memory above the 1F1B budget at every point: reported regardless, as the paper "
                                   "evaluates static schedules" if (ivst == 2).all() else str(sorted(set(ivst.tolist()))))
for key, (a, b_) in {"slowdown at max delay (lat=bw=4 T_F)": (-1, -1), "slowdown latency only (lat=4 T_F, bw=0)": (-1, 0),
                     "slowdown bandwidth only (lat=0, bw=4 T_F)": (0, -1)}.items():
    summary[key]["IV1F1B (Loop)"] = round(float(iv[a, b_]) / ref, 4)
summary["IV1F1B at zero delay vs ZBV"] = round(float(iv[0, 0]) / ref, 4)
table["ZBV (Wave)"] = (zv / ref).round(4).tolist()
g["ZBV (Wave)"] = zv
for key, (a, b_) in {"slowdown at max delay (lat=bw=4 T_F)": (-1, -1), "slowdown latency only (lat=4 T_F, bw=0)": (-1, 0),
                     "slowdown bandwidth only (lat=0, bw=4 T_F)": (0, -1)}.items():
    summary[key]["ZBV (Wave)"] = round(float(zv[a, b_]) / ref, 4)
best_ud = np.min(np.stack([g[n] for n in ("1F1B", "ZB-H1")]), axis=0)
summary["Wave better at low delay, UD as delays grow (PAPER.md:495)"] = {
    "ZBV < best static UD at zero delay": bool(zv[0, 0] < best_ud[0, 0]),
    "best static UD < ZBV at max delay": bool(best_ud[-1, -1] < zv[-1, -1]),
    "points where ZBV < best static UD": int((zv < best_ud).sum())}
summary["WGrad-split beats unified (PAPER.md:494)"] = {
    "ZB-H1 <= 1F1B": f"{int((g['ZB-H1'] <= g['1F1B']).sum())} of {zv.size} points",
    "ZBV <= IV1F1B": f"{int((zv <= iv).sum())} of {zv.size} points"}
summary["Loop vs Wave (PAPER.md:496 'Loop schedules show the highest sensitivity')"] = {
    "IV1F1B slower than ZBV at": f"{int((iv > zv).sum())} of {zv.size} points",
    "on the latency-only axis": f"{int((iv[:, 0] > zv[:, 0]).sum())} of {len(grid.lat)}",
    "on the bandwidth-only axis": f"{int((iv[0, :] > zv[0, :]).sum())} of {len(grid.bw)}",
    "growth over own zero delay at max delay": {"IV1F1B": round(float(iv[-1, -1] / iv[0, 0]), 4),
                                                "ZBV": round(float(zv[-1, -1] / zv[0, 0]), 4),
                                                "ZB-H1": round(float(g["ZB-H1"][-1, -1] / g["ZB-H1"][0, 0]), 4),
                                                "1F1B": round(float(g["1F1B"][-1, -1] / g["1F1B"][0, 0]), 4)}}
# oracle spot check of 24 points (and of IV1F1B at 6 points)
from oracle import oracle as O
O.build()
ci, li_ = O.build_static("iv1f1b", 4, 8)
cv, lv = O.build_static("zbv", 4, 8)
for k in np.random.default_rng(8).choice(len(ib), 6, replace=False):
    w = O.simulate_loop(ib.item(int(k)), ci, li_)
    assert int(ir["makespan"][int(k)]) == w["makespan"], (k, int(ir["makespan"][int(k)]), w["makespan"])
    w = O.simulate_wave(vb.item(int(k)), cv, lv)
    assert int(vr["makespan"][int(k)]) == w["makespan"], (k, int(vr["makespan"][int(k)]), w["makespan"])
G, keep = O.to_or_grid(grid)
rng = np.random.default_rng(7)
flat = cm.reshape(-1, 6)
checked = 0
for k in rng.choice(grid.n_points, 24, replace=False):
    key, cms = O.sweep_point(grid, int(k), G=G)
    assert list(flat[k]) == cms, (k, list(flat[k]), cms)
    checked += 1
doc = {"workload": "E1: p=4, 2 DCs (2+2), m=8, F=D=W=T_F=38000 ticks, M_L = 1F1B budget, zero DP",
       "axes": {"T_lat/T_F": ratios, "T_bw/T_F": ratios}, "candidates": names + ["IV1F1B (Loop)", "ZBV (Wave)"],
       "slowdown_vs_zbv_zero_delay": table, "summary": summary, "oracle_spot_checked_points": checked,
       "zbv_note": "ZBV = reading Q35's stand-in: unit-time list schedule of the Wave data flow with ZB-V's "
                   "published properties (zero bubble at zero delay, 2p chunk activations), not Qi et al.'s exact "
                   "block order; every slowdown here is normalised to it and its delayed column inherits that choice"}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(doc, f)
print(json.dumps(summary, indent=1))
