"""E3 (§5.3 "Further Bubble Reduction" :620-692, Tables tab:extra_gbs_mem and tab:4dc) at the
model level: runtime per microbatch of 1F1B, ZB-H1, ZBV (static) and the greedy CrossUDSub (best of
n_sub 1/2/4) for the M70 setup (n_PP = 8, T_F = 0.038 s; D = W = T_F), 2 DCs (4 + 4
stages) and 4 DCs (2 stages each), at (T_lat/T_F, T_bw/T_F) in {(0,0), (0.25,0.25), (0.25,2), (2,0.25),
(2,2)}, for the paper's three cases:
  Case 1: GBS = m = 16, memory budget 1.0x (1F1B), no recomputation;
  Case 2: m = 32, budget 1.0x, layer-wise recomputation (reading Q37: every D first recomputes the
          stage's forward, t_d' = t_d + t_f, and only layer inputs stay resident, 1/10 of the full
          activation for 10 layers per stage, so the 1.0x budget holds 10x the microbatches);
  Case 3: m = 32, budget 2.0x, no recomputation.
The paper's numbers are GH200 measurements (context, not a target); the model-level
table checks its qualitative claims (:686-689).  CrossUD / CrossWave are solver schedules (out of
reach at p = 8, m >= 16) and are not reproduced.  usage: python tools/e3_table.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_00217_b200 as cp
from workloads import configs as K
from workloads.core import InstanceBatch

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/e3_gbs_memory_r01.json"
TF = K.T_F                                   # 38,000 ticks of 1 us = 0.038 s
P = 8
DELAYS = [(0, 0), (0.25, 0.25), (0.25, 2), (2, 0.25), (2, 2)]
CASES = {1: dict(m=16, budget=1000, recompute=False), 2: dict(m=32, budget=1000, recompute=True),
         3: dict(m=32, budget=2000, recompute=False)}
PAPER = {  # Table tab:extra_gbs_mem (2 DCs) and tab:4dc, s per microbatch: 1F1B, ZBH1, ZBV, UDSub (None: '-')
    2: {(0, 0): {1: (0.151, 0.133, 0.118, 0.137), 2: (0.174, 0.168, 0.161, None), 3: (None, None, None, 0.121)},
        (0.25, 0.25): {1: (0.168, 0.15, 0.148, 0.149), 2: (0.193, 0.187, 0.177, None), 3: (None, None, None, 0.123)},
        (0.25, 2): {1: (0.241, 0.23, 0.315, 0.181), 2: (0.262, 0.259, 0.33, None), 3: (None, None, None, 0.144)},
        (2, 0.25): {1: (0.242, 0.229, 0.314, 0.16), 2: (0.262, 0.258, 0.329, None), 3: (None, None, None, 0.127)},
        (2, 2): {1: (0.321, 0.309, 0.473, 0.198), 2: (0.333, 0.331, 0.476, None), 3: (None, None, None, 0.145)}},
    4: {(0, 0): {1: (0.149, 0.133, 0.119, 0.138), 2: (0.173, 0.168, 0.16, None), 3: (None, None, None, 0.123)},
        (0.25, 0.25): {1: (0.177, 0.158, 0.161, 0.155), 2: (0.198, 0.19, 0.181, None), 3: (None, None, None, 0.126)},
        (0.25, 2): {1: (0.269, 0.249, 0.339, 0.216), 2: (0.274, 0.269, 0.331, None), 3: (None, None, None, 0.158)},
        (2, 0.25): {1: (0.268, 0.248, 0.337, 0.2), 2: (0.274, 0.269, 0.33, None), 3: (None, None, None, 0.138)},
        (2, 2): {1: (0.359, 0.338, 0.512, 0.268), 2: (0.349, 0.346, 0.479, None), 3: (None, None, None, 0.178)}}}


def ud(ndc, m, a, b, case, n_sub=1):
    c = CASES[case]
    td = TF + (TF if c["recompute"] else 0)
    x = 10 * c["budget"] if c["recompute"] else c["budget"]
    return K.uniform_instance(P, m, ndc, TF, td, TF, lat=int(a * TF), bw=int(b * TF), mlim_x1000=x, n_sub=n_sub)


def wave(ndc, m, a, b, case):
    c = CASES[case]
    h = TF // 2
    td = h + (h if c["recompute"] else 0)
    x = 2 * (10 * c["budget"] if c["recompute"] else c["budget"])
    return K.uniform_instance(P, m, ndc, h, td, h, m_f=1, m_d=0, m_w=-1, lat=int(a * TF), bw=int(b * TF), mlim_x1000=x)


table, checks = {}, {}
from oracle import oracle as O
O.build()
for ndc in (2, 4):
    rows = []
    for (a, b) in DELAYS:
        for case, c in CASES.items():
            m = c["m"]
            base = InstanceBatch.concat([ud(ndc, m, a, b, case)])
            inst = cp.Instances(base)
            res = {}
            for kind in ("1f1b", "zbh1"):
                o, l_ = cp.build_static(kind, inst)
                res[kind] = int(cp.simulate(inst, o, l_)["makespan"][0])
            vi = cp.Instances(wave(ndc, m, a, b, case))
            vo, vl = cp.build_static("zbv", vi)
            res["zbv"] = int(cp.simulate(vi, vo, vl, wave=True)["makespan"][0])
            g = [int(cp.greedy(cp.Instances(ud(ndc, m, a, b, case, ns)))["makespan"][0]) for ns in (1, 2, 4)]
            res["udsub"] = min(g)
            # oracle spot check of this cell
            d = ud(ndc, m, a, b, case).item(0)
            assert res["1f1b"] == O.simulate(d, *O.build_static("1f1b", P, m))["makespan"]
            assert res["zbv"] == O.simulate_wave(wave(ndc, m, a, b, case).item(0), *O.build_static("zbv", P, m))["makespan"]
            assert g[0] == O.greedy(d)["makespan"]
            per_mb = {k: round(v * 1e-6 / m, 4) for k, v in res.items()}
            rows.append({"T_lat/T_F": a, "T_bw/T_F": b, "case": case, "model_s_per_mb": per_mb,
                         "paper_s_per_mb": dict(zip(("1f1b", "zbh1", "zbv", "udsub"), PAPER[ndc][(a, b)][case]))})
    table[f"{ndc}dc"] = rows
    R = {(r["T_lat/T_F"], r["T_bw/T_F"], r["case"]): r["model_s_per_mb"] for r in rows}
    checks[f"{ndc}dc"] = {
        "zero delay, case 1: ZBV best static (paper: bold ZBV)": R[0, 0, 1]["zbv"] < min(R[0, 0, 1]["1f1b"], R[0, 0, 1]["zbh1"]),
        "cells (of 15) where UDSub <= 1F1B": sum(R[a, b, c]["udsub"] <= R[a, b, c]["1f1b"] for (a, b) in DELAYS for c in CASES),
        "cells (of 15) where UDSub <= ZB-H1": sum(R[a, b, c]["udsub"] <= R[a, b, c]["zbh1"] for (a, b) in DELAYS for c in CASES),
        "delayed points where UDSub < ZB-H1 strictly (case 1)": sum(
            R[a, b, 1]["udsub"] < R[a, b, 1]["zbh1"] for (a, b) in DELAYS if (a, b) != (0, 0)),
        "every point: case 3 (2x memory, GBS 32) UDSub < case 1 UDSub": all(
            R[a, b, 3]["udsub"] < R[a, b, 1]["udsub"] for (a, b) in DELAYS),
        "UDSub gain case 1 -> 3 at (2, 2) (paper: up to 1.33x for CrossUD)": round(R[2, 2, 1]["udsub"] / R[2, 2, 3]["udsub"], 3),
        "bandwidth vs latency, case 1 UDSub (0.25, 2) / (2, 0.25) (paper 2DC 1.13, 4DC 1.08)":
            round(R[0.25, 2, 1]["udsub"] / R[2, 0.25, 1]["udsub"], 3),
        "ZBV degrades most under delay (paper: ZBV 0.473 at (2,2), 2DC)": R[2, 2, 1]["zbv"] > max(R[2, 2, 1]["1f1b"], R[2, 2, 1]["zbh1"]),
        "recomputation (case 2) slower than case 1 for static 1F1B at zero delay": R[0, 0, 2]["1f1b"] > R[0, 0, 1]["1f1b"],
    }
doc = {"workload": "E3 model level: M70 (T_F = 0.038 s), n_PP = 8, D = W = T_F, 2 DCs (4+4) and 4 DCs (2 each); "
                   "cases 1-3 of PAPER.md :625-628; reading Q37 for recomputation",
       "table": table, "checks": checks}
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(doc, f)
for ndc in (2, 4):
    print(f"--- {ndc} DCs  (model | paper), s per microbatch: 1F1B ZBH1 ZBV UDSub")
    for r in table[f"{ndc}dc"]:
        mm, pp = r["model_s_per_mb"], r["paper_s_per_mb"]
        print(r["T_lat/T_F"], r["T_bw/T_F"], r["case"], [mm[k] for k in ("1f1b", "zbh1", "zbv", "udsub")], [pp[k] for k in ("1f1b", "zbh1", "zbv", "udsub")])
print(json.dumps(checks, indent=1))
