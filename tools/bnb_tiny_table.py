#!/usr/bin/env python3
"""Writes tests/golden/bnb_tiny_grid.json: the exact optimum (oracle branch and bound, oracle/bnb.c)
of BASELINE config 1 / the paper's E1 setup (4 stages over 2 DCs, 8
microbatches, uniform T_F = T_D = T_W = 100 ticks, 1F1B memory budget) at the 16 points of
(T_lat/T_F, T_bw/T_F) in {0, .5, 1, 2}^2, beside the greedy CrossUD (n_sub = 1) and CrossUDSub
(best of n_sub 1/2/4).  Calls only oracle/ (a stored value written by a committed oracle script)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from workloads import configs as K  # noqa: E402


def main():
    rows = []
    for a in (0, 0.5, 1, 2):
        for b in (0, 0.5, 1, 2):
            d = K.tiny(a, b).item(0)
            t = time.time()
            r = O.bnb_opt(d)
            assert r["proven"], (a, b)
            sub = {k: O.greedy(dict(d, n_sub=k))["makespan"] for k in (1, 2, 4)}
            rows.append({"lat_ratio": a, "bw_ratio": b, "optimum": r["makespan"], "greedy_nsub1": sub[1],
                         "crossudsub": min(sub.values()), "greedy_by_nsub": sub, "root_bound": r["root_bound"],
                         "nodes": r["nodes"], "seconds": round(time.time() - t, 2)})
            print(rows[-1], flush=True)
    out = {"source": "tools/bnb_tiny_table.py (oracle/bnb.c branch and bound, oracle/oracle.c greedy)",
           "setup": "p=4, 2 DCs, m=8, T_F=T_D=T_W=100 ticks, m_f=2, m_lim=8 (1F1B budget), n_sub=1 plans",
           "points": rows}
    with open(os.path.join(ROOT, "tests", "golden", "bnb_tiny_grid.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
