"""Pins of the oracle's branch and bound (oracle/bnb.c) against things other
than itself: exhaustive enumeration and Python brute force on small instances (SPEC.md:547
acceptance 4), the optimality sandwich against every static and greedy plan (reading
Q25), the zero-delay closed form (3m + p - 1)·f (Z6, a lower bound by counting), random valid plans
on the paper's 4 x 8 E1 setup, and the B&B with its dominance cut or its
Jackson bound switched off (independent cut logic, same optimum).  Runs without a GPU.
"""
import json
import os

import numpy as np
import pytest

from tests.helpers_independent import brute_force_opt, random_valid_plan
from workloads import configs as K

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _small(n, seed, max_p, max_m):
    b = K.random_instances(n, seed=seed, max_p=max_p, max_m=max_m, intra_delay=True)
    out = []
    for i in range(len(b)):
        d = b.item(i)
        d["n_sub"] = 1
        out.append(d)
    return out


def test_bnb_equals_exhaustive_enumeration(oracle_lib):
    """SPEC.md:547 acceptance 4: on randomized instances (DP tails, ZeRO-1, per-stage costs, intra-
    and cross-DC delays, memory budgets) the B&B optimum equals exhaustive enumeration exactly, and
    the search finishes (proven)."""
    n_cmp = 0
    for d in _small(400, 31, 4, 4):
        if oracle_lib.validate_instance(d):
            continue
        e = oracle_lib.enumerate_opt(d, max_plans=400_000)
        if e["evaluated"] < 0:
            continue
        r = oracle_lib.bnb_opt(d)
        assert r["rc"] == 1 and r["proven"], d
        assert r["makespan"] == e["makespan"], (d, r["makespan"], e["makespan"])
        assert r["bound"] == r["makespan"]
        n_cmp += 1
    assert n_cmp >= 150


def test_bnb_equals_python_brute_force_up_to_14_ops(oracle_lib):
    """<= 14 compute ops, against brute force over every per-stage permutation
    (tests/helpers_independent.py, the fixed-point formulation, no oracle code)."""
    n = 0
    for d in _small(120, 37, 2, 2):
        if oracle_lib.validate_instance(d) or 3 * d["p"] * d["m"] > 14:
            continue
        assert oracle_lib.bnb_opt(d)["makespan"] == brute_force_opt(d), d
        n += 1
    assert n >= 40


def test_bnb_sandwich(oracle_lib):
    """Optimality sandwich (Q25): exact <= greedy (n_sub = 1, same plan space and
    budget), exact <= ZB-H1 and exact <= 1F1B (their split realisations are in the plan set)."""
    for d in _small(200, 41, 4, 5):
        if oracle_lib.validate_instance(d):
            continue
        r = oracle_lib.bnb_opt(d, max_nodes=2_000_000)
        if not r["proven"]:
            continue
        assert r["makespan"] <= oracle_lib.greedy(d)["makespan"]
        for kind in ("zbh1", "1f1b"):
            c, ln = oracle_lib.build_static(kind, d["p"], d["m"])
            w = oracle_lib.simulate(d, c, ln)
            if w["status"] == 0:
                assert r["makespan"] <= w["makespan"], kind


@pytest.mark.parametrize("p,m", [(2, 2), (2, 5), (3, 3), (3, 6), (4, 4), (4, 8)])
def test_bnb_zero_delay_closed_form(oracle_lib, p, m):
    """Z6: uniform f = t_d = t_w, no delays, 1F1B budget p·m_f, m >= p.  The last stage cannot start
    before (p - 1)·f and then runs 3m blocks, so (3m + p - 1)·f is a lower bound of every plan; the
    B&B must reach exactly it (the greedy does)."""
    d = K.uniform_instance(p, m, 2, 100, 100, 100, mlim_x1000=1000).item(0)
    r = oracle_lib.bnb_opt(d)
    assert r["proven"] and r["makespan"] == (3 * m + p - 1) * 100


@pytest.mark.parametrize("p,m,lat,bw", [(3, 4, 100, 50), (4, 3, 60, 150), (3, 5, 200, 200)])
def test_bnb_without_dominance_or_jacks_bound_agrees(oracle_lib, p, m, lat, bw):
    """The same optimum with the dominance cut off, and with the Jackson bound replaced by the
    per-block head + duration + tail bound: a wrong dominance vector or an invalid (too strong)
    bound would cut the optimum in one search but not the other."""
    d = K.uniform_instance(p, m, 2, 100, 90, 70, lat=lat, bw=bw, mlim_x1000=1000).item(0)
    full = oracle_lib.bnb_opt(d)
    nojps = oracle_lib.bnb_opt(d, flags=oracle_lib.BNB_NO_JPS)
    assert full["proven"] and nojps["proven"]
    assert full["makespan"] == nojps["makespan"]
    if p * m <= 12:
        nodom = oracle_lib.bnb_opt(d, flags=oracle_lib.BNB_NO_DOMINANCE, max_nodes=40_000_000)
        assert nodom["proven"] and nodom["makespan"] == full["makespan"]


def test_bnb_tiny_grid_e1_setup(oracle_lib):
    """Config 1 / E1 setup (4 stages, 2 DCs, 8 microbatches, uniform costs, 1F1B
    memory budget) at all 16 points of {0, .5, 1, 2}^2: proven optimum; its plan re-simulates to it;
    it is <= the greedy, ZB-H1 and 200 random valid plans per point; and SPEC.md:548 acceptance 5(d),
    CrossUDSub (best greedy of n_sub 1/2/4) within 5% of the exact CrossUD on >= 80% of points.
    The table tests/golden/bnb_tiny_grid.json is written by tools/bnb_tiny_table.py (oracle only)."""
    gold = json.load(open(os.path.join(GOLD, "bnb_tiny_grid.json")))["points"]
    within5 = 0
    rng = np.random.default_rng(5)
    for row in gold:
        a, b = row["lat_ratio"], row["bw_ratio"]
        d = K.tiny(a, b).item(0)
        r = oracle_lib.bnb_opt(d)
        assert r["proven"] and r["makespan"] == row["optimum"], (a, b)
        assert oracle_lib.simulate(d, r["codes"], r["len"])["makespan"] == r["makespan"]
        assert oracle_lib.check_plan(d, r["codes"], r["len"]) == 0
        g = oracle_lib.greedy(d)["makespan"]
        assert r["makespan"] <= g == row["greedy_nsub1"]
        c, ln = oracle_lib.build_static("zbh1", 4, 8)
        assert r["makespan"] <= oracle_lib.simulate(d, c, ln)["makespan"]
        for _ in range(200):
            assert r["makespan"] <= oracle_lib.simulate(d, random_valid_plan(d, rng))["makespan"]
        ud_sub = min(oracle_lib.greedy(dict(d, n_sub=k))["makespan"] for k in (1, 2, 4))
        assert ud_sub == row["crossudsub"]
        within5 += ud_sub <= 1.05 * r["makespan"]
    assert len(gold) == 16 and within5 >= 13            # >= 80% of 16 points
