"""Pins of the CPU oracle against things other than itself (runs without a GPU).

Each test names the passage / closed form / brute force it pins.  A plausible
mistake in the oracle (dropped term, wrong sign/index, transposed operand, wrong
link direction, wrong memory timing) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

from tests.helpers_independent import B, D, F, W, brute_force_opt, bubble, fp_simulate, random_valid_plan
from workloads import configs as K

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def inst(p, m, n_dc, f, d, w, **kw):
    return K.uniform_instance(p, m, n_dc, f, d, w, **kw).item(0)


# --------------------------------------------------------------------------- SPEC worked examples
def test_spec_simulate_p2_m1(oracle_lib):
    g = gold("spec_examples.json")["simulate_p2_m1_unit"]
    d = inst(2, 1, 1, 1, 1, 1, m_f=1, m_d=0, m_w=-1)
    r = oracle_lib.simulate(d, g["plan"])
    assert r["status"] == 0 and r["makespan"] == g["makespan"]


def test_spec_1f1b_p4_m8_and_bubble(oracle_lib):
    g = gold("spec_examples.json")["simulate_1f1b_p4_m8"]
    d = inst(4, 8, 1, 1, 1, 1)
    r = oracle_lib.simulate(d, *oracle_lib.build_static("1f1b", 4, 8))
    assert r["makespan"] == g["makespan"]
    loc, glo = bubble(r["first_start"][0], r["last_end"][0], r["busy"][0], r["makespan"])
    assert abs(loc - g["stage0_bubble_num"] / g["stage0_bubble_den"]) < 1e-9
    assert abs(glo - g["stage0_bubble_num"] / g["stage0_bubble_den"]) < 1e-9


def test_spec_greedy_p2_m1(oracle_lib):
    g = gold("spec_examples.json")["greedy_p2_m1_unit"]
    d = inst(2, 1, 1, 1, 1, 1, m_f=1, m_d=0, m_w=-1)
    assert oracle_lib.greedy(d)["makespan"] == g["makespan"]


def test_reserve_window_spec(oracle_lib):
    for c in gold("spec_examples.json")["reserve_window"]["cases"]:
        assert list(oracle_lib.reserve_window(c["intervals"], c["t_ready"], c["width"])) == c["window"]


def test_reserve_window_vs_exhaustive_gap_scan(oracle_lib):
    """first-fit equals an exhaustive scan on 1000 random interval sets."""
    rng = np.random.default_rng(1)
    for _ in range(1000):
        k = int(rng.integers(0, 8))
        pts = np.sort(rng.choice(200, size=2 * k, replace=False))
        ivs = [(int(pts[2 * i]), int(pts[2 * i + 1])) for i in range(k)]
        t, w = int(rng.integers(0, 200)), int(rng.integers(1, 30))
        x = t
        while any(not (x + w <= a or x >= b) for a, b in ivs):
            x += 1
        assert oracle_lib.reserve_window(ivs, t, w) == (x, x + w)


def test_two_simultaneous_messages_serialize(oracle_lib):
    """SPEC.md:551 / fig:comm_model: second ends at first_end + width."""
    assert oracle_lib.reserve_window([(3, 10)], 3, 7) == (10, 17)


# --------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("kind", ["1f1b", "gpipe"])
def test_Z1_zero_delay(oracle_lib, kind):
    """Z1: (m + p - 1)(f + b) at zero delay, including m < p (reading Q23)."""
    rng = np.random.default_rng(2)
    for _ in range(60):
        p, m = int(rng.integers(1, 12)), int(rng.integers(1, 20))
        f, dd, w = (int(x) for x in rng.integers(1, 50, size=3))
        d = inst(p, m, 2, f, dd, w, mlim_x1000=10**6)
        r = oracle_lib.simulate(d, *oracle_lib.build_static(kind, p, m))
        assert r["makespan"] == (m + p - 1) * (f + dd + w)


def test_Z2_gpipe_with_delays(oracle_lib):
    """Z2: p(f+b) + k(T_f+L_f+T_b+L_b) + (m-1)(max(f,T_f) + max(b,T_b)), k >= 1 boundaries."""
    rng = np.random.default_rng(3)
    for _ in range(80):
        n_dc = int(rng.integers(2, 5))
        p = int(rng.integers(n_dc, 12))
        m = int(rng.integers(1, 16))
        f, dd, w = (int(x) for x in rng.integers(1, 60, size=3))
        Lf, Tf, Lb, Tb = (int(x) for x in rng.integers(0, 120, size=4))
        d = inst(p, m, n_dc, f, dd, w, lat=Lf, bw=Tf, lat_b=Lb, bw_b=Tb, mlim_x1000=10**6)
        k = min(n_dc, p) - 1                     # contiguous even split: one boundary per DC pair
        b = dd + w
        want = p * (f + b) + k * (Tf + Lf + Tb + Lb) + (m - 1) * (max(f, Tf) + max(b, Tb))
        r = oracle_lib.simulate(d, *oracle_lib.build_static("gpipe", p, m))
        assert r["makespan"] == want, (p, m, n_dc, f, b, Lf, Tf, Lb, Tb)


def test_Z3_1f1b_two_stages(oracle_lib):
    """Z3: 1F1B, p=2, one boundary, T <= min(f,b), m >= 2: (m+1)(f+b) + 2*ceil(m/2)*(L+T)."""
    rng = np.random.default_rng(4)
    for _ in range(80):
        m = int(rng.integers(2, 30))
        f, dd, w = (int(x) for x in rng.integers(1, 60, size=3))
        b = dd + w
        L = int(rng.integers(0, 200))
        T = int(rng.integers(0, min(f, b) + 1))
        d = inst(2, m, 2, f, dd, w, lat=L, bw=T, mlim_x1000=10**6)
        r = oracle_lib.simulate(d, *oracle_lib.build_static("1f1b", 2, m))
        assert r["makespan"] == (m + 1) * (f + b) + 2 * math.ceil(m / 2) * (L + T)


def test_Z5_1f1b_peak_memory(oracle_lib):
    """Z5: 1F1B peak on stage s = min(p - s, m) * m_f."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        p, m = int(rng.integers(1, 16)), int(rng.integers(1, 20))
        mf = int(rng.integers(1, 5))
        md = -int(rng.integers(0, mf + 1))
        d = inst(p, m, 2, 3, 4, 5, m_f=mf, m_d=md, m_w=-mf - md, mlim_x1000=10**6)
        r = oracle_lib.simulate(d, *oracle_lib.build_static("1f1b", p, m))
        assert list(r["peak"]) == [min(p - s, m) * mf for s in range(p)]


def test_Z6_greedy_matches_zbh1_closed_form(oracle_lib):
    """Z6: greedy, zero delay, f=t_d=t_w, m_lim = p*m_f, m >= p: (3m + p - 1) f; this equals
    ZB-H1's m(f+d+w) + (p-1)(f+d-w) and backs PAPER.md:443 ("Equivalent performance to ZB-H1")."""
    rng = np.random.default_rng(6)
    for _ in range(60):
        p = int(rng.integers(1, 12))
        m = int(rng.integers(p, 3 * p + 1))
        f = int(rng.integers(4, 60))
        ns = int(rng.choice([1, 2, 4]))
        d = inst(p, m, 2, f, f, f, n_sub=ns)
        r = oracle_lib.greedy(d)
        assert r["status"] == 0 and r["makespan"] == (3 * m + p - 1) * f


# --------------------------------------------------------------------------- ZB-H1 (reading Q31)
def test_zbh1_closed_form_zero_delay(oracle_lib):
    """ZB-H1's published bubble (p-1)(T_F + T_B - T_W) (Qi et al. via PAPER.md :443,
    :472): makespan m(f+d+w) + (p-1)(f+d-w) at zero delay with uniform costs, m >= p and
    w <= min(f, d); every built plan is valid (Q29)."""
    rng = np.random.default_rng(31)
    for _ in range(120):
        p = int(rng.integers(1, 9))
        m = int(rng.integers(p, 3 * p + 2))
        d_, f = (int(x) for x in rng.integers(1, 200, size=2))
        w = int(rng.integers(1, min(f, d_) + 1))
        dd = inst(p, m, int(rng.integers(1, 5)), f, d_, w, mlim_x1000=1000)
        c, l_ = oracle_lib.build_static("zbh1", p, m)
        assert oracle_lib.check_plan(dd, c, l_) == 0
        r = oracle_lib.simulate(dd, c, l_)
        assert r["status"] == 0 and r["makespan"] == m * (f + d_ + w) + (p - 1) * (f + d_ - w), (p, m, f, d_, w)


def test_zbh1_peak_memory_and_budget(oracle_lib):
    """Q31 memory: with m >= p, stage s peaks at (p-s) m_f - s m_w, which never exceeds the 1F1B
    device budget p m_f (Q9; "unchanged peak activation memory")."""
    rng = np.random.default_rng(32)
    for _ in range(80):
        p = int(rng.integers(1, 9))
        m = int(rng.integers(p, 3 * p + 2))
        mf = int(rng.integers(1, 6))
        md = -int(rng.integers(0, mf + 1))
        mw = -mf - md
        dd = inst(p, m, 1, 7, 5, 3, m_f=mf, m_d=md, m_w=mw, mlim_x1000=1000)
        r = oracle_lib.simulate(dd, *oracle_lib.build_static("zbh1", p, m))
        assert list(r["peak"]) == [(p - s) * mf - s * mw for s in range(p)]
        assert max(r["peak"]) <= p * mf and r["status"] == 0


def test_zbh1_vs_1f1b_and_greedy_zero_delay(oracle_lib):
    """makespan(ZB-H1) <= makespan(1F1B) at zero delay, uniform, t_d = t_w; SPEC.md
    acceptance 3 / PAPER.md :443: the greedy with the 1F1B memory budget matches ZB-H1 (n_pp in
    {4, 8}, n_mb = 2 n_pp; exact here, Z6)."""
    for p in (4, 8):
        m = 2 * p
        for f, b in ((100, 100), (60, 100), (100, 40)):
            dd = inst(p, m, 2, f, b, b, mlim_x1000=1000)
            z = oracle_lib.simulate(dd, *oracle_lib.build_static("zbh1", p, m))["makespan"]
            one = oracle_lib.simulate(dd, *oracle_lib.build_static("1f1b", p, m))["makespan"]
            assert z <= one
        dd = inst(p, m, 2, 100, 100, 100, mlim_x1000=1000)
        z = oracle_lib.simulate(dd, *oracle_lib.build_static("zbh1", p, m))["makespan"]
        assert oracle_lib.greedy(dd)["makespan"] == z == (3 * m + p - 1) * 100


def test_dp_tail_and_zero1_shift(oracle_lib):
    """DP overlap: AR after the last W/B -> 1F1B zero delay ends at Z1 + T_dp;
    ZeRO-1 AG before the first F shifts everything by T_ag (uniform); zero volume = no change."""
    p, m, f, dd, w = 4, 8, 10, 7, 5
    Z1 = (m + p - 1) * (f + dd + w)
    c, ln = oracle_lib.build_static("1f1b", p, m)
    assert oracle_lib.simulate(inst(p, m, 1, f, dd, w, t_dp=0), c, ln)["makespan"] == Z1
    assert oracle_lib.simulate(inst(p, m, 1, f, dd, w, t_dp=37), c, ln)["makespan"] == Z1 + 37
    assert oracle_lib.simulate(inst(p, m, 1, f, dd, w, zero1=1, t_ag=11), c, ln)["makespan"] == Z1 + 11


def test_appendix_c_bubble_strides(oracle_lib):
    """App. C + SPEC.md:479: 1F1B delay accumulates (> 1.5 T_F extra), zero-delay = Z1."""
    g = gold("spec_examples.json")["appendix_c_bubble_strides"]
    p, m, TF = g["p"], g["m"], g["T_F"]
    c, ln = oracle_lib.build_static("1f1b", p, m)
    r0 = oracle_lib.simulate(inst(p, m, 2, TF, TF, TF, mlim_x1000=1000), c, ln)
    r1 = oracle_lib.simulate(inst(p, m, 2, TF, TF, TF, lat=g["lat"], mlim_x1000=1000), c, ln)
    assert r0["makespan"] == (m + p - 1) * 3 * TF
    assert r1["makespan"] - r0["makespan"] > 1.5 * TF
    # SPEC.md:550 "critical-path crossing count >= 2": the makespan is piecewise linear in the boundary
    # latency with slope = the number of DC-boundary crossings on the critical path (one tick apart)
    r2 = oracle_lib.simulate(inst(p, m, 2, TF, TF, TF, lat=g["lat"] + 1, mlim_x1000=1000), c, ln)
    assert r2["makespan"] - r1["makespan"] >= 2
    gr0 = oracle_lib.greedy(inst(p, m, 2, TF, TF, TF))
    gr1 = oracle_lib.greedy(inst(p, m, 2, TF, TF, TF, lat=g["lat"]))
    assert gr0["makespan"] == (3 * m + p - 1) * TF                  # Z6
    assert gr1["makespan"] - gr0["makespan"] < r1["makespan"] - r0["makespan"]
    reg = gold("survey_check_tiny.json")["appendix_c"]                # regression (survey check)
    assert (r0["makespan"], r1["makespan"], gr0["makespan"], gr1["makespan"]) == (
        reg["1f1b_zero"], reg["1f1b_lat"], reg["greedy1_zero"], reg["greedy1_lat"])


def test_Z7_monotone_and_convex_in_latency(oracle_lib):
    """Z7 + SPEC.md:289: fixed-plan makespan is non-decreasing in every lat/bw entry and
    convex piecewise-linear with integer slopes in a uniform boundary latency."""
    rng = np.random.default_rng(7)
    for _ in range(25):
        d = K.random_instances(1, seed=int(rng.integers(1 << 30)), max_p=6, max_m=6).item(0)
        if d["p"] < 2:
            continue
        codes = random_valid_plan(d, rng)
        base = oracle_lib.simulate(d, codes)["makespan"]
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            e = dict(d)
            e[fld] = d[fld].copy()
            e[fld][int(rng.integers(d["p"] - 1))] += int(rng.integers(1, 50))
            assert oracle_lib.simulate(e, codes)["makespan"] >= base
        vals = []
        for L in range(0, 60, 3):
            e = dict(d)
            e["lat_f"] = np.full(d["p"] - 1, L)
            e["lat_b"] = np.full(d["p"] - 1, L)
            vals.append(oracle_lib.simulate(e, codes)["makespan"])
        sec = np.diff(vals, 2)
        assert np.all(sec >= 0)


# --------------------------------------------------------------------------- independent formulation
def test_simulate_equals_fixed_point_formulation(oracle_lib):
    """SPEC.md:292 brute-force equivalence: the oracle's Kahn/first-fit evaluation equals the
    least fixed point of the §3.5 equations with FIFO links (App. X1 equivalence under UD)."""
    rng = np.random.default_rng(8)
    batch = K.random_instances(150, seed=9, max_p=6, max_m=6, intra_delay=True)
    for i in range(len(batch)):
        d = batch.item(i)
        codes = random_valid_plan(d, rng)
        r = oracle_lib.simulate(d, codes, timeline=True)
        fp = fp_simulate(d, codes)
        assert not fp["deadlock"]
        assert r["makespan"] == fp["makespan"]
        for s in range(d["p"]):
            assert list(r["t_start"][s, :len(codes[s])]) == fp["start"][s]


def test_deadlock_matches_fixed_point_divergence(oracle_lib):
    """Plans with swapped entries: oracle DEADLOCK <=> the fixed-point iteration diverges."""
    rng = np.random.default_rng(10)
    batch = K.random_instances(80, seed=11, max_p=5, max_m=5)
    seen = deadlocks = 0
    for i in range(len(batch)):
        d = batch.item(i)
        d["m_lim"] = d["m_lim"] * 100
        codes = random_valid_plan(d, rng)
        s = int(rng.integers(d["p"]))
        if len(codes[s]) < 2:
            continue
        k = int(rng.integers(len(codes[s]) - 1))
        codes[s][k], codes[s][k + 1] = codes[s][k + 1], codes[s][k]
        st = oracle_lib.check_plan(d, codes)
        r = oracle_lib.simulate(d, codes)
        if st:
            assert r["status"] == st
            continue
        fp = fp_simulate(d, codes)
        assert (r["status"] & 1 == 1) == fp["deadlock"]
        deadlocks += fp["deadlock"]
        if not fp["deadlock"]:
            assert r["makespan"] == fp["makespan"]
        seen += 1
    assert seen > 20 and deadlocks >= 3


def test_bad_plan_rules(oracle_lib):
    """Reading Q29: counts, W prefix, B mixed with D/W."""
    d = inst(2, 2, 1, 1, 1, 1)
    good = [[0, 0, 2, 3, 2, 3], [0, 2, 3, 0, 2, 3]]
    assert oracle_lib.check_plan(d, good) == 0
    assert oracle_lib.check_plan(d, [[0, 0, 3, 2, 2, 3], good[1]]) == 4     # W before its D
    assert oracle_lib.check_plan(d, [[0, 0, 2, 2, 3], good[1]]) == 4        # missing W
    assert oracle_lib.check_plan(d, [[0, 0, 0, 2, 3, 2, 3], good[1]]) == 4  # extra F
    assert oracle_lib.check_plan(d, [[0, 0, 1, 2, 3], good[1]]) == 4        # B mixed with D/W
    assert oracle_lib.check_plan(d, [[0, 0, 1, 1], [0, 1, 0, 1]]) == 0      # all combined


# --------------------------------------------------------------------------- greedy properties
def test_greedy_properties(oracle_lib):
    """Alg. 1 pins: iteration count 3*n_mb*n_sub*n_PP; re-simulating the plan
    reproduces the greedy timeline; peak <= M_L; determinism."""
    batch = K.random_instances(200, seed=12, max_p=10, max_m=12)
    for i in range(len(batch)):
        d = batch.item(i)
        g = oracle_lib.greedy(d, timeline=True)
        assert g["status"] == 0
        assert g["iterations"] == 3 * d["m"] * d["n_sub"] * d["p"]
        assert np.all(g["peak"] <= d["m_lim"])
        r = oracle_lib.simulate(d, g["codes"], g["len"], timeline=True)
        assert r["status"] == 0 and r["makespan"] == g["makespan"]
        assert np.array_equal(r["t_start"], g["t_start"])
        fp = fp_simulate(d, [list(g["codes"][s, :g["len"][s]]) for s in range(d["p"])])
        assert fp["makespan"] == g["makespan"]
        g2 = oracle_lib.greedy(d)
        assert np.array_equal(g2["codes"], g["codes"])


def test_greedy_priority_examples(oracle_lib):
    """SPEC.md:348-350 select_op examples, observed on a 1-stage instance:
    warm-up prefers F; after an F the D is preferred; memory-blocked F -> W sub-block."""
    d = inst(1, 3, 1, 2, 2, 2, m_f=2, m_d=-1, m_w=-1, mlim_x1000=2000)   # m_lim = 4: two F in flight
    g = oracle_lib.greedy(d)
    seq = list(g["codes"][0, :g["len"][0]])
    assert seq[0] == 0                       # warm-up: F first
    assert seq[1] == 2                       # after F, D (local F -> D on last stage)
    d2 = inst(1, 2, 1, 2, 2, 2, m_f=2, m_d=0, m_w=-2, mlim_x1000=1000)   # m_lim = 2
    s2 = list(oracle_lib.greedy(d2)["codes"][0, :9])
    assert s2[:4] == [0, 2, 3, 0]            # F blocked by memory until W releases


# --------------------------------------------------------------------------- brute force
def test_exhaustive_optimum_vs_python_brute_force(oracle_lib):
    """§4.1 validity set: the oracle's enumeration optimum equals a Python brute force over all
    per-stage permutations evaluated by the fixed-point formulation (SPEC.md:547 <= 14 ops)."""
    rng = np.random.default_rng(13)
    cases = [(2, 2), (2, 1), (3, 1), (1, 3), (2, 2), (4, 1)]
    for p, m in cases:
        d = K.random_instances(1, seed=int(rng.integers(1 << 30)), max_p=1, max_m=1).item(0)
        d = inst(p, m, int(rng.integers(1, 3)), int(rng.integers(1, 9)), int(rng.integers(1, 9)),
                 int(rng.integers(1, 9)), lat=int(rng.integers(0, 6)), bw=int(rng.integers(0, 6)),
                 mlim_x1000=int(rng.choice([1000, 1500, 3000])))
        e = oracle_lib.enumerate_opt(d)
        assert e["evaluated"] > 0
        assert e["makespan"] == brute_force_opt(d)


def test_optimal_le_greedy_le_and_le_1f1b(oracle_lib):
    """North star / Q25: optimal <= greedy(n_sub=1) (theorem, same space and budget) and
    optimal <= 1F1B; greedy <= 1F1B is only reported (empirical), not asserted."""
    rng = np.random.default_rng(14)
    for _ in range(30):
        p, m = [(2, 2), (2, 3), (3, 2), (4, 1), (3, 1)][int(rng.integers(5))]
        f = int(rng.integers(1, 9))
        d = inst(p, m, 2, f, int(rng.integers(1, 9)), int(rng.integers(1, 9)),
                 lat=int(rng.integers(0, 12)), bw=int(rng.integers(0, 8)), mlim_x1000=1000)
        e = oracle_lib.enumerate_opt(d)
        g = oracle_lib.greedy(d)
        s = oracle_lib.simulate(d, *oracle_lib.build_static("1f1b", p, m))
        assert e["makespan"] <= g["makespan"]
        assert e["makespan"] <= s["makespan"]


def test_p1_optimum_is_total_work(oracle_lib):
    """One stage: every valid order is gap-free, so optimum = greedy = m (f + d + w)."""
    d = inst(1, 3, 1, 3, 4, 5, mlim_x1000=3000)
    assert oracle_lib.enumerate_opt(d)["makespan"] == 3 * 12 == oracle_lib.greedy(d)["makespan"]


# --------------------------------------------------------------------------- regression (survey check)
def test_survey_check_tiny_config(oracle_lib):
    """REGRESSION (SURVEY.md §8(c) survey-check table; same reading, not independent).
    The (0,0) column is independently fixed by Z1 (3300) and Z6 (2700); GPipe at (1,.5) by Z2."""
    for pt in gold("survey_check_tiny.json")["points"]:
        d = K.tiny(pt["lat_ratio"], pt["bw_ratio"]).item(0)
        assert oracle_lib.simulate(d, *oracle_lib.build_static("gpipe", 4, 8))["makespan"] == pt["gpipe"]
        assert oracle_lib.simulate(d, *oracle_lib.build_static("1f1b", 4, 8))["makespan"] == pt["1f1b"]
        for ns, want in zip((1, 2, 4), pt["greedy"]):
            e = dict(d); e["n_sub"] = ns
            assert oracle_lib.greedy(e)["makespan"] == want


# --------------------------------------------------------------------------- quantization
def test_quantize_grounding(oracle_lib):
    """Q21 quantization pinned to PAPER.md:618 numbers: T_F = 0.038 s -> 38,000 ticks @1 us;
    1 GB at 421 Gb/s -> 19.0024 ms -> 19,002 ticks; alpha 19 ms -> 19,000; half-away rounding."""
    g = gold("spec_examples.json")["m70_grounding"]
    spec = {"p": 2, "m": 4, "n_sub": 1, "zero1": 0, "n_dc": 2, "dc_of_stage": [0, 1],
            "t_f": [0.038, 0.038], "t_d": [0.038, 0.038], "t_w": [2.5e-6, 0.0000015],
            "m_f": [2e9, 2e9], "m_d": [-1e9, -1e9], "m_w": [-1e9, -1e9], "m_lim": [8.5e9, 8e9],
            "t_dp": [0.0, 0.0], "t_ag": [0.0, 0.0],
            "alpha": [[0, 0.019], [0.076, 0]], "beta": [[0, 8 / 421e9], [8 / 105e9, 0]],
            "msg_f": [g["msg_bytes"]], "msg_b": [g["msg_bytes"]], "tick_s": 1e-6, "mem_unit": 1e9}
    q = oracle_lib.quantize(spec)
    assert q["status"] == 0
    assert list(q["t_f"]) == [38000, 38000]
    assert list(q["t_w"]) == [3, 2]                 # 2.5 -> 3 (half away from zero), 1.5 -> 2
    assert list(q["lat_f"]) == [19000] and list(q["lat_b"]) == [76000]
    assert list(q["bw_f"]) == [19002]               # 1e9*8/421e9 s = 19.0024 ms
    assert list(q["bw_b"]) == [76190]               # 1e9*8/105e9 s = 76.190 ms
    assert list(q["m_lim"]) == [8, 8]               # budgets floor: 8.5 -> 8
    bad = dict(spec, dc_of_stage=[1, 0])
    assert oracle_lib.quantize(bad)["status"] == 8  # non-contiguous DC assignment
    bad2 = dict(spec, m_w=[-2e9, -1e9])
    assert oracle_lib.quantize(bad2)["status"] == 8  # deltas do not sum to zero


def test_message_size_and_presets():
    """message size b*s*d*n_DP*2; preset beta = 8 / (Gb/s * 1e9) s/B."""
    g = gold("spec_examples.json")
    for b, s, dd, ndp, bpe, want in g["message_size"]["cases"]:
        assert b * s * dd * ndp * bpe == want
    assert K.bw_ticks(421.0)[()] == 19002 and K.bw_ticks(105.0)[()] == 76190


# --------------------------------------------------------------------------- sweep synthesis
def test_grid_instance_synthesis(oracle_lib):
    """the oracle's grid point decode equals an instance built directly
    (workloads.uniform_instance) for random points of the config-5 grid."""
    g = K.full_sweep_grid()
    rng = np.random.default_rng(15)
    for k in rng.integers(0, g.n_points, size=40):
        i_pp, i_mb, i_lat, i_bw, i_mem, i_dp = (int(x) for x in g.point_axes(int(k)))
        p, m = g.pp_vals[i_pp], g.mb_vals[i_mb]
        want = K.uniform_instance(p, m, g.n_dc, int(g.base.t_f[0, 0]), int(g.base.t_d[0, 0]), int(g.base.t_w[0, 0]),
                                  lat=int(g.lat[i_lat]), bw=int(g.bw[i_bw]), mlim_x1000=int(g.mlim_x1000[i_mem]),
                                  t_dp=int(g.tdp[i_dp]), tick_s=g.base.tick_s).item(0)
        got = oracle_lib.grid_instance(g, int(k))
        for key in want:
            assert np.array_equal(np.asarray(got[key]), np.asarray(want[key])), key


def test_sweep_point_tiny(oracle_lib):
    """Sweep argmin on the tiny grid point (1, .5): GPipe infeasible (peak 16 > 8), so the
    winner is greedy; candidate makespans match Z2 (GPipe) and direct evaluation."""
    from workloads.core import Grid
    base = K.tiny(0, 0)
    g = Grid(base=base, n_dc=2, pp_vals=[4], mb_vals=[8], lat=np.array([100]), bw=np.array([50]),
             mlim_x1000=np.array([1000]), tdp=np.array([0]), cand_mask=0b11111)
    key, cm = oracle_lib.sweep_point(g, 0)
    assert cm[0] == -1                                  # GPipe memory-infeasible at M_L = p*m_f
    assert cm[1] == 4500 and cm[2] == cm[3] == cm[4] == 3300
    assert key == (3300 << 8) | 2
    # candidate 5 = ZB-H1 (Q30, Q31): the direct simulation of its built plan; key = lowest
    # (makespan, id) over all six
    g.cand_mask = 0b111111
    key6, cm6 = oracle_lib.sweep_point(g, 0)
    d = oracle_lib.grid_instance(g, 0)
    z = oracle_lib.simulate(d, *oracle_lib.build_static("zbh1", 4, 8))
    assert z["status"] == 0 and cm6[5] == z["makespan"] and cm6[:5] == cm[:5] and cm[5] == -1
    assert key6 == min(((c_ << 8) | i) for i, c_ in enumerate(cm6) if c_ >= 0)


# --------------------------------------------------------------------------- Wave pattern (reading Q32)
def test_wave_equals_fixed_point_formulation(oracle_lib):
    """The oracle's Wave DAG simulation (Kahn order, first-fit link windows) == the least fixed
    point of the §3.5 start-time equations over the Wave data flow with FIFO links
    (helpers_independent.fp_simulate_wave), start tick by start tick, on random valid plans
    (split and combined, n_sub 1-4, delays, ZeRO-1, DP tails)."""
    from tests.helpers_independent import fp_simulate_wave
    from workloads.wave import random_wave_plan
    rng = np.random.default_rng(320)
    for _ in range(150):
        b = K.random_instances(1, seed=int(rng.integers(1 << 30)), max_p=6, max_m=5, intra_delay=True)
        d = b.item(0)
        rows = random_wave_plan(d["p"], d["m"], d["n_sub"], rng, combined=bool(rng.random() < 0.25))
        r = oracle_lib.simulate_wave(d, rows, timeline=True)
        f = fp_simulate_wave(d, rows)
        assert r["status"] & ~2 == 0 and r["makespan"] == f["makespan"]
        for s in range(d["p"]):
            assert list(r["t_start"][s][:len(rows[s])]) == f["start"][s]


def test_wave_single_microbatch_four_crossings(oracle_lib):
    """One microbatch, every stage F0 F1 D1 D0 W1 W0: the chain F0 out, F1 back, D1 out, D0 back
    crosses every boundary four times ("4 for Wave and 2 for UD"), so the makespan
    is 2p(t_f + t_d) + 2 t_w + 2 sum_b(lat_f + bw_f + lat_b + bw_b)."""
    rng = np.random.default_rng(321)
    for _ in range(60):
        p, n_dc = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        f, dd_, w = (int(x) for x in rng.integers(1, 100, size=3))
        lat, bw, latb, bwb = (int(x) for x in rng.integers(0, 80, size=4))
        d = inst(p, 1, n_dc, f, dd_, w, lat=lat, bw=bw, lat_b=latb, bw_b=bwb, mlim_x1000=10**6)
        rows = [[F, F | 4, D | 4, D, W | 4, W] for _ in range(p)]
        r = oracle_lib.simulate_wave(d, rows)
        cross = sum(int(d["lat_f"][b] + d["bw_f"][b] + d["lat_b"][b] + d["bw_b"][b]) for b in range(p - 1))
        assert r["status"] == 0 and r["makespan"] == 2 * p * (f + dd_) + 2 * w + 2 * cross


def test_wave_plan_rules_and_deadlock(oracle_lib):
    """Q29 per chunk: F count m, D+B count m, W = n_sub * D with the prefix rule, no B/D mixing,
    codes < 8; a turn-around taken in the wrong order (F1 before F0 on the last stage) deadlocks."""
    d = inst(3, 2, 1, 5, 5, 5, mlim_x1000=10**6)
    good = [[F, F, F | 4, F | 4, D | 4, D | 4, D, D, W | 4, W | 4, W, W] for _ in range(3)]
    assert oracle_lib.check_plan_wave(d, good) == 0
    assert oracle_lib.simulate_wave(d, good)["status"] == 0
    bad_count = [r[:] for r in good]; bad_count[1] = bad_count[1][:-1] + [W | 4]
    bad_prefix = [r[:] for r in good]; bad_prefix[0] = [W] + bad_prefix[0][:-1]
    bad_mix = [r[:] for r in good]; bad_mix[2] = [F, F, F | 4, F | 4, B | 4, B | 4, D, D, W, W]
    bad_code = [r[:] for r in good]; bad_code[0][0] = 9
    for plan in (bad_count, bad_prefix, bad_mix, bad_code):
        assert oracle_lib.check_plan_wave(d, plan) == 4 and oracle_lib.simulate_wave(d, plan)["status"] == 4
    cyc = [r[:] for r in good]
    cyc[2] = [F | 4, F, F, F | 4, D | 4, D | 4, D, D, W | 4, W | 4, W, W]
    assert oracle_lib.simulate_wave(d, cyc)["status"] == 1


# --------------------------------------------------------------------------- Loop pattern (reading Q33)
def test_loop_equals_fixed_point_formulation(oracle_lib):
    """The oracle's Loop DAG simulation == the least fixed point of the §3.5 equations over the Loop
    data flow with FIFO links including the two wrap-around links (helpers_independent.
    fp_simulate_loop), start tick by start tick, on random valid plans."""
    from tests.helpers_independent import fp_simulate_loop
    from workloads.wave import random_loop_plan
    rng = np.random.default_rng(330)
    for _ in range(150):
        b = K.random_instances(1, seed=int(rng.integers(1 << 30)), max_p=6, max_m=5, intra_delay=True)
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):                 # the wrap link, boundary p-1
            getattr(b, fld)[0, b.p[0] - 1] = int(rng.integers(0, 200)) if rng.random() < 0.7 else 0
        d = b.item(0)
        rows = random_loop_plan(d["p"], d["m"], d["n_sub"], rng, combined=bool(rng.random() < 0.25))
        r = oracle_lib.simulate_loop(d, rows, timeline=True)
        f = fp_simulate_loop(d, rows)
        assert r["status"] & ~2 == 0 and r["makespan"] == f["makespan"]
        for s in range(d["p"]):
            assert list(r["t_start"][s][:len(rows[s])]) == f["start"][s]


def test_loop_single_microbatch_six_crossings(oracle_lib):
    """One microbatch, every stage F0 F1 D1 D0 W1 W0: F0 out, wrap, F1 out, D1 back, wrap, D0 back.
    Every inner boundary is crossed four times and the wrap link twice, so with 2 DCs a microbatch
    makes 6 cross-DC transfers ("6 per microbatch" for Loop): makespan =
    2p(t_f + t_d) + 2 t_w + 2 sum_{b<p-1}(lat_f + bw_f + lat_b + bw_b) + (wrap lat + bw both ways)."""
    rng = np.random.default_rng(331)
    for _ in range(60):
        p, n_dc = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        f, dd_, w = (int(x) for x in rng.integers(1, 100, size=3))
        lat, bw, latb, bwb = (int(x) for x in rng.integers(0, 80, size=4))
        b = K.uniform_instance(p, 1, n_dc, f, dd_, w, lat=lat, bw=bw, lat_b=latb, bw_b=bwb, mlim_x1000=10**6)
        wrap = [int(x) for x in rng.integers(0, 90, size=4)]
        b.lat_f[0, p - 1], b.bw_f[0, p - 1], b.lat_b[0, p - 1], b.bw_b[0, p - 1] = wrap
        d = b.item(0)
        rows = [[F, F | 4, D | 4, D, W | 4, W] for _ in range(p)]
        r = oracle_lib.simulate_loop(d, rows)
        inner = sum(int(d["lat_f"][s] + d["bw_f"][s] + d["lat_b"][s] + d["bw_b"][s]) for s in range(p - 1))
        assert r["status"] == 0 and r["makespan"] == 2 * p * (f + dd_) + 2 * w + 2 * inner + sum(wrap)
        if n_dc == 2 and p >= 2:
            crossings = 2 * int(np.count_nonzero(d["lat_f"][:p - 1])) + 2 * int(np.count_nonzero(d["lat_b"][:p - 1])) + 2
            assert lat == 0 or latb == 0 or crossings == 6


def test_loop_deadlock_and_wrap_validation(oracle_lib):
    """F1 before F0 on stage 0 closes a cycle through the wrap link (DEADLOCK); a negative wrap delay
    is an invalid instance."""
    d = inst(3, 1, 1, 5, 5, 5, mlim_x1000=10**6)
    good = [[F, F | 4, D | 4, D, W | 4, W] for _ in range(3)]
    assert oracle_lib.simulate_loop(d, good)["status"] == 0
    cyc = [r[:] for r in good]
    cyc[0] = [F | 4, F, D | 4, D, W | 4, W]
    assert oracle_lib.simulate_loop(d, cyc)["status"] == 1
    d["lat_b"] = np.array([0, 0, -1])
    assert oracle_lib.simulate_loop(d, good)["status"] == 8


def test_iv1f1b_closed_form_and_memory(oracle_lib):
    """Reading Q34 (interleaved 1F1B on the Loop pattern, 2 chunks, combined B): at zero delay with
    uniform costs and m % p == 0 the makespan is 2m(f+b) + (p-1)(f+b) with b = t_d + t_w -- 1F1B's
    pipeline fill (p-1)(f+b) per chunk, halved relative to running the two chunks as one block (the
    interleaving's purpose, :471 "Bubble Ratio: Medium"); stage s holds w_s + 1 microbatch-chunks,
    w_s = min(2(p-s-1) + p, 2m), so its peak is (w_s + 1) m_f."""
    rng = np.random.default_rng(34)
    for _ in range(80):
        p = int(rng.integers(1, 9))
        m = p * int(rng.integers(1, 4))
        f, dd_, w = (int(x) for x in rng.integers(1, 80, size=3))
        mf = int(rng.integers(1, 5))
        md = -int(rng.integers(0, mf + 1))
        d = inst(p, m, int(rng.integers(1, 5)), f, dd_, w, m_f=mf, m_d=md, m_w=-mf - md, mlim_x1000=10**6)
        c, l_ = oracle_lib.build_static("iv1f1b", p, m)
        assert oracle_lib.check_plan_wave(d, c, l_) == 0
        r = oracle_lib.simulate_loop(d, c, l_)
        b = dd_ + w
        assert r["status"] == 0 and r["makespan"] == 2 * m * (f + b) + (p - 1) * (f + b), (p, m, f, dd_, w)
        assert list(r["peak"]) == [(min(2 * (p - s - 1) + p, 2 * m) + 1) * mf if min(2 * (p - s - 1) + p, 2 * m) < 2 * m
                                   else 2 * m * mf for s in range(p)]


# --------------------------------------------------------------------------- ZB-V (reading Q35)
def test_zbv_zero_bubble_at_the_lower_bound(oracle_lib):
    """Reading Q35 (ZB-V, Wave pattern, split W), SPEC.md:545 acceptance 2 ("bubble ratio <= 0.02 on
    every stage" for uniform t_f = t_d = t_w, zero delay, m >= 2p): here every stage's bubble ratio
    over its active window is exactly 0 and the makespan is the lower bound
    (6m + p - 1) t -- the last stage cannot start before (p - 1) t (chunk 0 crosses p - 1 stages)
    and then runs 6m blocks of t.  Peak memory stays within 2p chunk activations, the 1F1B stage-0
    peak of p full-stage activations (Table :473, "Memory: Medium")."""
    rng = np.random.default_rng(35)
    for p in range(1, 9):
        for m in sorted({2 * p, 2 * p + 1, 3 * p, 4 * p + 3}):
            t = int(rng.integers(1, 50))
            d = inst(p, m, int(rng.integers(1, 5)), t, t, t, m_f=1, m_d=0, m_w=-1, mlim_x1000=10**6)
            c, l_ = oracle_lib.build_static("zbv", p, m)
            assert list(l_) == [6 * m] * p and oracle_lib.check_plan_wave(d, c, l_) == 0
            r = oracle_lib.simulate_wave(d, c, l_, timeline=True)
            assert r["status"] == 0 and r["makespan"] == (6 * m + p - 1) * t, (p, m)
            for s in range(p):
                st = r["t_start"][s][:6 * m]
                assert st.max() + t - st.min() == 6 * m * t, (p, m, s)        # busy window: no idle tick
            assert max(r["peak"]) <= 2 * p


def test_zbv_small_m_and_dominance(oracle_lib):
    """m < 2p: the plan is valid and completes within the 2p budget (no zero-bubble claim).  Zero-delay
    dominance (Fig. 6's left edge): with the stage cost split over two half-cost
    chunks, makespan(ZBV) <= makespan(ZBH1) <= makespan(1F1B) at t_d = t_w."""
    for p in range(1, 9):
        for m in range(1, 2 * p):
            d = inst(p, m, 2, 10, 10, 10, m_f=1, m_d=0, m_w=-1, mlim_x1000=10**6)
            c, l_ = oracle_lib.build_static("zbv", p, m)
            r = oracle_lib.simulate_wave(d, c, l_)
            assert oracle_lib.check_plan_wave(d, c, l_) == 0 and r["status"] == 0 and max(r["peak"]) <= 2 * p
    for p in (4, 8):
        for m in (2 * p, 3 * p):
            for f, b in ((100, 100), (60, 100), (100, 40)):
                ud = inst(p, m, 2, f, b, b, mlim_x1000=10**6)
                half = inst(p, m, 2, f // 2, b // 2, b // 2, m_f=1, m_d=0, m_w=-1, mlim_x1000=10**6)
                zv = oracle_lib.simulate_wave(half, *oracle_lib.build_static("zbv", p, m))["makespan"]
                zh = oracle_lib.simulate(ud, *oracle_lib.build_static("zbh1", p, m))["makespan"]
                one = oracle_lib.simulate(ud, *oracle_lib.build_static("1f1b", p, m))["makespan"]
                assert zv <= zh <= one, (p, m, f, b, zv, zh, one)


def test_e1_orderings_spec_acceptance_5(oracle_lib):
    """SPEC.md:548 acceptance 5 on the §5.1 setup (4 stages, 2 DCs x 2, 8 microbatches, F = D = W = T_F,
    UD memory budget = 1F1B's) over (T_lat/T_F, T_bw/T_F) in {0, 0.5, 1, 2}^2, slowdowns relative to
    ZBV at zero delay (PAPER.md :486): (a) at zero delay Wave <= every UD schedule; (b) at (2, 2) every
    UD schedule <= Wave; (c) Loop (IV1F1B) >= Wave and >= the WGrad-split UD schedules (ZB-H1, greedy)
    at every nonzero point (:496).  Two-chunk schedules run half-cost chunks; the Loop wrap link
    crosses DCs.  (The unified-backward 1F1B stays above IV1F1B at small delays: DESIGN.md §12.)"""
    O = oracle_lib
    f, h = 200, 100
    cz, lz = O.build_static("zbv", 4, 8)
    ci, li_ = O.build_static("iv1f1b", 4, 8)
    res = {}
    for a in (0, 0.5, 1, 2):
        for b in (0, 0.5, 1, 2):
            lat, bw = int(a * f), int(b * f)
            ud = inst(4, 8, 2, f, f, f, lat=lat, bw=bw)
            r = {k: O.simulate(ud, *O.build_static(k, 4, 8))["makespan"] for k in ("1f1b", "zbh1")}
            r["greedy"] = min(O.greedy(inst(4, 8, 2, f, f, f, lat=lat, bw=bw, n_sub=ns))["makespan"] for ns in (1, 2, 4))
            r["zbv"] = O.simulate_wave(inst(4, 8, 2, h, h, h, m_f=1, m_d=0, m_w=-1, mlim_x1000=2000, lat=lat, bw=bw),
                                       cz, lz)["makespan"]
            lb = K.uniform_instance(4, 8, 2, h, h, h, m_f=1, m_d=-1, m_w=0, lat=lat, bw=bw, mlim_x1000=10**6)
            lb.lat_f[0, 3], lb.bw_f[0, 3], lb.lat_b[0, 3], lb.bw_b[0, 3] = lat, bw, lat, bw
            r["iv1f1b"] = O.simulate_loop(lb.item(0), ci, li_)["makespan"]
            res[a, b] = r
    ud_all = ("1f1b", "zbh1", "greedy")
    assert all(res[0, 0]["zbv"] <= res[0, 0][k] for k in ud_all), res[0, 0]
    assert all(res[2, 2][k] <= res[2, 2]["zbv"] for k in ud_all), res[2, 2]
    for (a, b), r in res.items():
        if (a, b) != (0, 0):
            assert r["iv1f1b"] >= max(r["zbv"], r["zbh1"], r["greedy"]), ((a, b), r)


# --------------------------------------------------------------------------- instance invariants
# One hand-built violation per invariant of SPEC.md:46-50 (ProblemSpec invariants) and of the
# readings that add to them (Q10 memory signs, Q12 every block >= n_sub ticks, Q19 DP times >= 0,
# CP_MAX_STAGES).  Each starts from a valid instance and changes one invariant at one stage (the
# memory cases move a second delta so that only the named invariant breaks), so a validator that
# skips, mis-indexes or inverts any single test fails here.  The boundary value that must stay
# VALID (equality case or zero) is checked beside each.
_INVARIANT_CASES = [
    # (SPEC / reading, fields, stage, bad values, still-valid values)
    ("SPEC.md:46 n_pp >= 1", ("p",), None, (0,), (1,)),
    ("SPEC.md:46 n_mb >= 1", ("m",), None, (0,), (1,)),
    ("SPEC.md:46 n_sub >= 1", ("n_sub",), None, (0,), (1,)),
    ("CP_MAX_STAGES p <= 32", ("p",), None, (33,), (32,)),
    ("SPEC.md:46 durations > 0 (F)", ("t_f",), 2, (0,), (1,)),
    ("SPEC.md:46 durations > 0 (D)", ("t_d",), 0, (-5,), (1,)),
    ("SPEC.md:46 durations > 0 (W)", ("t_w",), 3, (0,), (1,)),
    ("SPEC.md:46 alpha >= 0 (fwd latency)", ("lat_f",), 1, (-1,), (0,)),
    ("SPEC.md:46 beta >= 0 (fwd window)", ("bw_f",), 0, (-1,), (0,)),
    ("SPEC.md:46 alpha >= 0 (bwd latency)", ("lat_b",), 2, (-3,), (0,)),
    ("SPEC.md:46 beta >= 0 (bwd window)", ("bw_b",), 1, (-2,), (0,)),
    ("SPEC.md:37 m_f > 0", ("m_f", "m_d", "m_w"), 1, (0, 0, 0), (1, 0, -1)),
    ("SPEC.md:37 m_d <= 0", ("m_d", "m_w"), 2, (1, -3), (0, -2)),
    ("SPEC.md:37 m_w <= 0", ("m_w", "m_d"), 0, (1, -3), (0, -2)),
    ("SPEC.md:48 m_f + m_d + m_w = 0", ("m_w",), 3, (-2,), (-1,)),
    ("SPEC.md:49 m_limit >= m_f", ("m_lim",), 1, (1,), (2,)),
    ("Q19 t_dp >= 0", ("t_dp",), 2, (-1,), (0,)),
    ("Q19 t_ag >= 0", ("t_ag",), 0, (-1,), (0,)),
]


def _full(batch, i=0):
    """Instance i as a dict with all 32 per-stage / per-boundary slots (item() trims to p)."""
    d = {"p": int(batch.p[i]), "m": int(batch.m[i]), "n_sub": int(batch.n_sub[i]), "zero1": int(batch.zero1[i])}
    for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag", "lat_f", "bw_f", "lat_b", "bw_b"):
        d[k] = np.array(getattr(batch, k)[i], copy=True)
    return d


@pytest.mark.parametrize("why,fields,stage,bad,ok", _INVARIANT_CASES, ids=[c[0] for c in _INVARIANT_CASES])
def test_validate_instance_each_invariant(oracle_lib, why, fields, stage, bad, ok):
    b = K.uniform_instance(4, 3, 2, 10, 10, 10, lat=5, bw=3, mlim_x1000=1000)
    if "p" in fields and bad[0] > 4:          # a 33- / 32-stage variant: fill every slot validly
        b = K.uniform_instance(32, 3, 2, 10, 10, 10, lat=5, bw=3, mlim_x1000=1000)
    base = _full(b)
    assert oracle_lib.validate_instance(base) == 0

    def with_values(vals):
        d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
        for f, x in zip(fields, vals):
            if stage is None:
                d[f] = x
            else:
                d[f][stage] = x
        return d

    bad_d = with_values(bad)
    assert oracle_lib.validate_instance(bad_d) == 8, why
    assert oracle_lib.validate_instance(with_values(ok)) == 0, why
    if 1 <= bad_d["p"] <= 32 and bad_d["m"] >= 1 and bad_d["n_sub"] >= 1:
        # the greedy and the simulator refuse it with the same status
        assert oracle_lib.greedy(bad_d)["status"] == 8, why
        c, ln = oracle_lib.build_static("1f1b", bad_d["p"], bad_d["m"])
        assert oracle_lib.simulate(bad_d, c, ln)["status"] == 8, why


@pytest.mark.parametrize("n_sub", [2, 4])
@pytest.mark.parametrize("fld", ["t_f", "t_d", "t_w"])
def test_validate_instance_every_block_at_least_n_sub(oracle_lib, n_sub, fld):
    """Q12 (changed from t_w only): every sub-block of every block (PAPER.md:377 splits every
    computation block into n_sub) lasts >= 1 tick, so each of t_f, t_d, t_w must be >= n_sub."""
    d = _full(K.uniform_instance(3, 2, 1, 10, 10, 10, n_sub=n_sub))
    d[fld][1] = n_sub - 1
    assert oracle_lib.validate_instance(d) == 8
    d[fld][1] = n_sub
    assert oracle_lib.validate_instance(d) == 0


def test_validate_instance_ignores_padding_and_unused_boundary(oracle_lib):
    """Only stages s < p and boundaries s < p - 1 are inspected: garbage past p (and in boundary
    p - 1, the Loop wrap slot, unused under UD) leaves a valid instance valid."""
    d = _full(K.uniform_instance(3, 2, 1, 10, 10, 10))
    for k in ("t_f", "t_d", "t_w", "m_f", "m_lim"):
        d[k][3:] = -7
    for k in ("lat_f", "bw_f", "lat_b", "bw_b"):
        d[k][2:] = -9
    assert oracle_lib.validate_instance(d) == 0
