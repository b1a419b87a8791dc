"""E2 (§5.2 :503-516, App. E :855-858; reading Q36): cross-DC PP vs cross-DC DP for
Llama-3-405B, evaluated by the oracle and pinned to the numbers the paper prints: PP over DP "up to
3.05x" at 4 GB/s (:507), "only a 1.3x slowdown at 64 GB/s" against the ideal single-DC run (:507),
the gap "negligible beyond 1024 GB/s" (:507; checked at 4096 GB/s), latency 4-128 ms of "little impact" (:507).  The
paper's t_PP is the exact CrossUD/CrossWave optimum; here it is the greedy CrossUDSub (best of n_sub
1/2/4) with the 1F1B memory budget, an upper bound on the CrossUD optimum, as SPEC.md:500 prescribes
at n_PP = 16.  (The static ZBV order beats it at high bandwidth and low latency but, unlike a
solver-built CrossWave, cannot adapt to 128 ms: tools/e2_ppdp.py reports it as a separate column.)
Tolerances: SPEC.md:549 (+-15 %, 5 %)."""
import numpy as np
import pytest

from workloads import ppdp as E


def _t_pp(O, alpha, bw):
    return min(O.greedy(E.pp_instance(alpha, bw, n_sub=ns).item(0))["makespan"] for ns in (1, 2, 4)) * E.TICK_S


def test_preset_calibration():
    """T_F from App. E's T_layer = C_layer / (P_GPU n_TP) with 8 layers per stage is the paper's
    ~109 ms anchor (:507); m = GBS / n_DP = 32; the PP message b s d n_DP 2."""
    assert abs(E.stage_forward_s() - 0.109) < 0.002
    assert E.n_microbatches() == 32 and E.pp_message_bytes() == 8192 * 16384 * 64 * 2
    assert abs(E.layer_params() * 126 / 405e9 - 1) < 0.02          # ~405 B parameters in the 126 layers


def test_pp_vs_dp_reproduces_section_5_2(oracle_lib):
    O = oracle_lib
    zbv = O.simulate_wave(E.wave_instance(0.0, float("inf")).item(0),
                          *O.build_static("zbv", 16, E.n_microbatches()))["makespan"] * E.TICK_S
    assert zbv == pytest.approx((6 * 32 + 15) * E.ticks(E.stage_forward_s() / 2) * E.TICK_S)   # Q35 lower bound
    bws = [4, 16, 64, 256, 1024, 4096]
    sp, slow = {}, {}
    for lat_ms in (4, 128):
        for g in bws:
            t_pp = _t_pp(O, lat_ms * 1e-3, g * 1e9)
            t_dp = zbv + E.dp_cost_s(lat_ms * 1e-3, g * 1e9)
            sp[lat_ms, g], slow[lat_ms, g] = t_dp / t_pp, t_pp / zbv
    assert 3.05 * 0.85 <= max(sp[l, 4] for l in (4, 128)) <= 3.05 * 1.15, sp
    assert 1.3 * 0.85 <= slow[4, 64] <= 1.3 * 1.15, slow
    assert abs(sp[4, 4096] - 1) <= 0.05 and sp[4, 1024] < 1.15, sp
    for g in bws:                                                   # latency 4 -> 128 ms: < 5 % on t_PP
        assert abs(slow[128, g] / slow[4, g] - 1) < 0.05, (g, slow)
    for lat_ms in (4, 128):                                         # non-increasing in bandwidth (1 % slack:
        s = [sp[lat_ms, g] for g in bws]                            # t_PP is a greedy upper bound)
        assert all(b <= a * 1.01 for a, b in zip(s, s[1:])), (lat_ms, s)
