"""Concrete workloads of BASELINE.json `configs` (recipes: SURVEY.md §8(d)).

All values are integers (ticks, memory units).  Tick = 1 us unless stated.
T_F = 38,000 ticks is the M70 forward time ("T_F = 0.038 s");
PP messages are 1e9 B ("= 1 GB", 1 GB = 1e9 B per reading Q26).
"""
from __future__ import annotations

import numpy as np

from .core import MAXP, Grid, InstanceBatch, cross_dc_boundaries, splitmix64

T_F = 38_000
MSG_BYTES = 10**9
SEED = 0x250700217


def bw_ticks(gbps, msg_bytes=MSG_BYTES, tick_s=1e-6):
    """T_bw = beta * msg in ticks for a link of `gbps` Gb/s: round(msg*8/(gbps*1e9)/tick)."""
    g = np.asarray(gbps, dtype=np.float64)
    return np.floor(msg_bytes * 8.0 / (g * 1e9) / tick_s + 0.5).astype(np.int64)


def uniform_instance(p, m, n_dc, t_f, t_d, t_w, *, m_f=2, m_d=-1, m_w=-1, mlim_x1000=1000,
                     lat=0, bw=0, lat_b=None, bw_b=None, n_sub=1, t_dp=0, zero1=0, t_ag=0,
                     tick_s=1e-6) -> InstanceBatch:
    """One homogeneous instance; cross-DC boundaries (contiguous even split) carry (lat, bw)."""
    b = InstanceBatch.empty(1, tick_s)
    b.p[0], b.m[0], b.n_sub[0], b.zero1[0], b.n_dc[0] = p, m, n_sub, zero1, n_dc
    b.t_f[0, :p], b.t_d[0, :p], b.t_w[0, :p] = t_f, t_d, t_w
    b.m_f[0, :p], b.m_d[0, :p], b.m_w[0, :p] = m_f, m_d, m_w
    b.m_lim[0, :p] = (mlim_x1000 * p * m_f + 500) // 1000
    b.t_dp[0, :p] = t_dp
    b.t_ag[0, :p] = t_ag if zero1 else 0
    cross = cross_dc_boundaries(p, n_dc)
    lb = lat if lat_b is None else lat_b
    wb = bw if bw_b is None else bw_b
    b.lat_f[0, :p - 1] = np.where(cross, lat, 0)
    b.bw_f[0, :p - 1] = np.where(cross, bw, 0)
    b.lat_b[0, :p - 1] = np.where(cross, lb, 0)
    b.bw_b[0, :p - 1] = np.where(cross, wb, 0)
    return b


# ---------------------------------------------------------------------------------------
# config 1 -- tiny: 2 DCs, 4 stages, 8 microbatches, uniform F/B/W costs
def tiny(lat_ratio=1.0, bw_ratio=0.5, f=100, n_sub=1) -> InstanceBatch:
    return uniform_instance(4, 8, 2, f, f, f, lat=int(round(lat_ratio * f)), bw=int(round(bw_ratio * f)),
                            n_sub=n_sub)


def tiny_grid(f=100) -> InstanceBatch:
    """{0, .5, 1, 2}^2 delay-ratio grid of PAPER.md:616 on the tiny setup."""
    r = [0.0, 0.5, 1.0, 2.0]
    return InstanceBatch.concat([tiny(a, b, f) for a in r for b in r])


def e1_grid(f=T_F, steps=33, top=4.0) -> Grid:
    """E1, the delay-sensitivity study of PAPER.md §5.1 (Fig. pre_delay_sensitivity, :474-499):
    4 stages over 2 DCs (2 stages each), 8 microbatches, uniform F = D = W = T_F, memory budget
    of 1F1B ("dynamic schedules ... with the same memory limits as their static counterparts
    (e.g., CrossUD mirrors 1F1B)"), T_lat/T_F and T_bw/T_F each on `steps` values in [0, top];
    all six sweep candidates (GPipe, 1F1B, greedy n_sub 1/2/4, ZB-H1)."""
    base = uniform_instance(4, 8, 2, f, f, f)
    r = np.linspace(0.0, top, steps)
    ticks = np.floor(r * f + 0.5).astype(np.int64)
    return Grid(base=base, n_dc=2, pp_vals=[4], mb_vals=[8], lat=ticks, bw=ticks.copy(),
                mlim_x1000=np.array([1000], np.int64), tdp=np.array([0], np.int64), cand_mask=0b111111,
                name="e1_delay_sensitivity")


# ---------------------------------------------------------------------------------------
# config 2 -- GPT-style 16 stages over 2 DCs, 32 microbatches, 64 latencies x 64 bandwidths
def gpt16_grid() -> Grid:
    base = uniform_instance(16, 32, 2, T_F, T_F, T_F)
    lat_s = np.concatenate([[0.0], np.geomspace(1e-4, 0.2, 63)])
    lat = np.floor(lat_s / 1e-6 + 0.5).astype(np.int64)
    # the App. C bubble-stride point: latency 1.5 * T_F = 57,000 ticks
    lat[int(np.argmin(np.abs(lat - 57_000)))] = 57_000
    bw = bw_ticks(np.geomspace(1.0, 800.0, 64))
    return Grid(base=base, n_dc=2, pp_vals=[16], mb_vals=[32], lat=lat, bw=bw,
                mlim_x1000=np.array([1000], np.int64), tdp=np.array([0], np.int64),
                cand_mask=0b00111, name="gpt16x2_sweep")


# ---------------------------------------------------------------------------------------
# config 3 -- greedy generation for 1e5 instances varying memory limit and DP overlap
def greedy_batch(n=100_000, seed=SEED, p=16, n_dc=2, m=32, id0=0) -> InstanceBatch:
    """Instances id0 .. id0+n-1 of the config-3 population (each drawn from its own id)."""
    b = InstanceBatch.empty(n)
    ids = np.arange(id0, id0 + n, dtype=np.uint64)

    def draw(tag, k):
        return (splitmix64(np.uint64(seed) ^ (ids * np.uint64(64)) ^ np.uint64(tag)) % np.uint64(k)).astype(np.int64)

    b.p[:], b.m[:], b.n_dc[:] = p, m, n_dc
    b.n_sub[:] = np.array([1, 2, 4])[draw(1, 3)]
    scale = np.array([1000, 1250, 1500, 1750, 2000])[draw(2, 5)]
    tdp = (np.array([0, 500, 1000, 2000, 4000])[draw(3, 5)] * T_F) // 1000
    b.zero1[:] = draw(4, 2)
    lat = draw(5, 9) * T_F // 4
    bw = draw(6, 9) * T_F // 4
    jitter = draw(7, 2) == 1
    for s in range(p):
        for fld, tag in (("t_f", 8), ("t_d", 9), ("t_w", 10)):
            j = draw(tag * 64 + s, 201) - 100                    # per mille, [-100, 100]
            getattr(b, fld)[:, s] = np.where(jitter, T_F * (1000 + j) // 1000, T_F)
    b.m_f[:, :p], b.m_d[:, :p], b.m_w[:, :p] = 2, -1, -1
    b.m_lim[:, :p] = ((scale * p * 2 + 500) // 1000)[:, None]
    b.t_dp[:, :p] = tdp[:, None]
    b.t_ag[:, :p] = np.where(b.zero1 == 1, tdp // 2, 0)[:, None]
    cross = cross_dc_boundaries(p, n_dc)
    for s in np.nonzero(cross)[0]:
        b.lat_f[:, s] = b.lat_b[:, s] = lat
        b.bw_f[:, s] = b.bw_b[:, s] = bw
    return b


# ---------------------------------------------------------------------------------------
# config 4 -- 1e6 randomly perturbed valid schedules of one 32-stage, 4-DC, 64-mb instance
def perturbed_instance() -> InstanceBatch:
    """L = T_F, T_bw = T_F/2 (421 Gb/s), memory budget 1.5x the 1F1B peak."""
    return uniform_instance(32, 64, 4, T_F, T_F, T_F, lat=T_F, bw=T_F // 2, mlim_x1000=1500)


PERTURB_SEED = SEED ^ 0x4


def loop_instance() -> InstanceBatch:
    """Loop bench instance (NEXT 1, reading Q33): config 4's setup with m = 32 and the wrap-around links
    p-1 -> 0 / 0 -> p-1 (boundary index p-1) crossing from the last DC back to the first with the same
    (L = T_F, T_bw = T_F/2); memory budget 3x the 1F1B device peak."""
    b = uniform_instance(32, 32, 4, T_F, T_F, T_F, lat=T_F, bw=T_F // 2, mlim_x1000=3000)
    b.lat_f[0, 31], b.bw_f[0, 31], b.lat_b[0, 31], b.bw_b[0, 31] = T_F, T_F // 2, T_F, T_F // 2
    return b


def wave_instance() -> InstanceBatch:
    """Wave bench instance (NEXT 1): config 4's setup (p=32, 4 DCs, L = T_F, T_bw = T_F/2) with m = 32, so
    each stage runs 2 chunks x 3 x 32 = 192 entries as in config 4; memory budget 3x the 1F1B device
    peak (two chunks' activations)."""
    return uniform_instance(32, 32, 4, T_F, T_F, T_F, lat=T_F, bw=T_F // 2, mlim_x1000=3000)


# ---------------------------------------------------------------------------------------
# config 5 -- full sweep: 4 DCs, 8-32 stages, 8-128 mb, latency x bandwidth x memory grid
def full_sweep_grid(tick_s=1e-5) -> Grid:
    """Tick = 10 us so that the int32 guard (Q21) holds at 1 Gb/s, m = 128."""
    tf = int(round(T_F * 1e-6 / tick_s))
    base = InstanceBatch.empty(1, tick_s)
    base.p[0], base.m[0], base.n_dc[0] = 32, 8, 4
    base.t_f[0, :], base.t_d[0, :], base.t_w[0, :] = tf, tf, tf
    base.m_f[0, :], base.m_d[0, :], base.m_w[0, :] = 2, -1, -1
    lat = np.floor(np.geomspace(1e-3, 0.1, 16) / tick_s + 0.5).astype(np.int64)
    bw = bw_ticks(np.geomspace(1.0, 400.0, 16), tick_s=tick_s)
    return Grid(base=base, n_dc=4, pp_vals=[8, 16, 24, 32], mb_vals=[8, 16, 32, 64, 128], lat=lat, bw=bw,
                mlim_x1000=np.array([1000, 1500, 2000, 4000], np.int64), tdp=np.array([0], np.int64),
                cand_mask=0b11111, name="full_sweep_4dc")


# ---------------------------------------------------------------------------------------
# random small instances for parity tests (edge cases included by construction)
def random_instances(n, seed=SEED ^ 0x77, max_p=MAXP, max_m=24, max_cost=200, max_delay=300,
                     intra_delay=False) -> InstanceBatch:
    rng = np.random.default_rng(seed)
    b = InstanceBatch.empty(n)
    for i in range(n):
        p = int(rng.integers(1, max_p + 1))
        m = int(rng.integers(1, max_m + 1))
        n_dc = int(rng.integers(1, 5))
        ns = int(rng.choice([1, 1, 2, 3, 4]))
        b.p[i], b.m[i], b.n_sub[i], b.n_dc[i] = p, m, ns, n_dc
        uni = rng.random() < 0.3
        for fld in ("t_f", "t_d", "t_w"):
            v = rng.integers(1, max_cost + 1, size=p) if not uni else np.full(p, rng.integers(1, max_cost + 1))
            getattr(b, fld)[i, :p] = v
        for fld in ("t_f", "t_d", "t_w"):            # every sub-block >= 1 tick (reading Q12)
            getattr(b, fld)[i, :p] = np.maximum(getattr(b, fld)[i, :p], ns)
        mf = rng.integers(1, 5, size=p)
        md = -rng.integers(0, mf + 1)
        b.m_f[i, :p], b.m_d[i, :p], b.m_w[i, :p] = mf, md, -mf - md
        b.m_lim[i, :p] = mf * rng.integers(1, p + 3, size=p) + rng.integers(0, 2, size=p)
        if rng.random() < 0.3:
            b.t_dp[i, :p] = rng.integers(0, 3 * max_cost, size=p)
        if rng.random() < 0.3:
            b.zero1[i] = 1
            b.t_ag[i, :p] = rng.integers(0, 2 * max_cost, size=p)
        cross = cross_dc_boundaries(p, n_dc)
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            v = rng.integers(0, max_delay + 1, size=max(p - 1, 0))
            if rng.random() < 0.2:
                v[:] = 0
            mask = cross | (intra_delay and rng.random() < 0.5)
            getattr(b, fld)[i, :p - 1] = np.where(mask, v, 0)
    return b
