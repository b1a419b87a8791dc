"""Workers for the every-item parity gate (tests/test_full_population_gpu.py).

Test infrastructure only.  Each job regenerates one slice of a benchmarked population on the
host from its seeds (workloads/, no method arithmetic), runs the CPU oracle on every item of the
slice, and returns the oracle's outputs as arrays.  The GPU side never feeds the oracle: the
plans the oracle sees come from the host generator, and a digest of their bytes is returned so
the test can check that the device generator produced the same plans.  No torch import, so
spawn-context workers start quickly.

Populations (BASELINE.json configs, SURVEY.md §8(d) "the oracle also checks parity on every
item of configs 1-5"; definitions PAPER.md:259 (§3.5 timeline), :383-412 (Alg. 1)):
  c3    -- config 3, 1e5 greedy instances: plan bytes, makespan, status, peak, per-stage stats
  c4    -- config 4, 1e6 perturbed schedules: makespan, status, peak, per-stage stats
  wave  -- the bench's Wave / Loop lines (NEXT 1), 2e5 plans each: makespan, status, peak, stats
  c5    -- config 5, 20,480 points: best key and every candidate's makespan
"""
import hashlib

import numpy as np


def _stats_rows(w, p):
    return np.stack([w["first_start"], w["last_end"], w["busy"], w["peak"]], axis=1)[:p]


def _fit32(a):
    a = np.asarray(a, dtype=np.int64)
    assert np.all(np.abs(a) < 2**31), "oracle value does not fit the int32 comparison array"
    return a.astype(np.int32)


def c4_slice(job):
    """Config 4 schedule ids [a, b): returns (a, b, plan_digest, ms, st, pk, stats [n, p, 4])."""
    a, b = job
    from oracle import oracle as O
    from workloads import configs as K, plans as PL, unpack_plans
    inst = K.perturbed_instance()
    d = inst.item(0)
    p = int(d["p"])
    ops, ln = PL.plans_host(inst, b - a, seed=K.PERTURB_SEED, id0=a, stride=32)
    h = hashlib.blake2b(ops.tobytes(), digest_size=16)
    h.update(ln.tobytes())
    codes, lens = unpack_plans(ops, ln)
    n = b - a
    ms = np.zeros(n, np.int64)
    st = np.zeros(n, np.int32)
    pk = np.zeros(n, np.int64)
    stats = np.zeros((n, p, 4), np.int64)
    for i in range(n):
        w = O.simulate(d, codes[i], lens[i])
        ms[i], st[i], pk[i] = w["makespan"], w["status"], w["peak_mem"]
        stats[i] = _stats_rows(w, p)
    return a, b, h.hexdigest(), ms, st, _fit32(pk), _fit32(stats)


def wave_slice(job):
    """Wave (loop=False) or Loop (loop=True) bench plans ids [a, b) of one p=32, m=32 instance."""
    a, b, loop = job
    from oracle import oracle as O
    from workloads import configs as K, plans as PL
    from workloads.wave import unpack_wave_plans
    inst = K.loop_instance() if loop else K.wave_instance()
    d = inst.item(0)
    p = int(d["p"])
    ops, ln = PL.wave_plans_host(32, 32, 1, b - a, seed=K.PERTURB_SEED ^ 0x3A, id0=a, q=1, stride=32, loop=loop)
    h = hashlib.blake2b(ops.tobytes(), digest_size=16)
    h.update(ln.tobytes())
    codes, lens = unpack_wave_plans(ops, ln)
    sim = O.simulate_loop if loop else O.simulate_wave
    n = b - a
    ms = np.zeros(n, np.int64)
    st = np.zeros(n, np.int32)
    pk = np.zeros(n, np.int64)
    stats = np.zeros((n, p, 4), np.int64)
    for i in range(n):
        w = sim(d, codes[i], lens[i])
        ms[i], st[i], pk[i] = w["makespan"], w["status"], w["peak_mem"]
        stats[i] = _stats_rows(w, p)
    return a, b, h.hexdigest(), ms, st, _fit32(pk), _fit32(stats)


def greedy_digest(status, makespan, peak, lens, codes, stats):
    """One greedy output: status, makespan, peak, per-stage row lengths, every 2-bit plan entry and the
    per-stage (first_start, last_end, busy, peak)."""
    h = hashlib.blake2b(digest_size=16)
    h.update(np.asarray([status, makespan, peak], dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(lens, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(codes, dtype=np.int8).tobytes())
    h.update(np.ascontiguousarray(stats, dtype=np.int64).tobytes())
    return h.hexdigest()


def c3_slice(job):
    """Config 3 instance ids [a, b): oracle Alg. 1 on each; returns (a, b, [digest per instance])."""
    a, b = job
    from oracle import oracle as O
    from workloads import configs as K
    batch = K.greedy_batch(b - a, id0=a)
    out = []
    for i in range(b - a):
        d = batch.item(i)
        w = O.greedy(d)
        p = d["p"]
        L = int(w["len"][0]) if p else 0
        out.append(greedy_digest(w["status"], w["makespan"], w["peak_mem"], w["len"][:p], w["codes"][:p, :L],
                                 _stats_rows(w, p)))
    return a, b, out


def c5_slice(job):
    """Config 5 point ids [a, b): returns (a, b, keys uint64 [n], cand_ms int64 [n, 6])."""
    a, b = job
    from oracle import oracle as O
    from workloads import configs as K
    grid = K.full_sweep_grid()
    G, keep = O.to_or_grid(grid)
    keys = np.zeros(b - a, np.uint64)
    cms = np.zeros((b - a, 6), np.int64)
    for k in range(a, b):
        key, cm = O.sweep_point(grid, k, G=G)
        keys[k - a] = key
        cms[k - a] = cm
    return a, b, keys, cms
