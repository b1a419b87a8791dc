"""Every-item parity gate (north_star: "bit-exact agreement with the CPU oracle on every generated
instance"; "the oracle also checks parity on every item of configs 1-5").

The CUDA path runs each benchmarked population once, in the launch configuration bench.py times
(and once more with per-stage stats), and every item is compared with the CPU oracle, element by
element.  Nothing is sampled.  The oracle runs in one spawn-context process per host core over
disjoint slices that it regenerates from their seeds (tests/full_parity_worker.py); the device
generator's plans are checked byte-equal to the host generator's by a digest per slice.

What is compared (definitions PAPER.md:259 §3.5, :383-412 Alg. 1, App. A :808):
  config 3 (1e5 instances)  -- greedy plan bytes, makespan, status, peak, per-stage stats
  config 4 (1e6 schedules)  -- makespan, status, peak, per-stage first/last/busy/peak
  Wave / Loop (2e5 each)    -- makespan, status, peak, per-stage stats (NEXT 1)
  config 5 (20,480 points)  -- best key and all six candidate makespans, single GPU and rank shards
Configs 1 and 2 and the E1 grid are checked at every point in tests/test_parity_gpu.py.
"""
import hashlib
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from tests import full_parity_worker as Wk  # noqa: E402
from workloads import configs as K, plans as PL, unpack_plans  # noqa: E402


def _procs():
    return max(1, min(64, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def pool():
    from oracle import oracle
    oracle.build()
    with mp.get_context("spawn").Pool(_procs()) as p:
        yield p


def _slices(n, k):
    step = (n + k - 1) // k
    return [(a, min(n, a + step)) for a in range(0, n, step)]


def _digest(ops_h, ln_h):
    h = hashlib.blake2b(ops_h.tobytes(), digest_size=16)
    h.update(ln_h.tobytes())
    return h.hexdigest()


def _check_fixed(name, jobs, fn, pool, ops, ln, r_bench, r_stats, p):
    """Compare one fixed-plan population slice by slice; returns the number of items checked."""
    ms, st, pk = (r_bench[k].cpu().numpy() for k in ("makespan", "status", "peak_mem"))
    ss = r_stats["stage_stats"].cpu().numpy()
    for k in ("makespan", "status", "peak_mem"):
        assert torch.equal(r_bench[k], r_stats[k]), (name, "bench launch vs stats launch", k)
    n_tot = 0
    for out in pool.imap_unordered(fn, jobs):
        a, b, dig, w_ms, w_st, w_pk, w_ss = out
        assert _digest(ops[a:b].cpu().numpy(), ln[a:b].cpu().numpy()) == dig, (name, "device plans != host", a)
        for lbl, got, want in (("makespan", ms[a:b], w_ms), ("status", st[a:b], w_st), ("peak", pk[a:b], w_pk)):
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (name, lbl, int(a + bad[0]), int(got[bad[0]]), int(want[bad[0]]), bad.size)
        bad = np.nonzero((ss[a:b, :p] != w_ss).any(axis=(1, 2)))[0]
        assert bad.size == 0, (name, "stage_stats", int(a + bad[0]), bad.size)
        n_tot += b - a
    return n_tot


def test_config4_every_schedule(pool):
    """Config 4: all 1e6 perturbed valid schedules (p=32, 4 DCs, m=64) in the bench launch (best key,
    no stats) and once with per-stage stats; every schedule against the oracle."""
    b = K.perturbed_instance()
    n = 1_000_000
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED, stride=32)
    inst = cp.Instances(b)
    rb = cp.simulate(inst, ops, ln, best=True)
    rs = cp.simulate(inst, ops, ln, stats=True)
    torch.cuda.synchronize()
    jobs = _slices(n, 8 * _procs())
    assert _check_fixed("config4", jobs, Wk.c4_slice, pool, ops, ln, rb, rs, 32) == n
    ms = rb["makespan"].cpu().numpy()
    assert np.all(rb["status"].cpu().numpy() == 0)
    bk = int(rb["best_key"][0])
    assert (bk >> 32) == ms.min() and (bk & 0xFFFFFFFF) == int(np.argmin(ms))


@pytest.mark.parametrize("loop", [False, True], ids=["wave", "loop"])
def test_two_chunk_bench_plans_every_plan(pool, loop):
    """The bench's Wave (Q32) / Loop (Q33) lines: all 2e5 plans of one p=32, 4-DC, m=32 instance."""
    b = K.loop_instance() if loop else K.wave_instance()
    n = 200_000
    ops, ln = PL.wave_plans_device(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32, loop=loop)
    inst = cp.Instances(b)
    kw = {"loop": True} if loop else {"wave": True}
    rb = cp.simulate(inst, ops, ln, best=True, **kw)
    rs = cp.simulate(inst, ops, ln, stats=True, **kw)
    torch.cuda.synchronize()
    jobs = [(a, c, loop) for a, c in _slices(n, 4 * _procs())]
    assert _check_fixed("loop" if loop else "wave", jobs, Wk.wave_slice, pool, ops, ln, rb, rs, 32) == n


def test_config3_every_greedy_instance(pool):
    """Config 3: all 1e5 greedy instances in the bench launch (plans + metrics) and once with stats:
    schedules byte for byte, makespan, status, peak and per-stage stats against sequential Alg. 1."""
    n = 100_000
    batch = K.greedy_batch(n)
    inst = cp.Instances(batch)
    gb = cp.greedy(inst)
    gs = cp.greedy(inst, stats=True)
    torch.cuda.synchronize()
    for k in ("ops", "len", "makespan", "status", "peak_mem"):
        assert torch.equal(gb[k], gs[k]), ("bench launch vs stats launch", k)
    codes, lens = unpack_plans(gs["ops"].cpu().numpy().view(np.uint32), gs["len"].cpu().numpy().view(np.uint16))
    st, ms, pk = (gs[k].cpu().numpy() for k in ("status", "makespan", "peak_mem"))
    ss = gs["stage_stats"].cpu().numpy()
    n_tot, bad = 0, []
    for a, b, want in pool.imap_unordered(Wk.c3_slice, _slices(n, 8 * _procs())):
        for i in range(a, b):
            p = int(batch.p[i])
            L = int(lens[i, 0])
            got = Wk.greedy_digest(st[i], ms[i], pk[i], lens[i, :p], codes[i, :p, :L], ss[i, :p])
            if got != want[i - a]:
                bad.append(i)
            n_tot += 1
    assert n_tot == n
    assert not bad, f"{len(bad)} of {n} instances differ; first {bad[:5]}"


def test_config5_every_point(pool):
    """Config 5: all 20,480 points with every candidate's makespan (single GPU), and the blocked
    8-rank shards assembled with MIN, against the oracle's per-point argmin."""
    grid = K.full_sweep_grid()
    keys, cm = cp.sweep_shard(grid, cand=True)
    acc = torch.full((grid.n_points,), cp.KEY_NONE, dtype=torch.int64, device="cuda")
    for rk in range(8):
        kr, _ = cp.sweep_shard_rank(grid, rk, 8)
        acc = torch.minimum(acc, kr)
    torch.cuda.synchronize()
    keys_h, cm_h, acc_h = keys.cpu().numpy(), cm.cpu().numpy(), acc.cpu().numpy()
    n_tot = 0
    for a, b, w_keys, w_cms in pool.imap_unordered(Wk.c5_slice, _slices(grid.n_points, 8 * _procs())):
        want = np.where(w_keys == np.uint64(2**64 - 1), np.int64(cp.KEY_NONE), w_keys.astype(np.int64))
        bad = np.nonzero(keys_h[a:b] != want)[0]
        assert bad.size == 0, ("key", int(a + bad[0]), int(keys_h[a + bad[0]]), int(want[bad[0]]))
        bad = np.nonzero((cm_h[a:b] != w_cms).any(axis=1))[0]
        assert bad.size == 0, ("cand_ms", int(a + bad[0]), list(cm_h[a + bad[0]]), list(w_cms[bad[0]]))
        assert np.array_equal(acc_h[a:b], want), ("8-rank shards", a)
        n_tot += b - a
    assert n_tot == grid.n_points
