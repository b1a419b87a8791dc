"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar: bit-exact on every integer output -- status, makespan, peak memory,
per-stage stats, the full start-tick timeline, and greedy schedules byte for byte.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from tests.gpu_util import codes_list_to_packed, compare_sim, plans_to_device, to_host  # noqa: E402
from tests.helpers_independent import random_valid_plan  # noqa: E402
from workloads import InstanceBatch, configs as K, pack_plans, plans as PL, unpack_plans  # noqa: E402


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def run_sim(batch, ops, ln, inst_of=None, stats=True, timeline=True, ring=None):
    inst = cp.Instances(batch)
    o, l_ = plans_to_device(ops, ln)
    io = torch.from_numpy(np.asarray(inst_of, dtype=np.int32)).cuda() if inst_of is not None else None
    r = cp.simulate(inst, o, l_, io, stats=stats, timeline=timeline, ring=ring)
    torch.cuda.synchronize()
    return to_host(r)


# ------------------------------------------------------------------------------------- simulate
@pytest.mark.parametrize("max_p,seed", [(32, 1), (8, 2), (4, 3), (16, 4)])
def test_simulate_random_valid_plans(O, max_p, seed):
    """Random instances (1..max_p stages, 1..24 mb, 1-4 DCs, n_sub 1-4, DP, ZeRO-1) x 4 random
    valid plans each; several lane segments per warp when max_p <= 16; full timelines compared."""
    batch = K.random_instances(120, seed=seed, max_p=max_p, max_m=24)
    plans, inst_of = [], []
    for i in range(len(batch)):
        ops, ln = PL.plans_host(batch, 4, seed=seed * 1000 + i, i=i, q=int(i % 5), stride=32)
        c, l_ = unpack_plans(ops, ln)
        for k in range(4):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2])
    assert np.all(r["status"] == 0)


@pytest.mark.parametrize("seed", [81, 82])
def test_simulate_fast_path_random_valid_plans(O, seed):
    """The bench kernel k_sim32 (stats only, stage stride 32, no timeline) on random instances (1-32
    stages in one batch, 1-24 mb, 1-4 DCs, n_sub 1-4, DP tails, ZeRO-1) x 4 random valid plans each,
    addressed through inst_of: status, makespan, peak and every stage's first / last / busy / peak."""
    batch = K.random_instances(160, seed=seed, max_p=32, max_m=24)
    plans, inst_of = [], []
    for i in range(len(batch)):
        ops, ln = PL.plans_host(batch, 4, seed=seed * 1000 + i, i=i, q=int(i % 5), stride=32)
        c, l_ = unpack_plans(ops, ln)
        for k in range(4):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of, stats=True, timeline=False)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2], timeline=False)
    assert np.all(r["status"] == 0)


def test_simulate_static_plans_and_overflow_path(O):
    """1F1B and GPipe (combined B) on random instances; GPipe exceeds the memory budget, which
    also drives the lead past the shared-memory ring -> global-ring fix-up pass must agree."""
    batch = K.random_instances(100, seed=5, max_p=32, max_m=30)
    plans, inst_of = [], []
    for i in range(len(batch)):
        p, m = int(batch.p[i]), int(batch.m[i])
        for kind in ("1f1b", "gpipe"):
            c, l_ = O.build_static(kind, p, m)
            plans.append([list(c[s, :l_[s]]) for s in range(p)])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2])
    assert np.any(r["status"] == 2)          # memory-exceeded items present


def test_simulate_invalid_plans(O):
    """Deadlocks (adjacent swaps), BAD_PLAN (missing/extra entries, W before D, B mixed with
    D/W), memory violations (budget cut after generation) -- status precedence included."""
    rng = np.random.default_rng(6)
    batch = K.random_instances(150, seed=7, max_p=12, max_m=10)
    plans, inst_of, mlim_cut = [], [], []
    for i in range(len(batch)):
        d = batch.item(i)
        base = random_valid_plan(d, rng)
        for kind in range(5):
            pl = [list(x) for x in base]
            s = int(rng.integers(d["p"]))
            if kind == 0 and len(pl[s]) > 1:                      # swap -> often deadlock
                k = int(rng.integers(len(pl[s]) - 1)); pl[s][k], pl[s][k + 1] = pl[s][k + 1], pl[s][k]
            elif kind == 1:                                        # drop an entry
                pl[s].pop(int(rng.integers(len(pl[s]))))
            elif kind == 2:                                        # extra F
                pl[s].insert(int(rng.integers(len(pl[s]) + 1)), 0)
            elif kind == 3:                                        # mix a B into a split stage
                pl[s][int(rng.integers(len(pl[s])))] = 1
            elif kind == 4:                                        # several random swaps
                for _ in range(3):
                    s2 = int(rng.integers(d["p"]))
                    if len(pl[s2]) > 1:
                        k = int(rng.integers(len(pl[s2]) - 1)); pl[s2][k], pl[s2][k + 1] = pl[s2][k + 1], pl[s2][k]
            plans.append(pl)
            inst_of.append(i)
    # memory-violating but valid plans: same plan, instance with a halved budget
    cut = InstanceBatch.concat([batch, batch.take(np.arange(len(batch)))])
    n0 = len(batch)
    cut.m_lim[n0:] = np.maximum(cut.m_f[n0:], cut.m_lim[n0:] // 3)
    for i in range(n0):
        plans.append(random_valid_plan(batch.item(i), rng))
        inst_of.append(n0 + i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(cut, ops, ln, inst_of)
    codes, lens = unpack_plans(ops, ln)
    seen = set()
    for j, i in enumerate(inst_of):
        w = compare_sim(O, cut.item(i), codes[j], lens[j], r, j, codes.shape[2])
        seen.add(w["status"])
    assert {0, 1, 2, 4} <= seen, seen


def test_simulate_edge_cases(O):
    """p = 1, m = 1, n_sub = 16, zero delays everywhere, p = 32 with one huge-bandwidth
    boundary, ZeRO-1 gate later than the pipeline start."""
    parts = [
        K.uniform_instance(1, 1, 1, 3, 4, 5),
        K.uniform_instance(1, 7, 1, 3, 4, 5, mlim_x1000=7000),
        K.uniform_instance(2, 1, 2, 1, 1, 1, lat=0, bw=0),
        K.uniform_instance(32, 40, 4, 7, 9, 16, lat=500, bw=300, n_sub=16, mlim_x1000=2000),
        K.uniform_instance(32, 3, 2, 5, 5, 5, lat=0, bw=100000, mlim_x1000=1000),
        K.uniform_instance(6, 9, 3, 11, 13, 17, lat=40, bw=25, t_dp=333, zero1=1, t_ag=1000),
    ]
    batch = InstanceBatch.concat(parts)
    plans, inst_of = [], []
    for i in range(len(batch)):
        ops, ln = PL.plans_host(batch, 3, seed=99 + i, i=i, stride=32)
        c, l_ = unpack_plans(ops, ln)
        for k in range(3):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2])


def test_bad_instances_and_overflow_guard(O):
    """Invalid records -> CPI_BAD_INSTANCE exactly when the oracle says so; a valid record
    whose horizon bound U >= 2^30 -> CPI_OVERFLOW (GPU int32 guard, reading Q21)."""
    batch = K.random_instances(60, seed=8, max_p=8, max_m=6)
    rng = np.random.default_rng(9)
    for i in range(len(batch)):
        k = int(rng.integers(6))
        s = int(rng.integers(batch.p[i]))
        if k == 0: batch.t_f[i, s] = 0
        elif k == 1: batch.m_w[i, s] -= 1
        elif k == 2: batch.m_lim[i, s] = batch.m_f[i, s] - 1
        elif k == 3:                                      # a block shorter than n_sub ticks (Q12)
            fld = ("t_f", "t_d", "t_w")[int(rng.integers(3))]
            getattr(batch, fld)[i, s] = batch.n_sub[i] - 1 if batch.n_sub[i] > 1 else 0
        elif k == 4 and batch.p[i] > 1: batch.lat_b[i, 0] = -1
        elif k == 5: batch.t_dp[i, s] = -5
    big = K.uniform_instance(4, 8, 2, 10**8, 10**8, 10**8)       # U = 9.6e9 >= 2^30
    batch = InstanceBatch.concat([batch, big])
    plans, inst_of = [], []
    for i in range(len(batch)):
        c, l_ = O.build_static("1f1b", int(batch.p[i]), int(batch.m[i]))
        plans.append([list(c[s, :l_[s]]) for s in range(int(batch.p[i]))])
        inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of[:-1]):
        w = O.simulate(batch.item(i), codes[j][:int(batch.p[i])], lens[j][:int(batch.p[i])])
        assert int(r["status"][j]) == w["status"], (j, int(r["status"][j]), w["status"])
    assert int(r["status"][-1]) == 16 and int(r["makespan"][-1]) == -1


def test_simulate_deterministic_and_ring_sizes(O):
    """Identical results for every arrival-ring size (fast path vs fix-up) and across runs."""
    batch = K.random_instances(40, seed=10, max_p=16, max_m=20)
    plans, inst_of = [], []
    for i in range(len(batch)):
        ops, ln = PL.plans_host(batch, 2, seed=5 + i, i=i, stride=16)
        c, l_ = unpack_plans(ops, ln)
        for k in range(2):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=16)
    ref = run_sim(batch, ops, ln, inst_of)
    for ring in (1, 2, 4, 64):
        r = run_sim(batch, ops, ln, inst_of, ring=ring)
        for k in ("makespan", "status", "peak_mem", "stage_stats", "t_start"):
            assert np.array_equal(r[k], ref[k]), (ring, k)


# ------------------------------------------------------------------------------------- greedy
def check_greedy(O, batch, g, idx):
    gc, gl = unpack_plans(g["ops"].view(np.uint32), g["len"].view(np.uint16))
    for i in idx:
        d = batch.item(i)
        w = O.greedy(d, timeline=True)
        p = d["p"]
        assert int(g["status"][i]) == w["status"], (i, int(g["status"][i]), w["status"])
        assert int(g["makespan"][i]) == w["makespan"], (i, int(g["makespan"][i]), w["makespan"])
        assert int(g["peak_mem"][i]) == w["peak_mem"], i
        assert np.array_equal(gl[i, :p], w["len"]), i
        L = int(w["len"][0])
        assert np.array_equal(gc[i, :p, :L], w["codes"][:, :L]), f"schedule differs at item {i}"
        if "stage_stats" in g:
            ss = g["stage_stats"][i]
            assert np.array_equal(ss[:p, 0], w["first_start"]) and np.array_equal(ss[:p, 1], w["last_end"])
            assert np.array_equal(ss[:p, 2], w["busy"]) and np.array_equal(ss[:p, 3], w["peak"])
        if "t_start" in g:
            assert np.array_equal(g["t_start"][i][:p, :L], w["t_start"][:, :L]), i


@pytest.mark.parametrize("max_p,seed", [(32, 11), (8, 12), (16, 13), (2, 14)])
def test_greedy_random_instances(O, max_p, seed):
    """Round-parallel greedy (two min-plus warp scans) == sequential Alg. 1, byte for byte."""
    batch = K.random_instances(300, seed=seed, max_p=max_p, max_m=20, intra_delay=True)
    inst = cp.Instances(batch)
    g = to_host(cp.greedy(inst, stats=True, timeline=True))
    check_greedy(O, batch, g, range(len(batch)))


def test_greedy_config3_sample(O):
    """Config 3 (1e5 instances; memory limit, DP overlap, ZeRO-1, n_sub, jitter): a 3000-instance
    slice end to end, every instance checked."""
    batch = K.greedy_batch(3000)
    inst = cp.Instances(batch)
    g = to_host(cp.greedy(inst, stats=True))
    check_greedy(O, batch, g, range(len(batch)))


def test_greedy_plans_resimulate(O):
    """Consistency: cp_simulate on cp_greedy's output reproduces its timeline."""
    batch = K.random_instances(100, seed=15, max_p=32, max_m=16)
    inst = cp.Instances(batch)
    g = cp.greedy(inst, stats=True, timeline=True)
    r = cp.simulate(inst, g["ops"], g["len"], stats=True, timeline=True, len_stride=g["t_start"].shape[2])
    torch.cuda.synchronize()
    for k in ("makespan", "status", "peak_mem", "stage_stats", "t_start"):
        assert torch.equal(r[k], g[k]), k


# ------------------------------------------------------------------------------------- sweep
def check_sweep(O, grid, keys, cm, pts):
    G, keep = O.to_or_grid(grid)
    for k in pts:
        key, cms = O.sweep_point(grid, int(k), G=G)
        want_key = cp.KEY_NONE if key == 2**64 - 1 else key
        assert int(keys[k]) == want_key, (k, int(keys[k]), want_key)
        assert list(cm[k]) == cms, (k, list(cm[k]), cms)


def test_sweep_tiny_grid(O):
    """Config 1 grid {0,.5,1,2}^2 with all 5 candidates, every point."""
    from workloads.core import Grid
    base = K.tiny(0, 0)
    r = [0, 50, 100, 200]
    grid = Grid(base=base, n_dc=2, pp_vals=[4], mb_vals=[8], lat=np.array(r), bw=np.array(r),
                mlim_x1000=np.array([1000, 2000]), tdp=np.array([0, 150]), cand_mask=0b11111)
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


def test_sweep_config2_every_point(O):
    """Config 2 (16 stages / 2 DCs / 32 mb, 64 x 64 latency x bandwidth): every point, each checked
    candidate by candidate."""
    grid = K.gpt16_grid()
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


def test_sweep_config5_sample_and_shards(O):
    """Config 5 (4 DCs, p 8-32, m 8-128, memory grid): 400 sampled points; shards over 1/2/4/8
    cost-balanced ranges assembled with MIN give byte-identical keys, and so do the rank shards --
    whose largest-n_mb greedy tasks run in launches of their own (DESIGN.md §7 Sweep) -- together
    with every candidate's makespan."""
    grid = K.full_sweep_grid()
    full, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    full_h = full.cpu().numpy()
    rng = np.random.default_rng(17)
    pts = np.concatenate([rng.choice(grid.n_points, 400, replace=False)])
    check_sweep(O, grid, full_h, cm.cpu().numpy(), pts)
    for world in (2, 4, 8):
        b = cp.sweep_partition(grid, world)
        acc = torch.full((grid.n_points,), cp.KEY_NONE, dtype=torch.int64, device="cuda")
        acc_r = acc.clone()
        acc_c = torch.full_like(cm, -1)
        for rk in range(world):
            kr, _ = cp.sweep_shard(grid, b[rk], b[rk + 1])
            acc = torch.minimum(acc, kr)
            kb, cb = cp.sweep_shard_rank(grid, rk, world, cand=True)   # blocked ownership
            acc_r = torch.minimum(acc_r, kb)
            acc_c = torch.maximum(acc_c, cb)                          # (not owned: -1)
        assert torch.equal(acc.cpu(), torch.from_numpy(full_h)), world
        assert torch.equal(acc_r.cpu(), torch.from_numpy(full_h)), ("rank shards", world)
        assert torch.equal(acc_c, cm), ("rank-shard candidate makespans", world)


def test_sweep_global_ring_fallback(O):
    """n_mb = 1024 with a budget that admits every microbatch in flight: the lead bound (1024 slots,
    256 KB of rings per warp) exceeds one block's shared memory, so the engine pass of that p-class
    runs with global-memory rings from the sweep workspace; greedy candidates fall back to it too.
    Every point and candidate against the oracle."""
    from workloads.core import Grid
    grid = Grid(base=K.uniform_instance(4, 8, 2, 100, 90, 80), n_dc=2, pp_vals=[2, 4], mb_vals=[1024],
                lat=np.array([0, 50]), bw=np.array([30]), mlim_x1000=np.array([600000]), tdp=np.array([0, 70]),
                cand_mask=0b111111)
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


# ------------------------------------------------------------------------------------- config 4 at full size
def test_config4_full_size_sampled(O):
    """Config 4 at BASELINE size (1e6 perturbed valid schedules, p=32, 4 DCs, m=64) in the bench
    launch configuration; 400 sampled schedules checked against the oracle, the GPU generator
    checked against the host generator, and the argmin key checked for consistency."""
    b = K.perturbed_instance()
    n = 1_000_000
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED)
    inst = cp.Instances(b)
    r = cp.simulate(inst, ops, ln, best=True)
    torch.cuda.synchronize()
    idx = np.random.default_rng(18).choice(n, 400, replace=False)
    h_ops, h_ln = PL.plans_host(b, 1, seed=K.PERTURB_SEED, id0=int(idx[0]))
    assert np.array_equal(ops[int(idx[0])].cpu().numpy().view(np.uint32), h_ops[0])
    ms = r["makespan"].cpu().numpy()
    st = r["status"].cpu().numpy()
    assert np.all(st == 0)
    sub_ops = ops[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint32)
    sub_ln = ln[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint16)
    codes, lens = unpack_plans(sub_ops, sub_ln)
    d = b.item(0)
    for j, i in enumerate(idx):
        w = O.simulate(d, codes[j], lens[j])
        assert (int(ms[i]), int(st[i])) == (w["makespan"], w["status"]), i
    bk = int(r["best_key"][0])
    assert (bk >> 32) == ms.min() and ms[bk & 0xFFFFFFFF] == ms.min()


def test_simulate_fast_path_invalid_and_overflow(O):
    """The one-item-per-warp fast path (k_sim32: p > 16, stride 32, no timeline) on valid,
    deadlocking, statically bad (counts / mixing), W-before-D, and memory-violating plans (which
    also overflow the shared-memory rings and go through the global-ring fix-up pass)."""
    rng = np.random.default_rng(19)
    big = K.random_instances(400, seed=20, max_p=32, max_m=12)
    keep = [i for i in range(len(big)) if big.p[i] >= 17][:70]
    batch = big.take(keep)
    plans, inst_of = [], []
    for i in range(len(batch)):
        d = batch.item(i)
        base = random_valid_plan(d, rng)
        for kind in range(7):
            pl = [list(x) for x in base]
            s = int(rng.integers(d["p"]))
            if kind == 1 and len(pl[s]) > 1:
                k = int(rng.integers(len(pl[s]) - 1)); pl[s][k], pl[s][k + 1] = pl[s][k + 1], pl[s][k]
            elif kind == 2:
                pl[s].pop(int(rng.integers(len(pl[s]))))
            elif kind == 3:
                pl[s].insert(int(rng.integers(len(pl[s]) + 1)), 0)
            elif kind == 4:
                pl[s][int(rng.integers(len(pl[s])))] = 1
            elif kind == 5 and 3 in pl[s]:                # move the first W to the front (W before its D)
                j = pl[s].index(3); pl[s].insert(0, pl[s].pop(j))
            elif kind == 6:
                for _ in range(4):
                    s2 = int(rng.integers(d["p"]))
                    if len(pl[s2]) > 1:
                        k = int(rng.integers(len(pl[s2]) - 1)); pl[s2][k], pl[s2][k + 1] = pl[s2][k + 1], pl[s2][k]
            plans.append(pl)
            inst_of.append(i)
    cut = InstanceBatch.concat([batch, batch.take(np.arange(len(batch)))])
    n0 = len(batch)
    cut.m_lim[n0:] = np.maximum(cut.m_f[n0:], cut.m_lim[n0:] // 3)
    for i in range(n0):
        plans.append(random_valid_plan(batch.item(i), rng))
        inst_of.append(n0 + i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(cut, ops, ln, inst_of, stats=True, timeline=False)
    codes, lens = unpack_plans(ops, ln)
    seen = set()
    for j, i in enumerate(inst_of):
        w = compare_sim(O, cut.item(i), codes[j], lens[j], r, j, codes.shape[2], timeline=False)
        seen.add(w["status"])
    assert {0, 1, 2, 4} <= seen, seen


def test_host_pipeline_matches_device_call():
    """cp.HostPipeline (chunked H2D / kernel / D2H overlap over pinned host buffers) returns the
    same per-schedule results and the same global best key as one device-resident cp_simulate."""
    b = K.perturbed_instance()
    n = 20_000
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED)
    inst = cp.Instances(b)
    ref = cp.simulate(inst, ops, ln, best=True)
    ops_h = ops.cpu().pin_memory(); ln_h = ln.cpu().pin_memory()
    ms_h = torch.empty(n, dtype=torch.int64).pin_memory()
    pk_h = torch.empty(n, dtype=torch.int32).pin_memory()
    st_h = torch.empty(n, dtype=torch.int32).pin_memory()
    pipe = cp.HostPipeline(inst, n, ops.shape[1], ops.shape[2], chunks=7)
    bk = pipe.run(ops_h, ln_h, ms_h, pk_h, st_h)
    torch.cuda.synchronize()
    assert torch.equal(ms_h, ref["makespan"].cpu()) and torch.equal(st_h, ref["status"].cpu())
    assert torch.equal(pk_h, ref["peak_mem"].cpu())
    assert int(bk[0]) == int(ref["best_key"][0])


@pytest.mark.parametrize("max_p,seed", [(32, 21), (16, 22), (8, 23), (3, 24)])
def test_greedy_fast_path_random_instances(O, max_p, seed):
    """cp_greedy without a timeline runs k_greedy_fast<W> (W = 8 / 16 / 32): byte-equal schedules,
    makespans, peaks and per-stage stats vs sequential Alg. 1 on random instances."""
    batch = K.random_instances(300, seed=seed, max_p=max_p, max_m=20, intra_delay=True)
    inst = cp.Instances(batch)
    g = to_host(cp.greedy(inst, stats=True))
    check_greedy(O, batch, g, range(len(batch)))


def test_fast_paths_ring_overflow_fixup(O):
    """Undersized ring hints force every fast-path item (k_sim32 / k_greedy_fast) through the
    stall -> overflow list -> global-ring fix-up pass; results must be unchanged."""
    b = K.perturbed_instance()
    ops, ln = PL.plans_device(b, 500, seed=K.PERTURB_SEED)
    inst = cp.Instances(b)
    ref = cp.simulate(inst, ops, ln, stats=True, best=True)
    for ring in (1, 3, 16):
        r = cp.simulate(inst, ops, ln, stats=True, best=True, ring=ring)
        for k in ("makespan", "status", "peak_mem", "stage_stats", "best_key"):
            assert torch.equal(r[k], ref[k]), (ring, k)
    batch = K.random_instances(200, seed=25, max_p=16, max_m=16)
    gi = cp.Instances(batch)
    gref = cp.greedy(gi, stats=True)
    for ring in (1, 2):
        g = cp.greedy(gi, stats=True, ring=ring)
        for k in ("makespan", "status", "peak_mem", "stage_stats", "ops", "len"):
            assert torch.equal(g[k], gref[k]), (ring, k)
    ms = ref["makespan"].cpu().numpy()
    c, l_ = unpack_plans(ops[:20].cpu().numpy().view(np.uint32), ln[:20].cpu().numpy().view(np.uint16))
    for i in range(20):
        assert ms[i] == O.simulate(b.item(0), c[i], l_[i])["makespan"]


def test_sweep_ring_tier_edges(O):
    """Greedy sweep tasks run in ring-size tiers by lead bound min(m, floor(M_L/m_f)) (<= 32,
    <= 64, rest; DESIGN.md §7 Sweep).  Memory scales chosen so the bound is exactly 31, 32, 33, 63,
    64, 65 and 96/128 at p = 16: every point and candidate checked against the oracle."""
    from workloads.core import Grid
    base = K.uniform_instance(16, 8, 2, 100, 120, 80)
    grid = Grid(base=base, n_dc=2, pp_vals=[16], mb_vals=[96, 128], lat=np.array([0, 150]), bw=np.array([0, 60]),
                mlim_x1000=np.array([1938, 2000, 2063, 3938, 4000, 4063, 8000]), tdp=np.array([0]),
                cand_mask=0b11111)
    leads = sorted({min(m, ((x * 16 * 2 + 500) // 1000) // 2) for m in (96, 128) for x in grid.mlim_x1000})
    assert leads == [31, 32, 33, 63, 64, 65, 96, 128], leads
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


def test_sweep_edge_grids(O):
    """Sweep grids with more DCs than stages (p = 2, 3 with 4 DCs), a ZeRO-1 base with allgather
    times, DP tails, and a candidate subset (1F1B + greedy n_sub = 2 only)."""
    from workloads.core import Grid
    base = K.uniform_instance(4, 8, 4, 30, 40, 20, zero1=1, t_ag=25)
    base.t_ag[0, :] = 25
    grid = Grid(base=base, n_dc=4, pp_vals=[2, 3, 4], mb_vals=[1, 5], lat=np.array([0, 45]), bw=np.array([0, 20, 70]),
                mlim_x1000=np.array([1000, 1700]), tdp=np.array([0, 90]), cand_mask=0b01010)
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


def test_generic_greedy_ring_overflow_fixup():
    """The generic engine's greedy (timeline requested) with an undersized ring must also hand
    over to the fix-up pass without changing a single decision."""
    batch = K.random_instances(150, seed=26, max_p=32, max_m=14)
    gi = cp.Instances(batch)
    ref = cp.greedy(gi, stats=True, timeline=True)
    g = cp.greedy(gi, stats=True, timeline=True, ring=1)
    for k in ("makespan", "status", "peak_mem", "stage_stats", "ops", "len", "t_start"):
        assert torch.equal(g[k], ref[k]), k


# ------------------------------------------------------------------------------------- static builders (NEXT 2)
@pytest.mark.parametrize("kind", ["gpipe", "1f1b", "zbh1"])
def test_build_static_matches_oracle_builders(O, kind):
    """cp_build_static (Q22, Q23, Q31) == the oracle's builders entry by entry, for p in 1..32 and
    m in 1..40 (m < p included), with stage_stride 32 > p and spare words: padding words and
    rows >= p are zero."""
    rng = np.random.default_rng({"gpipe": 40, "1f1b": 41, "zbh1": 42}[kind])
    n = 300
    batch = K.random_instances(n, seed=int(rng.integers(1 << 30)), max_p=32, max_m=40)
    inst = cp.Instances(batch)
    words = (3 * 40 + 15) // 16 + 2
    ops, ln = cp.build_static(kind, inst, stage_stride=32, words=words)
    torch.cuda.synchronize()
    codes, lens = unpack_plans(ops.cpu().numpy().view(np.uint32), ln.cpu().numpy().view(np.uint16))
    for i in range(n):
        p, m = int(batch.p[i]), int(batch.m[i])
        c, l_ = O.build_static(kind, p, m)
        assert np.array_equal(lens[i, :p], l_), i
        assert not lens[i, p:].any() and not codes[i, p:].any(), i
        for s in range(p):
            assert np.array_equal(codes[i, s, :l_[s]], c[s, :l_[s]]), (i, s)
            assert not codes[i, s, l_[s]:].any(), (i, s)


def test_simulate_zbh1_plans(O):
    """GPU-built ZB-H1 plans through cp_simulate (the k_sim32 fast path at stage_stride 32 and the
    generic engine with a timeline) == the oracle simulating its own ZB-H1 plans."""
    batch = K.random_instances(200, seed=43, max_p=32, max_m=24, intra_delay=True)
    batch.n_sub[:] = 1                                  # ZB-H1 holds whole W blocks
    inst = cp.Instances(batch)
    ops, ln = cp.build_static("zbh1", inst, stage_stride=32)
    for timeline in (False, True):
        r = to_host(cp.simulate(inst, ops, ln, stats=True, timeline=timeline))
        torch.cuda.synchronize()
        for i in range(len(batch)):
            d = batch.item(i)
            c, l_ = O.build_static("zbh1", d["p"], d["m"])
            compare_sim(O, d, c, l_, r, i, c.shape[1], timeline=timeline)


def test_sweep_six_candidates(O):
    """Sweep with all six candidates (ZB-H1 = candidate 5, Q30/Q31) over delays, memory budgets
    below and above the 1F1B budget and DP tails; every point and candidate vs the oracle."""
    from workloads.core import Grid
    base = K.uniform_instance(6, 8, 3, 90, 110, 70)
    grid = Grid(base=base, n_dc=3, pp_vals=[2, 6], mb_vals=[3, 8, 13], lat=np.array([0, 120]), bw=np.array([0, 45, 200]),
                mlim_x1000=np.array([700, 1000, 1600]), tdp=np.array([0, 80]), cand_mask=0b111111)
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    assert cm.shape[1] == 6
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


# ------------------------------------------------------------------------------------- Wave pattern (NEXT 1)
def _wave_batch(n, seed, max_p, max_m, combined_frac=0.25):
    from workloads.wave import pack_wave_plans, random_wave_plan
    rng = np.random.default_rng(seed)
    batch = K.random_instances(n, seed=seed, max_p=max_p, max_m=max_m, intra_delay=True)
    plans = [random_wave_plan(int(batch.p[i]), int(batch.m[i]), int(batch.n_sub[i]), rng,
                              combined=bool(rng.random() < combined_frac)) for i in range(n)]
    ops, ln = pack_wave_plans(plans, stage_stride=32)
    return batch, plans, ops, ln


def check_wave(O, batch, plans, r, timeline):
    for i, pl in enumerate(plans):
        d = batch.item(i)
        w = O.simulate_wave(d, pl, timeline=timeline)
        p = d["p"]
        assert int(r["status"][i]) == w["status"], (i, int(r["status"][i]), w["status"])
        assert int(r["makespan"][i]) == w["makespan"], (i, int(r["makespan"][i]), w["makespan"])
        assert int(r["peak_mem"][i]) == w["peak_mem"], i
        if w["makespan"] >= 0:
            ss = r["stage_stats"][i]
            assert np.array_equal(ss[:p, 0], w["first_start"]) and np.array_equal(ss[:p, 1], w["last_end"]), i
            assert np.array_equal(ss[:p, 2], w["busy"]) and np.array_equal(ss[:p, 3], w["peak"]), i
            if timeline:
                for s in range(p):
                    L = len(pl[s])
                    assert np.array_equal(r["t_start"][i][s, :L], w["t_start"][s, :L]), (i, s)


@pytest.mark.parametrize("max_p,seed", [(32, 50), (8, 51), (3, 52)])
def test_simulate_wave_random_plans(O, max_p, seed):
    """Wave plans (reading Q32) through cp_simulate (k_wave32) == the oracle's Wave DAG, status,
    makespan, peak, per-stage stats and every start tick; split and combined plans, n_sub 1-4,
    delays, ZeRO-1, DP tails."""
    batch, plans, ops, ln = _wave_batch(120, seed, max_p, 10)
    inst = cp.Instances(batch)
    o, l_ = plans_to_device(ops, ln)
    r = to_host(cp.simulate(inst, o, l_, stats=True, timeline=True, wave=True))
    check_wave(O, batch, plans, r, timeline=True)


def test_simulate_wave_ring_fixup_and_invalid(O):
    """A 1-slot first-pass ring forces the second pass (rings of n_mb slots) without changing any
    result; corrupted plans (counts, W before its D, stray chunk bits) report BAD_PLAN and a turn-
    around taken in the wrong order deadlocks, as in the oracle."""
    batch, plans, ops, ln = _wave_batch(80, 53, 16, 12, combined_frac=0.0)
    rng = np.random.default_rng(54)
    for i in range(0, 80, 4):
        s = int(rng.integers(batch.p[i]))
        k = int(rng.integers(4))
        row = plans[i][s]
        if k == 0:
            row[-1] = row[-1] ^ 4                        # W of the other chunk: counts break
        elif k == 1:
            j = row.index(next(x for x in row if (x & 3) == 3)); row.insert(0, row.pop(j))   # W first
        elif k == 2:
            row[0] = row[0] | 8                          # stray bit
        elif batch.p[i] > 1:
            pl = plans[i][int(batch.p[i]) - 1]           # last stage: F1 before F0 -> cycle
            a, b = pl.index(0), pl.index(4); pl[a], pl[b] = 4, 0
    from workloads.wave import pack_wave_plans
    ops, ln = pack_wave_plans(plans, stage_stride=32)
    inst = cp.Instances(batch)
    o, l_ = plans_to_device(ops, ln)
    ref = to_host(cp.simulate(inst, o, l_, stats=True, wave=True))
    small = to_host(cp.simulate(inst, o, l_, stats=True, wave=True, ring=1))
    for k in ("status", "makespan", "peak_mem", "stage_stats"):
        assert np.array_equal(ref[k], small[k]), k
    check_wave(O, batch, plans, ref, timeline=False)


def test_wave_bench_size_sampled(O):
    """The bench's Wave workload (p=32, 4 DCs, m=32; device-generated plans == host-generated plans)
    in the bench launch configuration; 30 sampled plans checked against the oracle."""
    from workloads.wave import unpack_wave_plans
    b = K.wave_instance()
    n = 20_000
    ops, ln = PL.wave_plans_device(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32)
    r = to_host(cp.simulate(cp.Instances(b), ops, ln, stats=True, best=True, wave=True))
    idx = np.random.default_rng(19).choice(n, 30, replace=False)
    hops, hln = PL.wave_plans_host(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32)
    assert np.array_equal(hops.view(np.int32), ops.cpu().numpy()) and np.array_equal(hln.view(np.int16), ln.cpu().numpy())
    codes, lens = unpack_wave_plans(hops, hln)
    d = b.item(0)
    for i in idx:
        w = O.simulate_wave(d, [list(codes[i, s, :lens[i, s]]) for s in range(32)])
        assert int(r["status"][i]) == w["status"] and int(r["makespan"][i]) == w["makespan"], i
        assert int(r["peak_mem"][i]) == w["peak_mem"], i
    ok = r["status"] == 0
    best = int(r["best_key"][0])
    assert best >> 32 == int(r["makespan"][ok].min())


# ------------------------------------------------------------------------------------- Loop pattern (NEXT 1)
def _loop_batch(n, seed, max_p, max_m, combined_frac=0.25):
    from workloads.wave import pack_wave_plans, random_loop_plan
    rng = np.random.default_rng(seed)
    batch = K.random_instances(n, seed=seed, max_p=max_p, max_m=max_m, intra_delay=True)
    for i in range(n):                                   # wrap links p-1 -> 0 / 0 -> p-1 (boundary p-1)
        p = int(batch.p[i])
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            getattr(batch, fld)[i, p - 1] = int(rng.integers(0, 300)) if rng.random() < 0.7 else 0
    plans = [random_loop_plan(int(batch.p[i]), int(batch.m[i]), int(batch.n_sub[i]), rng,
                              combined=bool(rng.random() < combined_frac)) for i in range(n)]
    ops, ln = pack_wave_plans(plans, stage_stride=32)
    return batch, plans, ops, ln


def check_loop(O, batch, plans, r, timeline):
    for i, pl in enumerate(plans):
        d = batch.item(i)
        w = O.simulate_loop(d, pl, timeline=timeline)
        p = d["p"]
        assert int(r["status"][i]) == w["status"], (i, int(r["status"][i]), w["status"])
        assert int(r["makespan"][i]) == w["makespan"], (i, int(r["makespan"][i]), w["makespan"])
        assert int(r["peak_mem"][i]) == w["peak_mem"], i
        if w["makespan"] >= 0:
            ss = r["stage_stats"][i]
            assert np.array_equal(ss[:p, 0], w["first_start"]) and np.array_equal(ss[:p, 1], w["last_end"]), i
            assert np.array_equal(ss[:p, 2], w["busy"]) and np.array_equal(ss[:p, 3], w["peak"]), i
            if timeline:
                for s in range(p):
                    L = len(pl[s])
                    assert np.array_equal(r["t_start"][i][s, :L], w["t_start"][s, :L]), (i, s)


@pytest.mark.parametrize("max_p,seed", [(32, 60), (8, 61), (2, 62)])
def test_simulate_loop_random_plans(O, max_p, seed):
    """Loop plans (reading Q33: wrap-around links at boundary p-1) through cp_simulate == the oracle's
    Loop DAG: status, makespan, peak, per-stage stats and every start tick."""
    batch, plans, ops, ln = _loop_batch(120, seed, max_p, 10)
    o, l_ = plans_to_device(ops, ln)
    r = to_host(cp.simulate(cp.Instances(batch), o, l_, stats=True, timeline=True, loop=True))
    check_loop(O, batch, plans, r, timeline=True)


def test_simulate_loop_ring_fixup(O):
    """1-slot first-pass rings force the second pass for Loop plans without changing any result."""
    batch, plans, ops, ln = _loop_batch(80, 63, 16, 12, combined_frac=0.0)
    inst = cp.Instances(batch)
    o, l_ = plans_to_device(ops, ln)
    ref = to_host(cp.simulate(inst, o, l_, stats=True, loop=True))
    small = to_host(cp.simulate(inst, o, l_, stats=True, loop=True, ring=1))
    for k in ("status", "makespan", "peak_mem", "stage_stats"):
        assert np.array_equal(ref[k], small[k]), k
    check_loop(O, batch, plans, ref, timeline=False)


def test_loop_bench_size_sampled(O):
    """The bench's Loop workload (p=32, 4 DCs, m=32, cross-DC wrap links; device plans == host
    plans) in the bench launch configuration; 30 sampled plans checked against the oracle."""
    from workloads.wave import unpack_wave_plans
    b = K.loop_instance()
    n = 20_000
    ops, ln = PL.wave_plans_device(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32, loop=True)
    r = to_host(cp.simulate(cp.Instances(b), ops, ln, stats=True, best=True, loop=True))
    hops, hln = PL.wave_plans_host(32, 32, 1, n, seed=K.PERTURB_SEED ^ 0x3A, q=1, stride=32, loop=True)
    assert np.array_equal(hops.view(np.int32), ops.cpu().numpy()) and np.array_equal(hln.view(np.int16), ln.cpu().numpy())
    codes, lens = unpack_wave_plans(hops, hln)
    d = b.item(0)
    for i in np.random.default_rng(20).choice(n, 30, replace=False):
        w = O.simulate_loop(d, [list(codes[i, s, :lens[i, s]]) for s in range(32)])
        assert int(r["status"][i]) == w["status"] and int(r["makespan"][i]) == w["makespan"], i
        assert int(r["peak_mem"][i]) == w["peak_mem"], i
    ok = r["status"] == 0
    assert int(r["best_key"][0]) >> 32 == int(r["makespan"][ok].min())


def test_build_iv1f1b_and_simulate_loop(O):
    """cp_build_static(IV1F1B) (reading Q34) == the oracle's builder entry by entry (items with
    m % p != 0 get all-zero rows), and the built plans through cp_simulate(loop) == the oracle's
    Loop simulation of its own IV1F1B plans, with delays on every link including the wraps."""
    from workloads.wave import unpack_wave_plans
    rng = np.random.default_rng(44)
    batch = K.random_instances(150, seed=45, max_p=16, max_m=4, intra_delay=True)
    for i in range(150):
        p = int(batch.p[i])
        batch.m[i] = p * int(rng.integers(1, 4)) if i % 10 else p + 1 if p > 1 else 1    # a few m % p != 0
        batch.n_sub[i] = 1
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            getattr(batch, fld)[i, p - 1] = int(rng.integers(0, 200))
    inst = cp.Instances(batch)
    ops, ln = cp.build_static("iv1f1b", inst, stage_stride=32)
    r = to_host(cp.simulate(inst, ops, ln, stats=True, timeline=True, loop=True))
    codes, lens = unpack_wave_plans(ops.cpu().numpy().view(np.uint32), ln.cpu().numpy().view(np.uint16))
    for i in range(150):
        d = batch.item(i)
        p, m = d["p"], d["m"]
        if m % p:
            assert not lens[i].any() and not codes[i].any(), i
            continue
        c, l_ = O.build_static("iv1f1b", p, m)
        assert np.array_equal(lens[i, :p], l_), i
        for s in range(p):
            assert np.array_equal(codes[i, s, :l_[s]], c[s, :l_[s]]), (i, s)
        w = O.simulate_loop(d, c, l_, timeline=True)
        assert int(r["status"][i]) == w["status"] and int(r["makespan"][i]) == w["makespan"], i
        for s in range(p):
            assert np.array_equal(r["t_start"][i][s, :l_[s]], w["t_start"][s, :l_[s]]), (i, s)


def test_build_zbv_and_simulate_wave(O):
    """cp_build_static(ZBV) (reading Q35; one warp per item, a round per unit tick) == the oracle's
    builder entry by entry, for p up to 32 and m on both sides of 2p (row capacity exactly 6 max_mb),
    and the built plans through cp_simulate(wave) == the oracle's Wave simulation of its own ZB-V
    plans, start tick by start tick, with delays on every link."""
    from workloads.wave import unpack_wave_plans
    rng = np.random.default_rng(47)
    n = 120
    batch = K.random_instances(n, seed=48, max_p=32, max_m=4, intra_delay=True)
    for i in range(n):
        p = int(batch.p[i])
        batch.m[i] = int(rng.integers(1, 2 * p)) if i % 3 == 0 else int(rng.integers(2 * p, 4 * p + 3))
        batch.n_sub[i] = 1
    batch.m[int(np.argmax(batch.p[:n]))] = 64                         # the widest item at m = 64
    inst = cp.Instances(batch)
    ops, ln = cp.build_static("zbv", inst, stage_stride=32)
    assert ops.shape[1] == (6 * int(batch.m[:n].max()) + 7) // 8
    r = to_host(cp.simulate(inst, ops, ln, stats=True, timeline=True, wave=True))
    codes, lens = unpack_wave_plans(ops.cpu().numpy().view(np.uint32), ln.cpu().numpy().view(np.uint16))
    for i in range(n):
        d = batch.item(i)
        p, m = d["p"], d["m"]
        c, l_ = O.build_static("zbv", p, m)
        assert np.array_equal(lens[i, :p], l_) and not lens[i, p:].any(), i
        assert not codes[i, p:].any() and not codes[i, :, 6 * m:].any(), i
        for s in range(p):
            assert np.array_equal(codes[i, s, :l_[s]], c[s, :l_[s]]), (i, s)
        w = O.simulate_wave(d, c, l_, timeline=True)
        assert int(r["status"][i]) == w["status"] and int(r["makespan"][i]) == w["makespan"], i
        for s in range(p):
            assert np.array_equal(r["t_start"][i][s, :l_[s]], w["t_start"][s, :l_[s]]), (i, s)


def test_exact_search_matches_oracle_enumeration(O):
    """cp_exact (NEXT 3) == the oracle's exhaustive optimum (or_enumerate_opt) on random tiny
    instances with delays, memory budgets, DP tails and ZeRO-1: same makespan and the same plan,
    entry by entry (both return the first optimum in product order).  Limits: n_sub != 1, m > 8 or a
    too-small max_plans give CPI_OVERFLOW; the plan through cp_simulate reproduces the makespan."""
    from workloads.core import unpack_plans
    rng = np.random.default_rng(51)
    n = 24
    batch = K.random_instances(n, seed=52, max_p=3, max_m=3, intra_delay=True)
    batch.n_sub[:n] = 1
    for i in range(n):
        p = int(batch.p[i])
        batch.m_lim[i, :p] = batch.m_f[i, :p] * int(rng.integers(1, 4))       # 1-3 activations in flight
    batch.n_sub[n - 1] = 2                                                  # unsupported -> overflow
    inst = cp.Instances(batch)
    r = cp.exact(inst)
    ms, st = r["makespan"].cpu().numpy(), r["status"].cpu().numpy()
    codes, lens = unpack_plans(r["ops"].cpu().numpy().view(np.uint32), r["len"].cpu().numpy().view(np.uint16))
    for i in range(n - 1):
        d = batch.item(i)
        e = O.enumerate_opt(d)
        assert e["evaluated"] >= 0, i
        if e["makespan"] < 0:
            assert st[i] == 1 and ms[i] == -1, i                           # every plan deadlocks
            continue
        assert st[i] == 0 and ms[i] == e["makespan"], (i, ms[i], e["makespan"])
        p = d["p"]
        for s in range(p):
            assert np.array_equal(codes[i, s, :lens[i, s]], e["codes"][s, :e["len"][s]]), (i, s)
    assert st[n - 1] == 16 and ms[n - 1] == -1
    sim = cp.simulate(inst, r["ops"][: n - 1], r["len"][: n - 1], inst_of=torch.arange(n - 1, dtype=torch.int32,
                                                                                     device="cuda"))
    ok = st[: n - 1] == 0
    assert np.array_equal(sim["makespan"].cpu().numpy()[ok], ms[: n - 1][ok])
    small = cp.exact(inst, max_plans=2)
    assert (small["status"].cpu().numpy()[:n - 1][ok] == 16).any()


def test_exact_search_bounds_greedy(O):
    """Beyond the oracle's reach (p = 3, m = 4 and p = 4, m = 3: up to ~10^7 plans): the optimum is a
    valid plan (oracle re-simulation gives the same makespan), and it is <= the greedy's and the
    static 1F1B's makespan (the optimality sandwich of SPEC.md:547)."""
    from workloads.core import unpack_plans
    parts = []
    for (p, m, lat, bw) in ((3, 4, 0, 0), (3, 4, 120, 60), (4, 3, 0, 0), (4, 3, 150, 40)):
        parts.append(K.uniform_instance(p, m, 2, 100, 100, 100, lat=lat, bw=bw, mlim_x1000=1000))
    from workloads.core import InstanceBatch
    batch = InstanceBatch.concat(parts)
    inst = cp.Instances(batch)
    r = cp.exact(inst)
    g = cp.greedy(inst)
    ms, st = r["makespan"].cpu().numpy(), r["status"].cpu().numpy()
    codes, lens = unpack_plans(r["ops"].cpu().numpy().view(np.uint32), r["len"].cpu().numpy().view(np.uint16))
    for i in range(len(parts)):
        d = batch.item(i)
        assert st[i] == 0
        assert O.simulate(d, codes[i, :d["p"]], lens[i, :d["p"]])["makespan"] == ms[i]
        assert ms[i] <= int(g["makespan"][i])
        assert ms[i] <= O.simulate(d, *O.build_static("1f1b", d["p"], d["m"]))["makespan"]
    # a warm start from the greedy's makespan (n_sub = 1: one of the enumerated plans) changes nothing
    w = cp.exact(inst, upper=g["makespan"])
    assert torch.equal(w["makespan"], r["makespan"]) and torch.equal(w["ops"], r["ops"])
    assert torch.equal(w["status"], r["status"])
    # an upper bound no plan reaches reports DEADLOCK (include/crosspipe.h)
    lo = cp.exact(inst, upper=r["makespan"] - 1)
    assert (lo["status"].cpu().numpy() == 1).all()


def test_two_chunk_plans_at_the_size_limit(O):
    """Wave / Loop plans at the GPU limit n_mb = 256 (p = 32, 1536 entries per row: the first pass's
    8-slot rings and the second pass's 256-slot rings in shared memory), ZB-V built at that size, all
    against the oracle; n_mb = 257 is refused with CP_EUNSUPPORTED (include/crosspipe.h)."""
    from workloads.wave import unpack_wave_plans
    for loop in (False, True):
        b = K.uniform_instance(32, 256, 4, 100, 100, 100, lat=100, bw=50, mlim_x1000=10**6)
        if loop:
            b.lat_f[0, 31], b.bw_f[0, 31], b.lat_b[0, 31], b.bw_b[0, 31] = 100, 50, 100, 50
        inst = cp.Instances(b)
        ops, ln = PL.wave_plans_device(32, 256, 1, 3, seed=61, stride=32, loop=loop)
        r = to_host(cp.simulate(inst, ops, ln, stats=True, wave=not loop, loop=loop))
        codes, lens = unpack_wave_plans(ops.cpu().numpy().view(np.uint32), ln.cpu().numpy().view(np.uint16))
        sim = O.simulate_loop if loop else O.simulate_wave
        for i in range(3):
            rows = [list(codes[i, s, :lens[i, s]]) for s in range(32)]
            w = sim(b.item(0), rows)
            assert int(r["status"][i]) == w["status"] and int(r["makespan"][i]) == w["makespan"], (loop, i)
    vb = K.uniform_instance(32, 256, 4, 100, 100, 100, m_f=1, m_d=0, m_w=-1, lat=100, bw=50, mlim_x1000=10**6)
    vinst = cp.Instances(vb)
    vo, vl = cp.build_static("zbv", vinst, stage_stride=32)
    rv = cp.simulate(vinst, vo, vl, wave=True)
    cz, lz = O.build_static("zbv", 32, 256)
    codes, lens = unpack_wave_plans(vo.cpu().numpy().view(np.uint32), vl.cpu().numpy().view(np.uint16))
    for s in range(32):
        assert np.array_equal(codes[0, s, :lens[0, s]], cz[s, :lz[s]]), s
    assert int(rv["makespan"][0]) == O.simulate_wave(vb.item(0), cz, lz)["makespan"]
    big = K.uniform_instance(32, 257, 4, 100, 100, 100, mlim_x1000=10**6)
    bo, bl = PL.wave_plans_device(32, 257, 1, 1, seed=62, stride=32)
    with pytest.raises(RuntimeError):
        cp.simulate(cp.Instances(big), bo, bl, wave=True)


def test_bubble_ratios(O):
    """cp.bubble_ratios (reading Q7) from the GPU stage stats == the ratios formed
    from the oracle's per-stage first / last / busy / makespan; SPEC.md:544 acceptance 1: 1F1B p = 4,
    m = 8, t_f = 1, t_d + t_w = 2, zero delay -> stage-0 ratio 9/33."""
    from tests.helpers_independent import bubble
    batch = K.random_instances(60, seed=71, max_p=32, max_m=6, intra_delay=True)
    inst = cp.Instances(batch)
    g = cp.greedy(inst, stats=True)
    loc, glo = cp.bubble_ratios(g, torch.from_numpy(batch.p[:60].astype(np.int64)).cuda())
    loc, glo = loc.cpu().numpy(), glo.cpu().numpy()
    for i in range(60):
        d = batch.item(i)
        r = O.greedy(d)
        if r["status"] & ~2:
            assert np.isnan(glo[i]).all(); continue
        for s in range(d["p"]):
            el, eg = bubble(r["first_start"][s], r["last_end"][s], r["busy"][s], r["makespan"])
            assert abs(glo[i, s] - eg) < 1e-12 and (abs(loc[i, s] - el) < 1e-12 or (np.isnan(loc[i, s]) and el != el)), (i, s)
    d = K.uniform_instance(4, 8, 1, 1, 1, 1, mlim_x1000=10**6)
    c, l_ = O.build_static("1f1b", 4, 8)
    o, l2 = plans_to_device(*codes_list_to_packed([[list(c[s, :l_[s]]) for s in range(4)]], stride=4))
    r = cp.simulate(cp.Instances(d), o, l2, stats=True)
    loc, glo = cp.bubble_ratios(r, 4)
    assert int(r["makespan"][0]) == 33 and abs(float(glo[0, 0]) - 9 / 33) < 1e-9


def test_e1_grid_every_point(O):
    """The E1 delay-sensitivity grid of PAPER.md §5.1 (4 stages / 2 DCs / 8 microbatches, T_lat/T_F x
    T_bw/T_F on 33 x 33 values in [0, 4], six candidates) -- every point and every candidate against
    the oracle (the table `tools/e1_grid.py` reports)."""
    grid = K.e1_grid()
    keys, cm = cp.sweep_shard(grid, cand=True)
    torch.cuda.synchronize()
    check_sweep(O, grid, keys.cpu().numpy(), cm.cpu().numpy(), range(grid.n_points))


def test_large_n_sub_greedy_and_simulate(O):
    """n_sub up to the GPU limit CP_MAX_SUB = 16 (W blocks in up to 16 sub-blocks; reading Q12: every
    sub-block >= 1 tick): the greedy's plans and makespans, and cp_simulate of random valid plans with
    those n_sub, against the oracle (the random-instance tests stop at n_sub = 4)."""
    batch = K.random_instances(48, seed=91, max_p=12, max_m=6, intra_delay=True)
    rng = np.random.default_rng(92)
    for i in range(48):
        ns = int(rng.choice([5, 8, 16]))
        p = int(batch.p[i])
        batch.n_sub[i] = ns
        for fld in ("t_f", "t_d", "t_w"):
            getattr(batch, fld)[i, :p] = np.maximum(getattr(batch, fld)[i, :p], ns)
    inst = cp.Instances(batch)
    g = to_host(cp.greedy(inst, stats=True))
    gc, gl = unpack_plans(g["ops"].view(np.uint32), g["len"].view(np.uint16))
    for i in range(48):
        d = batch.item(i)
        w = O.greedy(d)
        assert int(g["status"][i]) == w["status"] and int(g["makespan"][i]) == w["makespan"], i
        if w["makespan"] >= 0:
            for s in range(d["p"]):
                assert list(gc[i, s, :gl[i, s]]) == list(w["codes"][s, :w["len"][s]]), (i, s)
    plans, inst_of = [], []
    for i in range(48):
        ops, ln = PL.plans_host(batch, 2, seed=9300 + i, i=i, stride=32)
        c, l_ = unpack_plans(ops, ln)
        for k in range(2):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    r = run_sim(batch, ops, ln, inst_of, stats=True, timeline=False)
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2], timeline=False)
