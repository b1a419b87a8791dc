"""GPU parity at the edges of the round-2 first pass (k_chunk32f, chunk_fast.cu) against the oracle.

The first pass takes items with n_sub = 1 and n_mb <= 127 (byte counts) and lists everything it does
not finish for the exact second pass (k_sim32 for UD, k_chunk32 for Wave / Loop).  These tests mix,
in one batch, items on both sides of every boundary -- n_mb 126..129, n_sub 1 and 2, stage counts
that shrink and grow from item to item (ring columns a larger item wrote must not leak into a smaller
one), 2-slot rings that force most items into the second pass -- and compare every item with the
oracle: status, makespan, peak memory and every stage's first / last / busy / peak.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from tests.gpu_util import codes_list_to_packed, compare_sim, plans_to_device, to_host  # noqa: E402
from workloads import configs as K, plans as PL, unpack_plans  # noqa: E402


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def _ud_batch(seed):
    """Instances around the first pass's limits, stage counts alternating large / small."""
    shapes = [(32, 127, 1), (17, 128, 1), (32, 126, 1), (24, 129, 1), (18, 40, 2), (32, 127, 2),
              (20, 8, 1), (32, 64, 1), (17, 127, 1), (31, 100, 1), (19, 1, 1), (32, 128, 1)]
    b = K.random_instances(len(shapes), seed=seed, max_p=32, max_m=8)
    rng = np.random.default_rng(seed)
    for i, (p, m, ns) in enumerate(shapes):
        for fld in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "t_dp", "t_ag", "lat_f", "bw_f", "lat_b", "bw_b"):
            getattr(b, fld)[i, :] = 0
        b.p[i], b.m[i], b.n_sub[i], b.n_dc[i] = p, m, ns, int(rng.integers(1, 5))
        for fld in ("t_f", "t_d", "t_w"):
            getattr(b, fld)[i, :p] = np.maximum(rng.integers(1, 200, size=p), ns)
        mf = rng.integers(1, 5, size=p)
        md = -rng.integers(0, mf + 1)
        b.m_f[i, :p], b.m_d[i, :p], b.m_w[i, :p] = mf, md, -mf - md
        b.m_lim[i, :p] = mf * rng.integers(2, 40, size=p)
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            getattr(b, fld)[i, :p - 1] = rng.integers(0, 300, size=p - 1) * (rng.random(p - 1) < 0.5)
        if i % 3 == 0:
            b.zero1[i] = 1
            b.t_ag[i, :p] = rng.integers(0, 300, size=p)
        if i % 4 == 1:
            b.t_dp[i, :p] = rng.integers(0, 500, size=p)
    return b


@pytest.mark.parametrize("ring", [None, 1])
def test_ud_first_pass_boundaries(O, ring):
    """UD plans (the config-4 path: stats, no timeline, stage stride 32) on both sides of n_mb = 127
    and n_sub = 1, p from 17 to 32 in alternating order, 3 random valid plans each; with ring=1 the
    first pass runs 2-slot rings and lists most items.  Every item equals the oracle."""
    batch = _ud_batch(7 if ring is None else 8)
    plans, inst_of = [], []
    for i in range(len(batch)):
        ops, ln = PL.plans_host(batch, 3, seed=500 + i, i=i, q=int(i % 4), stride=32)
        c, l_ = unpack_plans(ops, ln)
        for k in range(3):
            plans.append([list(c[k, s, :l_[k, s]]) for s in range(int(batch.p[i]))])
            inst_of.append(i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    inst = cp.Instances(batch)
    o, l_ = plans_to_device(ops, ln)
    io = torch.from_numpy(np.asarray(inst_of, dtype=np.int32)).cuda()
    r = to_host(cp.simulate(inst, o, l_, io, stats=True, ring=ring))
    codes, lens = unpack_plans(ops, ln)
    for j, i in enumerate(inst_of):
        compare_sim(O, batch.item(i), codes[j], lens[j], r, j, codes.shape[2], timeline=False)
    assert np.all(r["status"] == 0)


def _two_chunk(loop, seed):
    from workloads.wave import pack_wave_plans, random_loop_plan, random_wave_plan
    shapes = [(32, 127), (5, 128), (9, 126), (2, 129), (4, 127), (1 if not loop else 2, 60), (17, 128), (3, 4)]
    rng = np.random.default_rng(seed)
    b = K.random_instances(len(shapes), seed=seed, max_p=32, max_m=8, intra_delay=True)
    for i, (p, m) in enumerate(shapes):
        b.p[i], b.m[i], b.n_sub[i] = p, m, 1
        for fld in ("t_f", "t_d", "t_w"):
            getattr(b, fld)[i, :p] = rng.integers(1, 200, size=p)
        mf = rng.integers(1, 5, size=p)
        md = -rng.integers(0, mf + 1)
        b.m_f[i, :p], b.m_d[i, :p], b.m_w[i, :p] = mf, md, -mf - md
        b.m_lim[i, :p] = mf * rng.integers(1, 400, size=p)
        for fld in ("lat_f", "bw_f", "lat_b", "bw_b"):
            getattr(b, fld)[i, :p] = rng.integers(0, 300, size=p) * (rng.random(p) < 0.6)
            if not loop and p > 0:
                getattr(b, fld)[i, p - 1] = 0
    gen = random_loop_plan if loop else random_wave_plan
    plans = [gen(int(b.p[i]), int(b.m[i]), 1, rng, combined=bool(i % 4 == 3)) for i in range(len(shapes))]
    ops, ln = pack_wave_plans(plans, stage_stride=32)
    return b, plans, ops, ln


@pytest.mark.parametrize("loop", [False, True], ids=["wave", "loop"])
def test_two_chunk_first_pass_boundaries(O, loop):
    """Wave / Loop plans on both sides of n_mb = 127 (the byte counts' limit), p from 1 (Wave) / 2
    (Loop) to 32 in alternating order, split and combined plans: every item equals the oracle, and
    the 2-slot-ring run (most items listed for the exact pass) gives the same results."""
    b, plans, ops, ln = _two_chunk(loop, 61 if loop else 60)
    inst = cp.Instances(b)
    o, l_ = plans_to_device(ops, ln)
    kw = {"loop": True} if loop else {"wave": True}
    r = to_host(cp.simulate(inst, o, l_, stats=True, **kw))
    small = to_host(cp.simulate(inst, o, l_, stats=True, ring=1, **kw))
    for k in ("status", "makespan", "peak_mem", "stage_stats"):
        assert np.array_equal(r[k], small[k]), k
    for i, pl in enumerate(plans):
        d = b.item(i)
        w = (O.simulate_loop if loop else O.simulate_wave)(d, pl)
        p = d["p"]
        assert int(r["status"][i]) == w["status"], (i, int(r["status"][i]), w["status"])
        assert int(r["makespan"][i]) == w["makespan"], (i, int(r["makespan"][i]), w["makespan"])
        assert int(r["peak_mem"][i]) == w["peak_mem"], i
        if w["makespan"] >= 0:
            ss = r["stage_stats"][i]
            assert np.array_equal(ss[:p, 0], w["first_start"]) and np.array_equal(ss[:p, 1], w["last_end"]), i
            assert np.array_equal(ss[:p, 2], w["busy"]) and np.array_equal(ss[:p, 3], w["peak"]), i
