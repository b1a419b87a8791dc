"""GPU parity of the k_sim32 launch variants (sim32.cu) against the CPU oracle.

- Timeline mode: start ticks staged in shared memory and written 8 per lane (two 16-B stores);
  every entry of every plan compared with the oracle's timeline (§3.5 start times;
  SPEC.md:80-85 Timeline).
- The ring-overflow second pass: items that stall on a full 8-slot ring are re-run by k_sim32
  itself with rings of R > n_mb slots (or, forced by CP_SIM32_ENGINE_FIXUP, by the generic engine
  with global rings); results must not depend on which pass evaluated an item.
- The block-shared cost table (one instance for all items) vs per-warp tables (CP_SIM32_NOSHARE).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from tests.gpu_util import compare_sim, to_host  # noqa: E402
from workloads import configs as K, plans as PL, unpack_plans  # noqa: E402


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        for k, v in self.kv.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_timeline_fast_path_bench_shape(O):
    """Config-4 plans (p=32, 4 DCs, m=64, 192 entries per stage) with the full timeline: every
    start tick of 3000 plans, plus makespan, peak, status and per-stage stats, against the oracle;
    the timeline launch agrees with the bench launch (no timeline) on every metric."""
    b = K.perturbed_instance()
    n = 3000
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED, id0=777)
    inst = cp.Instances(b)
    r = to_host(cp.simulate(inst, ops, ln, stats=True, timeline=True, best=True))
    rb = to_host(cp.simulate(inst, ops, ln, stats=True, best=True))
    for k in ("makespan", "status", "peak_mem", "stage_stats", "best_key"):
        assert np.array_equal(r[k], rb[k]), k
    codes, lens = unpack_plans(ops.cpu().numpy().view(np.uint32), ln.cpu().numpy().view(np.uint16))
    d = b.item(0)
    for i in range(n):
        compare_sim(O, d, codes[i], lens[i], r, i, codes.shape[2], timeline=True)
    assert np.all(r["status"] == 0)
    # entries past a row's length are untouched (the caller's zeros)
    assert not r["t_start"][:, :, 192:].any()


@pytest.mark.parametrize("ring", [1, 2, 3])
def test_overflow_second_pass_variants(O, ring):
    """Undersized rings push most items through the overflow list: the k_sim32 second pass (R > n_mb),
    the engine fallback, shared and per-warp tables, with and without a timeline -- all identical."""
    b = K.perturbed_instance()
    ops, ln = PL.plans_device(b, 600, seed=K.PERTURB_SEED, id0=31)
    inst = cp.Instances(b)
    ref = cp.simulate(inst, ops, ln, stats=True, timeline=True, best=True)
    variants = [{}, {"CP_SIM32_ENGINE_FIXUP": "1"}, {"CP_SIM32_NOSHARE": "1"}]
    for env in variants:
        with _env(**env):
            for tl in (False, True):
                r = cp.simulate(inst, ops, ln, stats=True, timeline=tl, best=True, ring=ring)
                keys = ("makespan", "status", "peak_mem", "stage_stats", "best_key") + (("t_start",) if tl else ())
                for k in keys:
                    assert torch.equal(r[k], ref[k]), (ring, env, tl, k)
    c, l_ = unpack_plans(ops[:40].cpu().numpy().view(np.uint32), ln[:40].cpu().numpy().view(np.uint16))
    h = to_host(ref)
    for i in range(40):
        compare_sim(O, b.item(0), c[i], l_[i], h, i, c.shape[2], timeline=True)


def test_timeline_fast_path_mixed_instances_and_invalid(O):
    """Random instances (17-32 stages, n_sub 1-4, DP, ZeRO-1) through inst_of with timelines: valid
    plans, adjacent swaps (deadlocks), and budgets cut below the plans' peaks (memory violations that
    also overflow the small rings); every completed item's timeline against the oracle."""
    from tests.gpu_util import codes_list_to_packed
    from tests.helpers_independent import random_valid_plan
    rng = np.random.default_rng(41)
    big = K.random_instances(300, seed=42, max_p=32, max_m=14)
    keep = [i for i in range(len(big)) if big.p[i] >= 17][:60]
    batch = big.take(keep)
    cut = batch.take(np.arange(len(batch)))
    from workloads import InstanceBatch
    both = InstanceBatch.concat([batch, cut])
    n0 = len(batch)
    both.m_lim[n0:] = np.maximum(both.m_f[n0:], both.m_lim[n0:] // 3)
    plans, inst_of = [], []
    for i in range(n0):
        d = batch.item(i)
        base = random_valid_plan(d, rng)
        plans.append(base); inst_of.append(i)
        sw = [list(x) for x in base]
        s = int(rng.integers(d["p"]))
        if len(sw[s]) > 1:
            k = int(rng.integers(len(sw[s]) - 1)); sw[s][k], sw[s][k + 1] = sw[s][k + 1], sw[s][k]
        plans.append(sw); inst_of.append(i)
        plans.append(base); inst_of.append(n0 + i)
    ops, ln = codes_list_to_packed(plans, stride=32)
    inst = cp.Instances(both)
    o = torch.from_numpy(np.ascontiguousarray(ops).view(np.int32)).cuda()
    l_ = torch.from_numpy(np.ascontiguousarray(ln).view(np.int16)).cuda()
    io = torch.tensor(inst_of, dtype=torch.int32, device="cuda")
    r = to_host(cp.simulate(inst, o, l_, io, stats=True, timeline=True))
    codes, lens = unpack_plans(ops, ln)
    seen = set()
    for j, i in enumerate(inst_of):
        w = compare_sim(O, both.item(i), codes[j], lens[j], r, j, codes.shape[2], timeline=True)
        seen.add(w["status"])
    assert {0, 1, 2} <= seen, seen


def test_timeline_unaligned_stride_uses_engine(O):
    """A timeline row stride that is not a multiple of 8 entries takes the generic engine: same
    results as the staged fast path."""
    b = K.perturbed_instance()
    ops, ln = PL.plans_device(b, 300, seed=K.PERTURB_SEED, id0=5)
    inst = cp.Instances(b)
    fast = cp.simulate(inst, ops, ln, stats=True, timeline=True)
    slow = cp.simulate(inst, ops, ln, stats=True, timeline=True, len_stride=16 * ops.shape[1] + 4)
    for k in ("makespan", "status", "peak_mem", "stage_stats"):
        assert torch.equal(fast[k], slow[k]), k
    assert torch.equal(fast["t_start"], slow["t_start"][:, :, :16 * ops.shape[1]])
