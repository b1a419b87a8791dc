"""GPU parity of cp_exact_bnb (parallel branch and bound, exact_bnb.cu) against the CPU oracle.

The optimum is unique, so makespans are compared exactly; several plans can reach it, so the GPU's
plan is checked for validity and re-simulated by the oracle (it must reach the optimum).
Definitions: PAPER.md §4.1 :313-363 (plan set, objective), E1 setup :486, :491.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K, unpack_plans  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def _plans(r):
    return unpack_plans(r["ops"].cpu().numpy().view(np.uint32), r["len"].cpu().numpy().view(np.uint16))


def _check_plan(O, d, codes, lens, want):
    p = d["p"]
    L = int(lens[0])
    c = np.ascontiguousarray(codes[:p, :L])
    assert O.check_plan(d, c, lens[:p]) == 0
    w = O.simulate(d, c, lens[:p])
    assert w["status"] == 0 and w["makespan"] == want, (w["status"], w["makespan"], want)


def test_bnb_gpu_tiny_grid_all_16_points(O):
    """BASELINE config 1 / E1 setup (4 stages, 2 DCs, 8 microbatches) at all 16 points of
    {0, .5, 1, 2}^2 in one batch: proven optimum equal to the oracle's (tests/golden/bnb_tiny_grid.json,
    written by tools/bnb_tiny_table.py from oracle/bnb.c), plan valid and reaching it."""
    gold = json.load(open(os.path.join(GOLD, "bnb_tiny_grid.json")))["points"]
    from workloads import InstanceBatch
    batch = InstanceBatch.concat([K.tiny(r["lat_ratio"], r["bw_ratio"]) for r in gold])
    r = cp.exact_bnb(cp.Instances(batch))
    torch.cuda.synchronize()
    codes, lens = _plans(r)
    for i, row in enumerate(gold):
        assert int(r["status"][i]) == 0, (i, int(r["status"][i]))
        assert int(r["makespan"][i]) == row["optimum"] == int(r["bound"][i]), (i, int(r["makespan"][i]), row)
        _check_plan(O, batch.item(i), codes[i], lens[i], row["optimum"])


def test_bnb_gpu_random_instances_vs_oracle(O):
    """Random small instances (1-4 stages, 1-5 microbatches, per-stage costs and memory, DP tails,
    ZeRO-1, intra- and cross-DC delays): GPU optimum == oracle branch and bound, plans valid."""
    b = K.random_instances(300, seed=71, max_p=4, max_m=5, intra_delay=True)
    b.n_sub[:] = 1
    keep = [i for i in range(len(b)) if O.validate_instance(b.item(i)) == 0]
    batch = b.take(keep)
    r = cp.exact_bnb(cp.Instances(batch))
    torch.cuda.synchronize()
    codes, lens = _plans(r)
    n = 0
    for i in range(len(batch)):
        d = batch.item(i)
        w = O.bnb_opt(d, max_nodes=3_000_000)
        if not w["proven"]:
            continue
        assert int(r["status"][i]) == 0, i
        assert int(r["makespan"][i]) == w["makespan"], (i, int(r["makespan"][i]), w["makespan"])
        _check_plan(O, d, codes[i], lens[i], w["makespan"])
        n += 1
    assert n >= 200


def test_bnb_gpu_matches_exhaustive_cp_exact(O):
    """Against the other GPU exact method (cp_exact, exhaustive product enumeration) on m <= 4 E1
    replicas with the greedy's makespan as `upper`, and against the oracle's enumeration where
    that is small enough."""
    from workloads import InstanceBatch
    pts = [(a, b) for a in (0, 0.5, 1, 2) for b in (0, 0.5, 1, 2)]
    batch = InstanceBatch.concat([K.uniform_instance(4, 3, 2, 100, 100, 100, lat=int(a * 100), bw=int(b * 100),
                                                     mlim_x1000=1000) for a, b in pts])
    inst = cp.Instances(batch)
    g = cp.greedy(inst)
    up = g["makespan"].to(torch.int32)
    rb = cp.exact_bnb(inst, upper=up)
    re = cp.exact(inst)
    torch.cuda.synchronize()
    assert torch.equal(rb["status"].cpu(), torch.zeros(len(pts), dtype=torch.int32))
    assert torch.equal(rb["makespan"].cpu(), re["makespan"].cpu())
    assert bool((rb["makespan"] <= up).all())
    codes, lens = _plans(rb)
    for i in range(len(pts)):
        _check_plan(O, batch.item(i), codes[i], lens[i], int(re["makespan"][i]))


def test_bnb_gpu_limits(O):
    """A node limit leaves the search incomplete: status CPI_INCOMPLETE (64), a valid plan no better
    than the optimum, and a lower bound no larger than it; out-of-range instances get CPI_OVERFLOW."""
    from workloads import InstanceBatch
    d2 = K.tiny(2, 2)
    big = K.uniform_instance(9, 2, 2, 100, 100, 100)              # p > 8
    nsub = K.tiny(1, 1, n_sub=2)                                   # n_sub != 1
    batch = InstanceBatch.concat([d2, big, nsub])
    r = cp.exact_bnb(cp.Instances(batch), max_nodes=500, budget=64)
    torch.cuda.synchronize()
    st = r["status"].cpu().tolist()
    assert st[0] == 64 and st[1] == 16 and st[2] == 16, st
    opt = 4300                                                     # tests/golden/bnb_tiny_grid.json, (2, 2)
    ms, bd = int(r["makespan"][0]), int(r["bound"][0])
    assert bd <= opt and (ms < 0 or ms >= opt)
    if ms >= 0:
        codes, lens = _plans(r)
        _check_plan(O, d2.item(0), codes[0], lens[0], ms)
