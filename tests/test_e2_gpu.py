"""GPU parity of the E2 grid (§5.2 :503-516, App. E :855-858; reading Q36): every
(latency, bandwidth) point of tools/e2_ppdp.py -- the greedy CrossUDSub at n_sub 1, 2 and 4 (cp_greedy:
plans byte for byte and makespans) and the ZBV stand-in (reading Q35, cp_build_static + cp_simulate on
the Wave pattern) -- against the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import ppdp as E, unpack_plans  # noqa: E402
from workloads.core import InstanceBatch  # noqa: E402


def test_e2_every_point_greedy_and_zbv(oracle_lib):
    O = oracle_lib
    pts = [(l, g) for l in E.LATENCIES_MS for g in E.BANDWIDTHS_GBS]
    gb = InstanceBatch.concat([E.pp_instance(l * 1e-3, g * 1e9, n_sub=ns) for ns in (1, 2, 4) for (l, g) in pts])
    gr = cp.greedy(cp.Instances(gb))
    codes, lens = unpack_plans(gr["ops"].cpu().numpy().view(np.uint32), gr["len"].cpu().numpy().view(np.uint16))
    ms, st = gr["makespan"].cpu().numpy(), gr["status"].cpu().numpy()
    for i in range(len(gb)):
        w = O.greedy(gb.item(i))
        assert (int(st[i]), int(ms[i])) == (w["status"], w["makespan"]), i
        L = int(w["len"][0])
        assert np.array_equal(codes[i][:16, :L], w["codes"][:16, :L]), i
    vb = InstanceBatch.concat([E.wave_instance(l * 1e-3, g * 1e9) for (l, g) in pts] + [E.wave_instance(0.0, float("inf"))])
    vinst = cp.Instances(vb)
    vo, vl = cp.build_static("zbv", vinst)
    vr = cp.simulate(vinst, vo, vl, wave=True)
    vms = vr["makespan"].cpu().numpy()
    cz, lz = O.build_static("zbv", 16, E.n_microbatches())
    for k in range(len(vb)):
        assert int(vms[k]) == O.simulate_wave(vb.item(k), cz, lz)["makespan"], k
    assert np.all(vr["status"].cpu().numpy() == 0)
