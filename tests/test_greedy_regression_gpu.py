"""Permanent regression: the round-parallel GPU greedy (two min-plus warp
scans) equals the sequential oracle Alg. 1 byte for byte on 10^5 random instances,
including zero latency / bandwidth, single-DC and one-stage-per-DC cases.  The oracle runs in one
process per host core (spawn context; tests/greedy_regress_worker.py).
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2507_00217_b200 as cp  # noqa: E402
from tests import greedy_regress_worker as Wk  # noqa: E402
from workloads import unpack_plans  # noqa: E402


def gpu_digests(batch):
    g = cp.greedy(cp.Instances(batch))
    torch.cuda.synchronize()
    codes, lens = unpack_plans(g["ops"].cpu().numpy().view(np.uint32), g["len"].cpu().numpy().view(np.uint16))
    st, ms, pk = g["status"].cpu().numpy(), g["makespan"].cpu().numpy(), g["peak_mem"].cpu().numpy()
    out = []
    for i in range(len(batch)):
        p = int(batch.p[i])
        L = int(lens[i, 0]) if p else 0
        out.append(Wk.digest(st[i], ms[i], pk[i], lens[i, :p], codes[i, :p, :L]))
    return out


def test_greedy_round_parallel_equals_sequential_1e5():
    from oracle import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    procs = max(1, min(32, os.cpu_count() or 1))
    n_bad, n_tot, first_bad = 0, 0, None
    with ctx.Pool(procs) as pool:
        for k, batch, want in pool.imap_unordered(Wk.run_chunk, range(Wk.N_CHUNKS)):
            got = gpu_digests(batch)
            for i, (a, b) in enumerate(zip(got, want)):
                n_tot += 1
                if a != b:
                    n_bad += 1
                    first_bad = first_bad or (k, i, Wk.chunk_params(k))
    assert n_tot == Wk.N_CHUNK * Wk.N_CHUNKS
    assert n_bad == 0, f"{n_bad} of {n_tot} instances differ; first (chunk, index, params): {first_bad}"
