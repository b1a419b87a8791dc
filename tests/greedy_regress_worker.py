"""Worker for the 10^5-instance greedy regression (tests/test_greedy_regression_gpu.py).

Test infrastructure only: generates one seeded chunk of random instances (workloads/, no method
arithmetic) and runs the oracle's sequential Alg. 1 on every instance, returning the batch and one
digest per instance.  No torch import, so spawn-context workers start quickly.
"""
import hashlib

import numpy as np

N_CHUNK = 1000
N_CHUNKS = 100
SEED0 = 0x5EED0000
MAX_P = (2, 4, 8, 16, 32)
MAX_M = (6, 12, 20)


def chunk_params(k):
    """Chunk k: instance mix (1..max_p stages incl. one stage per DC and single-DC cases, 1-4 DCs,
    zero and non-zero latency / bandwidth, intra-DC delays on every other chunk)."""
    return dict(seed=SEED0 + k, max_p=MAX_P[k % len(MAX_P)], max_m=MAX_M[(k // len(MAX_P)) % len(MAX_M)],
                intra_delay=(k % 2 == 0))


def digest(status, makespan, peak, lens, codes):
    """One instance's greedy output as a digest: status, makespan, peak memory, per-stage row
    lengths and every 2-bit plan entry."""
    h = hashlib.blake2b(digest_size=16)
    h.update(np.asarray([status, makespan, peak], dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(lens, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(codes, dtype=np.int8).tobytes())
    return h.hexdigest()


def run_chunk(k):
    from oracle import oracle as O
    from workloads import configs as K
    prm = chunk_params(k)
    batch = K.random_instances(N_CHUNK, seed=prm["seed"], max_p=prm["max_p"], max_m=prm["max_m"],
                               intra_delay=prm["intra_delay"])
    out = []
    for i in range(N_CHUNK):
        d = batch.item(i)
        w = O.greedy(d)
        p = d["p"]
        L = int(w["len"][0]) if p else 0
        out.append(digest(w["status"], w["makespan"], w["peak_mem"], w["len"][:p], w["codes"][:p, :L]))
    return k, batch, out
