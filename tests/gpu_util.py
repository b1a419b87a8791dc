"""Shared helpers for GPU parity tests: marshal neutral workloads into the product's
binding and compare with the oracle.  (Test infrastructure.)"""
from __future__ import annotations

import numpy as np

from workloads import InstanceBatch, pack_plans, unpack_plans


def plans_to_device(ops, ln):
    import torch
    return (torch.from_numpy(np.ascontiguousarray(ops).view(np.int32)).cuda(),
            torch.from_numpy(np.ascontiguousarray(ln).view(np.int16)).cuda())


def codes_list_to_packed(plans, stride=32, words=None):
    """list of per-stage code lists (one plan per item) -> packed (ops, len)."""
    n = len(plans)
    maxlen = max(max((len(r) for r in pl), default=0) for pl in plans)
    P = max(len(pl) for pl in plans)
    codes = np.zeros((n, P, max(maxlen, 1)), dtype=np.int8)
    lens = np.zeros((n, P), dtype=np.int32)
    for i, pl in enumerate(plans):
        for s, row in enumerate(pl):
            codes[i, s, :len(row)] = row
            lens[i, s] = len(row)
    words = words or max(1, (maxlen + 15) // 16)
    return pack_plans(codes, lens, stage_stride=stride, words=words)


def compare_sim(O, d, codes_s, len_s, r, i, maxlen, timeline=True):
    """Compare GPU result row i with the oracle on plan (codes_s [p, L], len_s [p])."""
    p = d["p"]
    w = O.simulate(d, np.ascontiguousarray(codes_s[:p, :maxlen]), np.asarray(len_s[:p]), timeline=timeline)
    st = int(r["status"][i])
    assert st == w["status"], (i, st, w["status"])
    assert int(r["makespan"][i]) == w["makespan"], (i, int(r["makespan"][i]), w["makespan"])
    assert int(r["peak_mem"][i]) == w["peak_mem"], (i, int(r["peak_mem"][i]), w["peak_mem"])
    if "stage_stats" in r:
        ss = r["stage_stats"][i]
        if w["makespan"] >= 0:
            assert np.array_equal(ss[:p, 0], w["first_start"]), i
            assert np.array_equal(ss[:p, 1], w["last_end"]), i
            assert np.array_equal(ss[:p, 2], w["busy"]), i
            assert np.array_equal(ss[:p, 3], w["peak"]), i
        else:
            assert not ss[:p].any()
    if timeline and "t_start" in r and w["makespan"] >= 0:
        ts = r["t_start"][i]
        for s in range(p):
            L = int(len_s[s])
            assert np.array_equal(ts[s, :L], w["t_start"][s, :L]), (i, s)
    return w


def to_host(r):
    return {k: v.cpu().numpy() for k, v in r.items()}


def batch_subset(batch: InstanceBatch, idx):
    return batch.take(idx)
