"""ctypes wrapper of the CrossPipe CPU oracle.  *** TEST INFRASTRUCTURE ONLY ***

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  It packs the neutral `workloads` formats into the
oracle's own C structs (its own packing code; nothing shared with the product).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
MAXP = 32
ST_DEADLOCK, ST_MEM, ST_BAD_PLAN, ST_BAD_INST = 1, 2, 4, 8

I64A = C.c_int64 * MAXP


class OrInst(C.Structure):
    _fields_ = [("p", C.c_int32), ("m", C.c_int32), ("n_sub", C.c_int32), ("zero1", C.c_int32)] + [
        (k, I64A) for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag",
                            "lat_f", "bw_f", "lat_b", "bw_b")]


class OrResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("makespan", C.c_int64), ("peak_mem", C.c_int64),
                ("first_start", I64A), ("last_end", I64A), ("busy", I64A), ("peak", I64A),
                ("iterations", C.c_int64)]


D64A = C.c_double * MAXP


class OrBnbInfo(C.Structure):
    _fields_ = [("greedy", C.c_int64), ("root_bound", C.c_int64), ("bound", C.c_int64), ("nodes", C.c_int64),
                ("table_bytes", C.c_int64), ("proven", C.c_int32)]


class OrSpecSI(C.Structure):
    _fields_ = [("p", C.c_int32), ("m", C.c_int32), ("n_sub", C.c_int32), ("zero1", C.c_int32),
                ("n_dc", C.c_int32), ("dc_of_stage", C.c_int32 * MAXP)] + [
        (k, D64A) for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag")] + [
        ("alpha", (C.c_double * 4) * 4), ("beta", (C.c_double * 4) * 4),
        ("msg_f", D64A), ("msg_b", D64A), ("tick_s", C.c_double), ("mem_unit", C.c_double)]


class OrLink(C.Structure):
    _fields_ = [("s", C.POINTER(C.c_int64)), ("e", C.POINTER(C.c_int64)), ("n", C.c_int32), ("cap", C.c_int32)]


class OrGrid(C.Structure):
    _fields_ = [("base", OrInst), ("n_dc", C.c_int32),
                ("n_pp_vals", C.c_int32 * 8), ("n_pp_n", C.c_int32), ("n_mb_vals", C.c_int32 * 8), ("n_mb_n", C.c_int32),
                ("lat", C.POINTER(C.c_int64)), ("n_lat", C.c_int32),
                ("bw", C.POINTER(C.c_int64)), ("n_bw", C.c_int32),
                ("mlim_x1000", C.POINTER(C.c_int64)), ("n_mem", C.c_int32),
                ("tdp", C.POINTER(C.c_int64)), ("n_dp", C.c_int32),
                ("cand_mask", C.c_uint32)]


def build(force=False):
    src = os.path.join(_HERE, "oracle.c")
    srcs = [src, os.path.join(_HERE, "bnb.c"), os.path.join(_HERE, "oracle.h")]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(x) for x in srcs):
        subprocess.check_call(["make", "-s", "-C", _HERE, "-B"] if force else ["make", "-s", "-C", _HERE])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.POINTER
        L.or_reserve_window.restype = C.c_int64
        L.or_reserve_window.argtypes = [P(OrLink), C.c_int64, C.c_int64]
        L.or_link_init.argtypes = [P(OrLink)]
        L.or_link_free.argtypes = [P(OrLink)]
        for fn in ("or_simulate", "or_greedy", "or_simulate_wave", "or_simulate_loop"):
            f = getattr(L, fn)
            f.restype = C.c_int32
            f.argtypes = [P(OrInst), P(C.c_int8), P(C.c_int32), C.c_int32, P(OrResult), P(C.c_int64)]
        L.or_check_plan.restype = C.c_int32
        L.or_check_plan.argtypes = [P(OrInst), P(C.c_int8), P(C.c_int32), C.c_int32]
        L.or_check_plan_wave.restype = C.c_int32
        L.or_check_plan_wave.argtypes = [P(OrInst), P(C.c_int8), P(C.c_int32), C.c_int32]
        for fn in ("or_build_1f1b", "or_build_gpipe", "or_build_zbh1"):
            getattr(L, fn).argtypes = [C.c_int32, C.c_int32, P(C.c_int8), P(C.c_int32), C.c_int32]
        L.or_build_zbv.restype = C.c_int32
        L.or_build_zbv.argtypes = [C.c_int32, C.c_int32, P(C.c_int8), P(C.c_int32), C.c_int32]
        L.or_build_iv1f1b.restype = C.c_int32
        L.or_build_iv1f1b.argtypes = [C.c_int32, C.c_int32, P(C.c_int8), P(C.c_int32), C.c_int32]
        L.or_enumerate_opt.restype = C.c_int64
        L.or_enumerate_opt.argtypes = [P(OrInst), C.c_int64, P(C.c_int8), P(C.c_int32), C.c_int32, P(OrResult)]
        L.or_bnb_opt.restype = C.c_int32
        L.or_bnb_opt.argtypes = [P(OrInst), C.c_int64, C.c_int64, C.c_int32, P(C.c_int8), P(C.c_int32), C.c_int32, P(OrResult),
                                 P(OrBnbInfo)]
        L.or_quantize.restype = C.c_int32
        L.or_quantize.argtypes = [P(OrSpecSI), P(OrInst)]
        L.or_validate_instance.restype = C.c_int32
        L.or_validate_instance.argtypes = [P(OrInst)]
        L.or_grid_points.restype = C.c_int64
        L.or_grid_points.argtypes = [P(OrGrid)]
        L.or_grid_instance.argtypes = [P(OrGrid), C.c_int64, P(OrInst)]
        L.or_sweep_point.restype = C.c_uint64
        L.or_sweep_point.argtypes = [P(OrGrid), C.c_int64, P(C.c_int64)]
        _lib = L
    return _lib


def to_or_inst(d) -> OrInst:
    """d: dict from InstanceBatch.item() (or any mapping with the same keys)."""
    o = OrInst()
    o.p, o.m, o.n_sub, o.zero1 = int(d["p"]), int(d["m"]), int(d["n_sub"]), int(d["zero1"])
    for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag", "lat_f", "bw_f", "lat_b", "bw_b"):
        arr = getattr(o, k)
        for i, v in enumerate(np.asarray(d[k]).ravel()[:MAXP]):
            arr[i] = int(v)
    return o


def _result(r: OrResult, p: int) -> dict:
    return {"status": r.status, "makespan": r.makespan, "peak_mem": r.peak_mem, "iterations": r.iterations,
            "first_start": np.array(r.first_start[:p]), "last_end": np.array(r.last_end[:p]),
            "busy": np.array(r.busy[:p]), "peak": np.array(r.peak[:p])}


def _codes_arr(codes, lens, p):
    """codes: list of per-stage sequences, or array [p, L]; returns (int8 [p, maxlen], int32 [p], maxlen)."""
    if isinstance(codes, np.ndarray) and codes.ndim == 2:
        c = np.ascontiguousarray(codes[:p], dtype=np.int8)
        ln = np.ascontiguousarray(np.asarray(lens)[:p], dtype=np.int32)
        return c, ln, c.shape[1]
    maxlen = max(1, max(len(x) for x in codes))
    c = np.zeros((p, maxlen), dtype=np.int8)
    ln = np.zeros(p, dtype=np.int32)
    for s, seq in enumerate(codes[:p]):
        c[s, :len(seq)] = seq
        ln[s] = len(seq)
    return c, ln, maxlen


def simulate(d, codes, lens=None, timeline=False) -> dict:
    L = lib()
    p = int(d["p"])
    c, ln, maxlen = _codes_arr(codes, lens, p)
    inst, res = to_or_inst(d), OrResult()
    ts = np.zeros((p, maxlen), dtype=np.int64) if timeline else None
    L.or_simulate(C.byref(inst), c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                  maxlen, C.byref(res), ts.ctypes.data_as(C.POINTER(C.c_int64)) if timeline else None)
    out = _result(res, p)
    if timeline:
        out["t_start"] = ts
    return out


def simulate_wave(d, codes, lens=None, timeline=False) -> dict:
    """Wave-pattern plan (entries type | chunk << 2), reading Q32."""
    L = lib()
    p = int(d["p"])
    c, ln, maxlen = _codes_arr(codes, lens, p)
    inst, res = to_or_inst(d), OrResult()
    ts = np.zeros((p, maxlen), dtype=np.int64) if timeline else None
    L.or_simulate_wave(C.byref(inst), c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                       maxlen, C.byref(res), ts.ctypes.data_as(C.POINTER(C.c_int64)) if timeline else None)
    out = _result(res, p)
    if timeline:
        out["t_start"] = ts
    return out


def simulate_loop(d, codes, lens=None, timeline=False) -> dict:
    """Loop-pattern plan, 2 chunks (entries type | chunk << 2), reading Q33; boundary index p-1 of
    lat_f/bw_f (p-1 -> 0) and lat_b/bw_b (0 -> p-1) is the wrap link."""
    L = lib()
    p = int(d["p"])
    c, ln, maxlen = _codes_arr(codes, lens, p)
    inst, res = to_or_inst(d), OrResult()
    ts = np.zeros((p, maxlen), dtype=np.int64) if timeline else None
    L.or_simulate_loop(C.byref(inst), c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                       maxlen, C.byref(res), ts.ctypes.data_as(C.POINTER(C.c_int64)) if timeline else None)
    out = _result(res, p)
    if timeline:
        out["t_start"] = ts
    return out


def check_plan_wave(d, codes, lens=None) -> int:
    p = int(d["p"])
    c, ln, maxlen = _codes_arr(codes, lens, p)
    return lib().or_check_plan_wave(C.byref(to_or_inst(d)), c.ctypes.data_as(C.POINTER(C.c_int8)),
                                    ln.ctypes.data_as(C.POINTER(C.c_int32)), maxlen)


def greedy(d, timeline=False) -> dict:
    L = lib()
    p, m, ns = int(d["p"]), int(d["m"]), int(d["n_sub"])
    maxlen = (2 + ns) * m
    c = np.zeros((p, maxlen), dtype=np.int8)
    ln = np.zeros(p, dtype=np.int32)
    ts = np.zeros((p, maxlen), dtype=np.int64) if timeline else None
    inst, res = to_or_inst(d), OrResult()
    L.or_greedy(C.byref(inst), c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                maxlen, C.byref(res), ts.ctypes.data_as(C.POINTER(C.c_int64)) if timeline else None)
    out = _result(res, p)
    out["codes"], out["len"] = c, ln
    if timeline:
        out["t_start"] = ts
    return out


def validate_instance(d) -> int:
    """Instance invariants (Q10, Q12, Q19, Q21): 0 or BAD_INSTANCE (8)."""
    return int(lib().or_validate_instance(C.byref(to_or_inst(d))))


def check_plan(d, codes, lens=None) -> int:
    p = int(d["p"])
    c, ln, maxlen = _codes_arr(codes, lens, p)
    return lib().or_check_plan(C.byref(to_or_inst(d)), c.ctypes.data_as(C.POINTER(C.c_int8)),
                               ln.ctypes.data_as(C.POINTER(C.c_int32)), maxlen)


def build_static(kind: str, p: int, m: int):
    """gpipe / 1f1b / zbh1 (UD plans), iv1f1b (Loop plans, 2 chunks, needs m % p == 0) or zbv (Wave
    plans, 2 chunks, split W)."""
    if kind == "zbv":
        maxlen = 6 * m
        c = np.zeros((p, maxlen), dtype=np.int8)
        ln = np.zeros(p, dtype=np.int32)
        rc = lib().or_build_zbv(p, m, c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                                maxlen)
        if rc:
            raise ValueError("zbv needs p >= 1, m >= 1")
        return c, ln
    if kind == "iv1f1b":
        maxlen = 4 * m
        c = np.zeros((p, maxlen), dtype=np.int8)
        ln = np.zeros(p, dtype=np.int32)
        rc = lib().or_build_iv1f1b(p, m, c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)),
                                   maxlen)
        if rc:
            raise ValueError("iv1f1b needs m % p == 0")
        return c, ln
    maxlen = 3 * m if kind == "zbh1" else 2 * m
    c = np.zeros((p, maxlen), dtype=np.int8)
    ln = np.zeros(p, dtype=np.int32)
    fn = {"1f1b": lib().or_build_1f1b, "gpipe": lib().or_build_gpipe, "zbh1": lib().or_build_zbh1}[kind]
    fn(p, m, c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)), maxlen)
    return c, ln


def enumerate_opt(d, max_plans=2_000_000) -> dict:
    p, m = int(d["p"]), int(d["m"])
    maxlen = 3 * m
    c = np.zeros((p, maxlen), dtype=np.int8)
    ln = np.zeros(p, dtype=np.int32)
    res = OrResult()
    n = lib().or_enumerate_opt(C.byref(to_or_inst(d)), max_plans, c.ctypes.data_as(C.POINTER(C.c_int8)),
                               ln.ctypes.data_as(C.POINTER(C.c_int32)), maxlen, C.byref(res))
    out = _result(res, p)
    out["evaluated"], out["codes"], out["len"] = n, c, ln
    return out


BNB_NO_DOMINANCE, BNB_NO_JPS = 1, 2


def bnb_opt(d, max_nodes=50_000_000, max_table_bytes=4 << 30, flags=0) -> dict:
    """Exact optimum (n_sub = 1 split plans) by branch and bound (bnb.c).  Returns the re-simulated best
    plan's result plus proven / bound / nodes / greedy / root_bound; rc -1 = not applicable."""
    p, m = int(d["p"]), int(d["m"])
    maxlen = 3 * m
    c = np.zeros((p, maxlen), dtype=np.int8)
    ln = np.zeros(p, dtype=np.int32)
    res, info = OrResult(), OrBnbInfo()
    rc = lib().or_bnb_opt(C.byref(to_or_inst(d)), int(max_nodes), int(max_table_bytes), int(flags),
                          c.ctypes.data_as(C.POINTER(C.c_int8)), ln.ctypes.data_as(C.POINTER(C.c_int32)), maxlen,
                          C.byref(res), C.byref(info))
    out = _result(res, p)
    out.update(rc=rc, codes=c, len=ln, proven=bool(info.proven), bound=info.bound, nodes=info.nodes,
               greedy=info.greedy, root_bound=info.root_bound, table_bytes=info.table_bytes)
    return out


def reserve_window(intervals, t_ready, width):
    """Reserve on a link pre-loaded with `intervals` (inserted in order via zero-contention reservations)."""
    L = lib()
    lk = OrLink()
    L.or_link_init(C.byref(lk))
    for (s, e) in intervals:
        got = L.or_reserve_window(C.byref(lk), s, e - s)
        assert got == e, "preload intervals must be disjoint and sorted"
    end = L.or_reserve_window(C.byref(lk), t_ready, width)
    L.or_link_free(C.byref(lk))
    return end - width, end


def quantize(spec: dict):
    s = OrSpecSI()
    for k, v in spec.items():
        if k in ("alpha", "beta"):
            arr = getattr(s, k)
            for i in range(4):
                for j in range(4):
                    arr[i][j] = float(v[i][j]) if i < len(v) and j < len(v[i]) else 0.0
        elif k in ("dc_of_stage",):
            arr = getattr(s, k)
            for i, x in enumerate(v):
                arr[i] = int(x)
        elif isinstance(v, (list, tuple, np.ndarray)):
            arr = getattr(s, k)
            for i, x in enumerate(v):
                arr[i] = float(x)
        else:
            setattr(s, k, v)
    o = OrInst()
    st = lib().or_quantize(C.byref(s), C.byref(o))
    out = {"status": st, "p": o.p, "m": o.m, "n_sub": o.n_sub, "zero1": o.zero1}
    for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag"):
        out[k] = np.array(getattr(o, k)[:o.p])
    for k in ("lat_f", "bw_f", "lat_b", "bw_b"):
        out[k] = np.array(getattr(o, k)[:max(o.p - 1, 0)])
    return out


def to_or_grid(g):
    """g: workloads.Grid -> (OrGrid, keepalive)."""
    G = OrGrid()
    G.base = to_or_inst(g.base.item(0) | {"p": int(g.base.p[0])})
    # base per-stage arrays must cover all 32 stages
    for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag"):
        arr = getattr(G.base, k)
        for i in range(MAXP):
            arr[i] = int(getattr(g.base, k)[0, i])
    G.n_dc = g.n_dc
    for i, v in enumerate(g.pp_vals):
        G.n_pp_vals[i] = v
    G.n_pp_n = len(g.pp_vals)
    for i, v in enumerate(g.mb_vals):
        G.n_mb_vals[i] = v
    G.n_mb_n = len(g.mb_vals)
    keep = []
    for name in ("lat", "bw", "mlim_x1000", "tdp"):
        a = np.ascontiguousarray(np.asarray(getattr(g, name), dtype=np.int64))
        keep.append(a)
        setattr(G, name, a.ctypes.data_as(C.POINTER(C.c_int64)))
    G.n_lat, G.n_bw, G.n_mem, G.n_dp = len(g.lat), len(g.bw), len(g.mlim_x1000), len(g.tdp)
    G.cand_mask = g.cand_mask
    return G, keep


def sweep_point(g, k: int, G=None):
    if G is None:
        G, keep = to_or_grid(g)
    cm = (C.c_int64 * 6)()
    key = lib().or_sweep_point(C.byref(G), int(k), cm)
    return int(key), list(cm)


def grid_instance(g, k: int, G=None) -> dict:
    if G is None:
        G, keep = to_or_grid(g)
    o = OrInst()
    lib().or_grid_instance(C.byref(G), int(k), C.byref(o))
    d = {"p": o.p, "m": o.m, "n_sub": o.n_sub, "zero1": o.zero1}
    for k2 in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag"):
        d[k2] = np.array(getattr(o, k2)[:o.p])
    for k2 in ("lat_f", "bw_f", "lat_b", "bw_b"):
        d[k2] = np.array(getattr(o, k2)[:o.p])          # index p-1: the (unused) wrap link, 0
    return d
