"""Thin Python binding of the CrossPipe C ABI (argument marshalling only).

Every step of the hot path runs in libcrosspipe.so kernels; this module only packs
records, allocates result tensors with torch (device memory / streams are torch's),
and forwards raw pointers.  Names follow include/crosspipe.h.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np
import torch

from . import _lib as L

INT32_MAX = 2**31 - 1
KEY_NONE = 2**63 - 1          # no feasible candidate / not owned (int64 max)
KEY_OVER = 2**63 - 2          # point exceeds GPU limits (CPI_OVERFLOW)


def _require_cuda(*tensors):
    if not torch.cuda.is_available():
        raise RuntimeError("CrossPipe hot path needs a CUDA device (sm_100a); there is no CPU fallback")
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("device tensors expected")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@contextlib.contextmanager
def _on_stream(stream, *inputs):
    """Run a call's allocation, initialization and launch on `stream` (default: torch's current
    stream).  A non-current stream first waits for the current one, so inputs written there are
    visible, and the input tensors are recorded on it, so the caching allocator keeps them alive
    until the launch has consumed them.  Tensors allocated inside belong to `stream`: the caller
    orders any other stream's use of the results after it (e.g. current.wait_stream(stream))."""
    cur = torch.cuda.current_stream()
    if stream is None or stream == cur:
        yield cur
        return
    stream.wait_stream(cur)
    for t in inputs:
        if t is not None:
            t.record_stream(stream)
    with torch.cuda.stream(stream):
        yield stream


# ---------------------------------------------------------------------------------------- records
def pack_instances(batch) -> np.ndarray:
    """workloads.InstanceBatch -> numpy array of cp_inst_v1 records (format conversion)."""
    n = len(batch)
    rec = np.zeros(n, dtype=L.INST_DTYPE)
    for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag", "lat_f", "bw_f", "lat_b", "bw_b"):
        v = np.asarray(getattr(batch, k))
        if v.size and (v.max() > INT32_MAX or v.min() < -INT32_MAX - 1):
            raise OverflowError(f"{k} does not fit int32")
        rec[k] = v
    rec["n_pp"] = batch.p
    rec["n_mb"] = batch.m
    rec["n_sub"] = batch.n_sub
    rec["flags"] = np.asarray(batch.zero1) & 1
    rec["n_dc"] = batch.n_dc if batch.n_dc is not None else 1
    rec["version"] = 1
    rec["tick_ns"] = int(round(batch.tick_s * 1e9))
    return rec


def records_to_device(rec: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(rec.view(np.uint8).reshape(len(rec), 1792).copy()).to(device)


def ring_hint(batch) -> int:
    """max over items of min(n_mb, max_s floor(m_lim/m_f)) -- in-flight F bound."""
    mf = np.maximum(np.asarray(batch.m_f), 1)
    bound = (np.asarray(batch.m_lim) // mf).max(axis=1)
    return int(np.max(np.minimum(bound, np.asarray(batch.m)))) if len(batch) else 1


class Instances:
    """Device-resident instance batch + the host-side hints the launcher needs."""

    def __init__(self, batch, device="cuda"):
        self.rec = pack_instances(batch)
        self.dev = records_to_device(self.rec, device)
        self.n = len(batch)
        self.max_pp = int(np.max(batch.p))
        self.max_mb = int(np.max(batch.m))
        self.ring = ring_hint(batch)
        self.max_sub = int(np.max(batch.n_sub))

    def desc(self, ring=None):
        return L.CpInstances(self.n, self.max_pp, self.max_mb, int(ring if ring is not None else self.ring),
                             self.dev.data_ptr())


def _workspace(which, desc, n_items, device):
    nb = L.load().cp_workspace_bytes(which, C.byref(desc), n_items)
    return torch.empty(max(int(nb), 256), dtype=torch.uint8, device=device)


def _results(n, stage_stride, stats, timeline, len_stride, device, best, index_base=0):
    r = {"makespan": torch.empty(n, dtype=torch.int64, device=device),
         "peak_mem": torch.empty(n, dtype=torch.int32, device=device),
         "status": torch.empty(n, dtype=torch.int32, device=device)}
    if stats:
        r["stage_stats"] = torch.empty((n, stage_stride, 4), dtype=torch.int32, device=device)
    if timeline:
        r["t_start"] = torch.zeros((n, stage_stride, len_stride), dtype=torch.int32, device=device)
    if best:
        r["best_key"] = torch.full((1,), KEY_NONE, dtype=torch.int64, device=device)
    cres = L.CpResults(r["makespan"].data_ptr(), r["peak_mem"].data_ptr(), r["status"].data_ptr(),
                       r["stage_stats"].data_ptr() if stats else None,
                       r["t_start"].data_ptr() if timeline else None, int(len_stride if timeline else 0),
                       int(index_base), r["best_key"].data_ptr() if best else None)
    return r, cres


# ---------------------------------------------------------------------------------------- calls
def simulate(inst: Instances, ops: torch.Tensor, lens: torch.Tensor, inst_of: torch.Tensor = None, *,
             stats=False, timeline=False, len_stride=None, best=False, ring=None, stream=None, ws=None,
             out=None, wave=False, loop=False, index_base=0):
    """cp_simulate: evaluate ops.shape[0] fixed plans.  ops uint32-as-int32 [n, words, stride], lens int16 [n, stride].
    wave=True / loop=True: two-chunk Wave (reading Q32) / Loop (Q33) plans, 4-bit entries type | chunk << 2,
    8 per word.  index_base: global id of plan 0, carried by best_key (makespan << 32 | index_base + i), so
    shards of one population (ranks, chunks) report traceable ids.  `stream`: see _on_stream; a
    caller-supplied `out` / `ws` must not be in use by another stream."""
    _require_cuda(ops, lens, inst_of)
    n, words, stride = ops.shape
    dev = ops.device
    d = inst.desc(ring)
    with _on_stream(stream, ops, lens, inst_of, inst.dev) as s:
        if out is None:
            out = _results(n, stride, stats, timeline, len_stride or (8 if (wave or loop) else 16) * words, dev, best,
                           index_base)
        r, cres = out
        if ws is None:
            ws = _workspace(0, d, n, dev)
        sc = L.CpSchedules(n, stride, words, 2 if loop else (1 if wave else 0), _ptr(inst_of), ops.data_ptr(),
                           lens.data_ptr())
        if best:
            r["best_key"].fill_(KEY_NONE)
        rc = L.load().cp_simulate(C.byref(d), C.byref(sc), C.byref(cres), C.c_void_p(ws.data_ptr()), ws.numel(),
                                  _stream(s))
    L.check(rc, "cp_simulate")
    return r


class HostPipeline:
    """cp_simulate over HOST (pinned) plan buffers with copy/compute overlap.

    The batch is cut into chunks; chunk k+1's host->device copy (copy stream) overlaps chunk k's
    kernel (compute stream), and results of chunk k stream back while later chunks run.  Every
    chunk is one cp_simulate call on device views with index_base = index_base + chunk start, so
    best_key carries global schedule ids.  Device buffers and streams are allocated once and reused."""

    def __init__(self, inst: Instances, n: int, words: int, stride: int, chunks: int = 32, device="cuda",
                 index_base: int = 0):
        self.inst, self.n, self.chunks, self.base = inst, n, max(1, chunks), int(index_base)
        self.ops_d = torch.empty((n, words, stride), dtype=torch.int32, device=device)
        self.len_d = torch.empty((n, stride), dtype=torch.int16, device=device)
        self.r, _ = _results(n, stride, False, False, 0, device, True)
        self.h2d, self.comp, self.d2h = (torch.cuda.Stream(device) for _ in range(3))
        self.bounds = [n * k // self.chunks for k in range(self.chunks + 1)]
        step = max(b - a for a, b in zip(self.bounds, self.bounds[1:]))
        self.ws = _workspace(0, inst.desc(), step, device)
        self.words, self.stride = words, stride

    def run(self, ops_h, len_h, makespan_h, peak_h, status_h):
        """Enqueue one evaluation of the host batch; results land in the pinned host tensors.
        Returns the device best_key tensor (valid after torch.cuda.synchronize())."""
        r = self.r
        cur = torch.cuda.current_stream()
        self.h2d.wait_stream(cur)
        self.comp.wait_stream(cur)
        with torch.cuda.stream(self.comp):
            r["best_key"].fill_(KEY_NONE)
        done_in, done_out = [], []
        for k in range(self.chunks):
            a, b = self.bounds[k], self.bounds[k + 1]
            with torch.cuda.stream(self.h2d):
                self.ops_d[a:b].copy_(ops_h[a:b], non_blocking=True)
                self.len_d[a:b].copy_(len_h[a:b], non_blocking=True)
                e = torch.cuda.Event(); e.record(self.h2d); done_in.append(e)
            self.comp.wait_event(done_in[k])
            d = self.inst.desc()
            sc = L.CpSchedules(b - a, self.stride, self.words, 0, None, self.ops_d[a].data_ptr(),
                               self.len_d[a].data_ptr())
            cres = L.CpResults(r["makespan"][a:].data_ptr(), r["peak_mem"][a:].data_ptr(), r["status"][a:].data_ptr(),
                               None, None, 0, self.base + int(a), r["best_key"].data_ptr())
            rc = L.load().cp_simulate(C.byref(d), C.byref(sc), C.byref(cres), C.c_void_p(self.ws.data_ptr()),
                                      self.ws.numel(), C.c_void_p(self.comp.cuda_stream))
            L.check(rc, "cp_simulate")
            e = torch.cuda.Event(); e.record(self.comp); done_out.append(e)
            self.d2h.wait_event(e)
            with torch.cuda.stream(self.d2h):
                makespan_h[a:b].copy_(r["makespan"][a:b], non_blocking=True)
                peak_h[a:b].copy_(r["peak_mem"][a:b], non_blocking=True)
                status_h[a:b].copy_(r["status"][a:b], non_blocking=True)
        cur.wait_stream(self.comp)
        cur.wait_stream(self.d2h)
        return r["best_key"]


def greedy(inst: Instances, *, stats=False, timeline=False, stage_stride=None, words=None, ring=None,
           stream=None, ws=None, out=None):
    """cp_greedy: one Alg.-1 schedule per instance -> dict(ops, len, makespan, peak_mem, status, ...)."""
    _require_cuda(inst.dev)
    dev = inst.dev.device
    n = inst.n
    stride = stage_stride or inst.max_pp
    if words is None:
        words = ((2 + inst.max_sub) * inst.max_mb + 15) // 16
    d = inst.desc(ring)
    with _on_stream(stream, inst.dev) as s:
        if out is None:
            r, cres = _results(n, stride, stats, timeline, 16 * words, dev, False)
            r["ops"] = torch.empty((n, words, stride), dtype=torch.int32, device=dev)
            r["len"] = torch.empty((n, stride), dtype=torch.int16, device=dev)
            out = (r, cres)
        r, cres = out
        if ws is None:
            ws = _workspace(1, d, n, dev)
        sc = L.CpSchedules(n, stride, words, 0, None, r["ops"].data_ptr(), r["len"].data_ptr())
        rc = L.load().cp_greedy(C.byref(d), C.byref(sc), C.byref(cres), C.c_void_p(ws.data_ptr()), ws.numel(),
                                _stream(s))
    L.check(rc, "cp_greedy")
    return r


def build_static(kind: str, inst: Instances, n=None, inst_of=None, *, stage_stride=None, words=None, stream=None):
    """cp_build_static: static plans ("gpipe", "1f1b", "zbh1"; "iv1f1b" for loop=True and "zbv" for
    wave=True simulation) for n items (item i uses instance
    inst_of[i], or i / 0 as in cp_simulate) -> (ops int32 [n, words, stride], len int16 [n, stride]),
    ready for simulate()."""
    _require_cuda(inst.dev)
    dev = inst.dev.device
    k = L.PLAN_KINDS[kind]
    n = inst.n if n is None else int(n)
    stride = stage_stride or inst.max_pp
    if words is None:
        per_mb = {"zbh1": 3, "iv1f1b": 4, "zbv": 6}.get(kind, 2)
        words = (per_mb * inst.max_mb + 7) // 8 if kind in ("iv1f1b", "zbv") else (per_mb * inst.max_mb + 15) // 16
    d = inst.desc(None)
    io = inst_of.data_ptr() if inst_of is not None else None
    with _on_stream(stream, inst.dev, inst_of) as s:
        ops = torch.empty((n, words, stride), dtype=torch.int32, device=dev)
        ln = torch.empty((n, stride), dtype=torch.int16, device=dev)
        sc = L.CpSchedules(n, stride, words, 0, io, ops.data_ptr(), ln.data_ptr())
        rc = L.load().cp_build_static(k, C.byref(d), C.byref(sc), _stream(s))
    L.check(rc, "cp_build_static")
    return ops, ln


def exact(inst: Instances, *, cap=65536, max_plans=1 << 32, upper=None, stage_stride=None, stream=None):
    """cp_exact: the makespan-optimal split plan (n_sub = 1) of every (tiny) instance by exhaustive
    search on the GPU -> dict(ops int32 [n, words, stride], len int16 [n, stride], makespan, status).
    Plans are in simulate()'s layout; status CPI_OVERFLOW (16) marks instances beyond the limits.
    upper: optional int32 [n] device tensor of feasible makespans (e.g. greedy(inst)["makespan"] for
    n_sub = 1 instances) seeding the search's cut; the result does not change."""
    _require_cuda(inst.dev)
    dev = inst.dev.device
    n = inst.n
    stride = stage_stride or inst.max_pp
    words = max(1, (3 * min(inst.max_mb, 8) + 15) // 16)
    nb = int(L.load().cp_exact_workspace_bytes(n, cap))
    d = inst.desc(None)
    with _on_stream(stream, inst.dev, upper) as s:
        ops = torch.empty((n, words, stride), dtype=torch.int32, device=dev)
        ln = torch.empty((n, stride), dtype=torch.int16, device=dev)
        ms = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.empty(n, dtype=torch.int32, device=dev)
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
        sc = L.CpSchedules(n, stride, words, 0, None, ops.data_ptr(), ln.data_ptr())
        up = None if upper is None else upper.to(device=dev, dtype=torch.int32).contiguous()
        rc = L.load().cp_exact(C.byref(d), C.byref(sc), _ptr(up), C.c_void_p(ms.data_ptr()), C.c_void_p(st.data_ptr()),
                               cap, int(max_plans), C.c_void_p(ws.data_ptr()), nb, _stream(s))
    L.check(rc, "cp_exact")
    return {"ops": ops, "len": ln, "makespan": ms, "status": st}


def exact_bnb(inst: Instances, *, upper=None, budget=2048, max_nodes=1 << 34, max_rounds=100000,
              front_cap=1 << 20, table_entries=1 << 20, stage_stride=None, stream=None):
    """cp_exact_bnb: the makespan-optimal split plan (n_sub = 1) of every tiny instance by parallel
    branch and bound on the GPU -> dict(ops, len, makespan, status, bound, nodes).  status 0 = proven
    optimal, CPI_INCOMPLETE (64) = stopped by a limit (bound = root lower bound).  upper: optional
    int32 [n] device tensor of feasible makespans (e.g. the greedy's), seeding the incumbent.  The
    call synchronizes its stream once per search round."""
    _require_cuda(inst.dev)
    dev = inst.dev.device
    n = inst.n
    stride = stage_stride or inst.max_pp
    words = max(1, (3 * min(inst.max_mb, 16) + 15) // 16)
    d = inst.desc(None)
    nb = int(L.load().cp_exact_bnb_workspace_bytes(C.byref(d), int(front_cap), int(table_entries)))
    with _on_stream(stream, inst.dev, upper) as s:
        ops = torch.empty((n, words, stride), dtype=torch.int32, device=dev)
        ln = torch.empty((n, stride), dtype=torch.int16, device=dev)
        ms = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.empty(n, dtype=torch.int32, device=dev)
        bd = torch.empty(n, dtype=torch.int32, device=dev)
        nd = torch.empty(n, dtype=torch.int64, device=dev)
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
        sc = L.CpSchedules(n, stride, words, 0, None, ops.data_ptr(), ln.data_ptr())
        up = None if upper is None else upper.to(device=dev, dtype=torch.int32).contiguous()
        rc = L.load().cp_exact_bnb(C.byref(d), C.byref(sc), _ptr(up), C.c_void_p(ms.data_ptr()),
                                   C.c_void_p(st.data_ptr()), C.c_void_p(bd.data_ptr()), C.c_void_p(nd.data_ptr()),
                                   int(budget), int(max_nodes), int(max_rounds), int(front_cap), int(table_entries),
                                   C.c_void_p(ws.data_ptr()), nb, _stream(s))
    L.check(rc, "cp_exact_bnb")
    return {"ops": ops, "len": ln, "makespan": ms, "status": st, "bound": bd, "nodes": nd}


def bubble_ratios(result: dict, n_pp):
    """Per-stage bubble ratios from simulate(..., stats=True) (reading Q7): local =
    1 - busy / (last_end - first_start) over the stage's active window, global = 1 - busy / makespan.
    n_pp: int or int tensor [n]; stages >= n_pp and items without a completed timeline give NaN.
    Returns (local, global), float64 tensors [n, stride] on the result's device."""
    st = result["stage_stats"].to(torch.float64)            # [n, stride, 4]: first, last, busy, peak
    ms = result["makespan"].to(torch.float64)[:, None]
    n, stride = st.shape[0], st.shape[1]
    pp = torch.as_tensor(n_pp, device=st.device).reshape(-1, 1)
    on = (torch.arange(stride, device=st.device)[None, :] < pp) & (result["status"][:, None] & ~2 == 0) & (ms > 0)
    win = st[..., 1] - st[..., 0]
    nan = torch.full_like(win, float("nan"))
    loc = torch.where(on & (win > 0), 1 - st[..., 2] / win.clamp(min=1), nan)
    glo = torch.where(on, 1 - st[..., 2] / ms.clamp(min=1), nan)
    return loc, glo


def to_cp_grid(grid) -> L.CpGrid:
    """workloads.Grid -> cp_grid (host struct, passed to the kernel by value)."""
    g = L.CpGrid()
    rec = pack_instances(grid.base)
    C.memmove(C.addressof(g.base), rec.ctypes.data, 1792)
    g.n_dc = int(grid.n_dc)
    if len(grid.pp_vals) > 8 or len(grid.mb_vals) > 8:
        raise ValueError("at most 8 n_pp / n_mb values")
    for i, v in enumerate(grid.pp_vals):
        g.n_pp_vals[i] = int(v)
    g.n_pp_n = len(grid.pp_vals)
    for i, v in enumerate(grid.mb_vals):
        g.n_mb_vals[i] = int(v)
    g.n_mb_n = len(grid.mb_vals)
    for name, cap in (("lat", L.GRID_MAX_AXIS), ("bw", L.GRID_MAX_AXIS), ("mlim_x1000", L.GRID_MAX_SMALL),
                      ("tdp", L.GRID_MAX_SMALL)):
        v = np.asarray(getattr(grid, name), dtype=np.int64)
        if len(v) > cap or (len(v) and (v.max() > INT32_MAX or v.min() < 0)):
            raise ValueError(f"grid axis {name}: at most {cap} int32 values >= 0")
        arr = getattr(g, name)
        for i, x in enumerate(v):
            arr[i] = int(x)
    g.n_lat, g.n_bw, g.n_mem, g.n_dp = len(grid.lat), len(grid.bw), len(grid.mlim_x1000), len(grid.tdp)
    g.cand_mask = int(grid.cand_mask)
    return g


def _sweep_buffers(g, npts, keys, cand, device):
    """Key table (INT64_MAX = not owned), optional per-candidate makespans, workspace; allocated and
    initialized on the current stream (the call's stream, under _on_stream)."""
    if keys is None:
        keys = torch.full((npts,), KEY_NONE, dtype=torch.int64, device=device)
    if cand is True:
        cm = torch.full((npts, L.N_CAND), -1, dtype=torch.int32, device=keys.device)
    else:
        cm = cand if cand is not False and cand is not None else None
    ws = torch.empty(int(L.load().cp_workspace_bytes(2, C.byref(g), 0)), dtype=torch.uint8, device=keys.device)
    return keys, cm, ws


def sweep_shard(grid, lo=0, hi=None, *, keys=None, cand=False, stream=None, device="cuda", cgrid=None):
    """cp_sweep_shard over points [lo, hi).  Returns (keys uint64-as-int64 [n_points], cand_ms or None).
    Keys outside [lo, hi) are INT64_MAX when `keys` is allocated here."""
    _require_cuda()
    g = cgrid if cgrid is not None else to_cp_grid(grid)
    npts = grid.n_points
    hi = npts if hi is None else hi
    with _on_stream(stream, keys) as s:
        keys, cm, ws = _sweep_buffers(g, npts, keys, cand, device)
        rc = L.load().cp_sweep_shard(C.byref(g), int(lo), int(hi), C.c_void_p(keys.data_ptr()),
                                     _ptr(cm), C.c_void_p(ws.data_ptr()), ws.numel(), _stream(s))
    L.check(rc, "cp_sweep_shard")
    return keys, cm


def sweep_shard_rank(grid, rank: int, world: int, *, keys=None, cand=False, stream=None, device="cuda", cgrid=None):
    """cp_sweep_shard_rank: the points rank `rank` of `world` owns under blocked ownership (slice
    `rank` of every (p, m) block).  Returns (keys int64 [n_points], cand_ms or None); keys of
    points not owned are INT64_MAX when `keys` is allocated here."""
    _require_cuda()
    g = cgrid if cgrid is not None else to_cp_grid(grid)
    npts = grid.n_points
    with _on_stream(stream, keys) as s:
        keys, cm, ws = _sweep_buffers(g, npts, keys, cand, device)
        rc = L.load().cp_sweep_shard_rank(C.byref(g), int(rank), int(world), C.c_void_p(keys.data_ptr()), _ptr(cm),
                                          C.c_void_p(ws.data_ptr()), ws.numel(), _stream(s))
    L.check(rc, "cp_sweep_shard_rank")
    return keys, cm


def sweep_partition(grid, world: int, cgrid=None):
    g = cgrid if cgrid is not None else to_cp_grid(grid)
    b = (C.c_int64 * (world + 1))()
    L.check(L.load().cp_sweep_partition(C.byref(g), int(world), b), "cp_sweep_partition")
    return [int(x) for x in b]


def decode_key(k: int):
    """packed sweep key -> (makespan, candidate) or None (no feasible candidate / overflow)."""
    k = int(k)
    if k >= KEY_OVER:
        return None
    return k >> 8, k & 0xFF


def quantize(spec: dict) -> tuple:
    """cp_quantize: SI spec dict -> (status, record numpy[1] of INST_DTYPE)."""
    s = L.CpSpecSI()
    for k, v in spec.items():
        if k in ("alpha", "beta"):
            arr = getattr(s, k)
            for i in range(min(4, len(v))):
                for j in range(min(4, len(v[i]))):
                    arr[i][j] = float(v[i][j])
        elif k == "dc_of_stage":
            arr = getattr(s, k)
            for i, x in enumerate(v):
                arr[i] = int(x)
        elif k in ("p", "m"):
            setattr(s, "n_pp" if k == "p" else "n_mb", int(v))
        elif isinstance(v, (list, tuple, np.ndarray)):
            arr = getattr(s, k)
            for i, x in enumerate(v):
                arr[i] = float(x)
        else:
            setattr(s, k, v)
    rec = np.zeros(1, dtype=L.INST_DTYPE)
    st = L.load().cp_quantize(C.byref(s), C.c_void_p(rec.ctypes.data))
    return int(st), rec


def validate_record(rec) -> tuple:
    buf = C.create_string_buffer(256)
    st = L.load().cp_validate_instance(C.c_void_p(rec.ctypes.data), buf, 256)
    return int(st), buf.value.decode()
