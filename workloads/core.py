"""Neutral data formats + counter-based RNG (format conversions only, no method arithmetic)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F, B, D, W = 0, 1, 2, 3          # op codes (documented format)
MAXP = 32                        # stages per instance (warp-per-instance design)

_STAGE_FIELDS = ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag")
_BOUNDARY_FIELDS = ("lat_f", "bw_f", "lat_b", "bw_b")
STAGE_FIELDS = _STAGE_FIELDS
BOUNDARY_FIELDS = _BOUNDARY_FIELDS

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """splitmix64 finalizer (Steele et al.), vectorised over uint64 numpy arrays."""
    z = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & M64
    with np.errstate(over="ignore"):
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return z ^ (z >> np.uint64(31))


@dataclass
class InstanceBatch:
    """n problem instances in integer ticks / memory units (struct of arrays).

    Per-stage arrays are [n, 32]; boundary arrays are [n, 32] indexed by boundary
    s = link s->s+1 (``*_f``) / s+1->s (``*_b``), valid for s < p-1, zero elsewhere.
    """
    p: np.ndarray
    m: np.ndarray
    n_sub: np.ndarray
    zero1: np.ndarray
    t_f: np.ndarray
    t_d: np.ndarray
    t_w: np.ndarray
    m_f: np.ndarray
    m_d: np.ndarray
    m_w: np.ndarray
    m_lim: np.ndarray
    t_dp: np.ndarray
    t_ag: np.ndarray
    lat_f: np.ndarray
    bw_f: np.ndarray
    lat_b: np.ndarray
    bw_b: np.ndarray
    n_dc: np.ndarray = None
    tick_s: float = 1e-6

    @staticmethod
    def empty(n: int, tick_s: float = 1e-6) -> "InstanceBatch":
        z = lambda: np.zeros((n, MAXP), dtype=np.int64)  # noqa: E731
        zi = lambda: np.zeros(n, dtype=np.int32)  # noqa: E731
        return InstanceBatch(p=zi(), m=zi(), n_sub=np.ones(n, np.int32), zero1=zi(),
                             t_f=z(), t_d=z(), t_w=z(), m_f=z(), m_d=z(), m_w=z(), m_lim=z(),
                             t_dp=z(), t_ag=z(), lat_f=z(), bw_f=z(), lat_b=z(), bw_b=z(),
                             n_dc=np.ones(n, np.int32), tick_s=tick_s)

    def __len__(self):
        return int(self.p.shape[0])

    def take(self, idx) -> "InstanceBatch":
        idx = np.atleast_1d(np.asarray(idx))
        kw = {k: getattr(self, k)[idx] for k in ("p", "m", "n_sub", "zero1", "n_dc") + _STAGE_FIELDS + _BOUNDARY_FIELDS}
        return InstanceBatch(tick_s=self.tick_s, **kw)

    def item(self, i: int) -> dict:
        """Plain-dict view of instance i (python ints / int64 arrays trimmed to p)."""
        p = int(self.p[i])
        d = {"p": p, "m": int(self.m[i]), "n_sub": int(self.n_sub[i]), "zero1": int(self.zero1[i])}
        for k in _STAGE_FIELDS:
            d[k] = getattr(self, k)[i, :p].copy()
        for k in _BOUNDARY_FIELDS:       # boundary s = link s -> s+1 (s < p-1); index p-1: Loop's wrap link
            d[k] = getattr(self, k)[i, :p].copy()
        return d

    @staticmethod
    def concat(parts) -> "InstanceBatch":
        kw = {k: np.concatenate([getattr(b, k) for b in parts]) for k in
              ("p", "m", "n_sub", "zero1", "n_dc") + _STAGE_FIELDS + _BOUNDARY_FIELDS}
        return InstanceBatch(tick_s=parts[0].tick_s, **kw)


def cross_dc_boundaries(p: int, n_dc: int) -> np.ndarray:
    """Boolean [p-1]: boundary s is cross-DC when stages are split contiguously and
    evenly over min(n_dc, p) DCs, dc(s) = floor(s * n_dc / p)."""
    ndc = min(n_dc, p)
    s = np.arange(max(p - 1, 0))
    return (s * ndc // p) != ((s + 1) * ndc // p)


@dataclass
class Grid:
    """Sweep grid.  Axis values are pre-quantized integers."""
    base: InstanceBatch                  # one instance: per-stage costs, memory deltas, n_sub, zero1, t_ag
    n_dc: int
    pp_vals: list
    mb_vals: list
    lat: np.ndarray                      # cross-DC latency ticks
    bw: np.ndarray                       # cross-DC window ticks (beta * msg)
    mlim_x1000: np.ndarray               # m_lim[s] = (x * p * m_f[s] + 500) // 1000
    tdp: np.ndarray                      # DP allreduce ticks
    cand_mask: int = 0b11111             # bit0 GPipe, bit1 1F1B, bit2..4 greedy n_sub = 1,2,4, bit5 ZB-H1
    name: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n_points(self) -> int:
        return (len(self.pp_vals) * len(self.mb_vals) * len(self.lat) * len(self.bw)
                * len(self.mlim_x1000) * len(self.tdp))

    def point_axes(self, k):
        """Mixed-radix decode (i_pp, i_mb, i_lat, i_bw, i_mem, i_dp) of point k (vectorised)."""
        k = np.asarray(k, dtype=np.int64)
        i_dp = k % len(self.tdp); k = k // len(self.tdp)
        i_mem = k % len(self.mlim_x1000); k = k // len(self.mlim_x1000)
        i_bw = k % len(self.bw); k = k // len(self.bw)
        i_lat = k % len(self.lat); k = k // len(self.lat)
        i_mb = k % len(self.mb_vals); k = k // len(self.mb_vals)
        return k, i_mb, i_lat, i_bw, i_mem, i_dp


def pack_plans(codes: np.ndarray, lens: np.ndarray, stage_stride: int = None, words: int = None):
    """codes int8 [n, P, L], lens [n, P] -> (ops uint32 [n, words, stage_stride], len uint16 [n, stage_stride]).

    2-bit codes, 16 per 32-bit word, LSB first; word-major / stage-minor so that the
    32 lanes of a warp read word k of their own stage rows in one 128-B transaction.
    """
    codes = np.asarray(codes, dtype=np.uint32)
    n, P, L = codes.shape
    stage_stride = stage_stride or P
    words = words or max(1, (int(np.max(lens)) + 15) // 16 if lens.size else 1)
    Lp = words * 16
    c = np.zeros((n, P, Lp), dtype=np.uint32)
    c[:, :, :min(L, Lp)] = codes[:, :, :min(L, Lp)]
    mask = np.arange(Lp)[None, None, :] < np.asarray(lens)[:, :, None]
    c = np.where(mask, c, 0).reshape(n, P, words, 16)
    shifts = (2 * np.arange(16, dtype=np.uint32))[None, None, None, :]
    w = np.bitwise_or.reduce(c << shifts, axis=3)            # [n, P, words]
    ops = np.zeros((n, words, stage_stride), dtype=np.uint32)
    ops[:, :, :P] = np.transpose(w, (0, 2, 1))
    ln = np.zeros((n, stage_stride), dtype=np.uint16)
    ln[:, :P] = lens
    return ops, ln


def unpack_plans(ops: np.ndarray, lens: np.ndarray, p: int = None):
    """Inverse of pack_plans -> (codes int8 [n, P, words*16], len int32 [n, P])."""
    ops = np.asarray(ops, dtype=np.uint32)
    n, words, S = ops.shape
    P = p or S
    w = np.transpose(ops[:, :, :P], (0, 2, 1))[:, :, :, None]    # [n, P, words, 1]
    shifts = (2 * np.arange(16, dtype=np.uint32))[None, None, None, :]
    c = ((w >> shifts) & 3).reshape(n, P, words * 16).astype(np.int8)
    return c, np.asarray(lens)[:, :P].astype(np.int32)
