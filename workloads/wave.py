"""Multi-chunk plans (NEXT 1): Wave (reading Q32) and Loop (Q33) random valid plans and the 4-bit
packed layout.

Input generation only.  A plan gives every stage an ordered list of entries `type | chunk << 2`
(type F=0, B=1, D=2, W=3 as in the UD layout; chunk 0 or 1).  The packed layout holds 8 entries
per 32-bit word, LSB-first, in [item][word][stage_stride] order (include/crosspipe.h, entry_bits
= 4).  Random valid plans come from a token game over the Wave data flow: a stage may append an
entry once its inputs have been appended by their producers, so every plan is a topological
order of the Wave dependency graph (and never deadlocks).
"""
from __future__ import annotations

import numpy as np

F, B, D, W = 0, 1, 2, 3


def random_wave_plan(p: int, m: int, n_sub: int = 1, rng=None, combined: bool = False, w_bias: float = 0.3):
    """One random valid Wave plan -> list (per stage) of entry codes."""
    rng = rng or np.random.default_rng()
    nF = np.zeros((2, p), np.int64)
    nD = np.zeros((2, p), np.int64)
    nW = np.zeros((2, p), np.int64)          # W sub-blocks
    rows = [[] for _ in range(p)]
    total = p * 2 * m * (2 if combined else 2 + n_sub)
    done = 0

    def ready(s):
        r = []
        if nF[0, s] < m and (s == 0 or nF[0, s - 1] > nF[0, s]):
            r.append((F, 0))
        if nF[1, s] < m and ((nF[0, s] > nF[1, s]) if s == p - 1 else (nF[1, s + 1] > nF[1, s])):
            r.append((F, 1))
        if nD[1, s] < m and ((nF[1, s] > nD[1, s]) if s == 0 else (nD[1, s - 1] > nD[1, s])):
            r.append((B if combined else D, 1))
        if nD[0, s] < m and ((nD[1, s] > nD[0, s]) if s == p - 1 else (nD[0, s + 1] > nD[0, s])):
            r.append((B if combined else D, 0))
        if not combined:
            for c in (0, 1):
                if nW[c, s] < n_sub * nD[c, s]:
                    r.append((W, c))
        return r

    while done < total:
        cand = [(s, ready(s)) for s in range(p)]
        cand = [(s, r) for s, r in cand if r]
        s, r = cand[int(rng.integers(len(cand)))]
        ws = [x for x in r if x[0] == W]
        if ws and rng.random() < w_bias:
            t, c = ws[int(rng.integers(len(ws)))]
        else:
            t, c = r[int(rng.integers(len(r)))]
        rows[s].append(t | (c << 2))
        if t == F:
            nF[c, s] += 1
        elif t == W:
            nW[c, s] += 1
        else:
            nD[c, s] += 1
        done += 1
    return rows


def random_loop_plan(p: int, m: int, n_sub: int = 1, rng=None, combined: bool = False, w_bias: float = 0.3):
    """One random valid Loop plan (reading Q33, 2 chunks) -> list (per stage) of entry codes."""
    rng = rng or np.random.default_rng()
    nF = np.zeros((2, p), np.int64)
    nD = np.zeros((2, p), np.int64)
    nW = np.zeros((2, p), np.int64)
    rows = [[] for _ in range(p)]
    total = p * 2 * m * (2 if combined else 2 + n_sub)
    done = 0

    def ready(s):
        r = []
        if nF[0, s] < m and (s == 0 or nF[0, s - 1] > nF[0, s]):
            r.append((F, 0))
        if nF[1, s] < m and ((nF[0, p - 1] > nF[1, s]) if s == 0 else (nF[1, s - 1] > nF[1, s])):
            r.append((F, 1))
        if nD[1, s] < m and ((nF[1, s] > nD[1, s]) if s == p - 1 else (nD[1, s + 1] > nD[1, s])):
            r.append((B if combined else D, 1))
        if nD[0, s] < m and ((nD[1, 0] > nD[0, s]) if s == p - 1 else (nD[0, s + 1] > nD[0, s])):
            r.append((B if combined else D, 0))
        if not combined:
            for c in (0, 1):
                if nW[c, s] < n_sub * nD[c, s]:
                    r.append((W, c))
        return r

    while done < total:
        cand = [(s, ready(s)) for s in range(p)]
        cand = [(s, r) for s, r in cand if r]
        s, r = cand[int(rng.integers(len(cand)))]
        ws = [x for x in r if x[0] == W]
        if ws and rng.random() < w_bias:
            t, c = ws[int(rng.integers(len(ws)))]
        else:
            t, c = r[int(rng.integers(len(r)))]
        rows[s].append(t | (c << 2))
        if t == F:
            nF[c, s] += 1
        elif t == W:
            nW[c, s] += 1
        else:
            nD[c, s] += 1
        done += 1
    return rows


def pack_wave_plans(plans, stage_stride: int = None, words: int = None):
    """list of plans (each a list of per-stage entry lists) -> (ops uint32 [n, words, S], len uint16 [n, S])."""
    n = len(plans)
    S = stage_stride or max(len(pl) for pl in plans)
    L = max(max((len(r) for r in pl), default=0) for pl in plans)
    words = words or max(1, (L + 7) // 8)
    ops = np.zeros((n, words, S), np.uint32)
    ln = np.zeros((n, S), np.uint16)
    for i, pl in enumerate(plans):
        for s, row in enumerate(pl):
            ln[i, s] = len(row)
            for k, x in enumerate(row):
                ops[i, k // 8, s] |= np.uint32((int(x) & 15) << (4 * (k % 8)))
    return ops, ln


def unpack_wave_plans(ops: np.ndarray, lens: np.ndarray, p: int = None):
    """Inverse of pack_wave_plans -> (codes int8 [n, P, words*8], len int32 [n, P])."""
    ops = np.asarray(ops, dtype=np.uint32)
    n, words, S = ops.shape
    P = p or S
    w = np.transpose(ops[:, :, :P], (0, 2, 1))[:, :, :, None]
    shifts = (4 * np.arange(8, dtype=np.uint32))[None, None, None, :]
    c = ((w >> shifts) & 15).reshape(n, P, words * 8).astype(np.int8)
    return c, np.asarray(lens)[:, :P].astype(np.int32)
