"""Independent re-formulations used to PIN the oracle (tests only).

Nothing here re-types the oracle's algorithm: the simulator below is the least fixed
point of the §3.5 start-time equations found by plain iteration, with
the link modelled as a FIFO queue (fig:comm_model caption: "the latter
messages need to wait for the previous ones to be placed on the transmission link
first") instead of the oracle's first-fit interval list, and no topological sort.
"""
from __future__ import annotations

import itertools

import numpy as np

F, B, D, W = 0, 1, 2, 3


def _label(codes, ns):
    out = []
    cF = cD = cW = 0
    for c in codes:
        c = int(c)
        if c == F:
            out.append((F, cF, 0)); cF += 1
        elif c in (B, D):
            out.append((c, cD, 0)); cD += 1
        else:
            out.append((W, cW // ns, cW % ns)); cW += 1
    return out


def _dur(d, s, typ, sub):
    ns = d["n_sub"]
    if typ == F:
        return int(d["t_f"][s])
    if typ == D:
        return int(d["t_d"][s])
    if typ == B:
        return int(d["t_d"][s] + d["t_w"][s])
    T = int(d["t_w"][s])
    return T // ns + (1 if sub < T % ns else 0)


def fp_simulate(d, codes):
    """Least fixed point of start(o) = max(end(prev on stage), arrivals of true preds).

    Returns dict(makespan, start[s][k], deadlock).  Deadlock <=> the iteration does not
    converge below a horizon bound (a cycle makes times grow without limit).
    """
    p, m = d["p"], d["m"]
    ops = [_label(codes[s], d["n_sub"]) for s in range(p)]
    st = [[0] * len(ops[s]) for s in range(p)]
    horizon = 1
    for s in range(p):
        horizon += sum(_dur(d, s, t, k) for (t, _, k) in ops[s])
        if d["zero1"]:
            horizon += int(d["t_ag"][s])
    for s in range(p - 1):
        horizon += m * int(d["lat_f"][s] + d["bw_f"][s] + d["lat_b"][s] + d["bw_b"][s])
    pos = [{} for _ in range(p)]
    for s in range(p):
        for k, (t, j, sub) in enumerate(ops[s]):
            pos[s][(t if t != B else D, j, sub)] = k
    for _ in range(10 * sum(len(o) for o in ops) + 10):
        end = [[st[s][k] + _dur(d, s, ops[s][k][0], ops[s][k][2]) for k in range(len(ops[s]))]
               for s in range(p)]
        # link arrivals: FIFO per directed boundary in producer (plan) order
        arrF = [dict() for _ in range(p)]   # arrF[s+1][j]
        arrD = [dict() for _ in range(p)]   # arrD[s-1][j]
        for s in range(p - 1):
            clk = None
            for k, (t, j, _) in enumerate(ops[s]):
                if t != F:
                    continue
                r = end[s][k]
                bw = int(d["bw_f"][s])
                ws = r if (bw == 0 or clk is None) else max(r, clk)
                if bw > 0:
                    clk = ws + bw
                arrF[s + 1][j] = ws + bw + int(d["lat_f"][s])
        for s in range(1, p):
            clk = None
            for k, (t, j, _) in enumerate(ops[s]):
                if t not in (D, B):
                    continue
                r = end[s][k]
                bw = int(d["bw_b"][s - 1])
                ws = r if (bw == 0 or clk is None) else max(r, clk)
                if bw > 0:
                    clk = ws + bw
                arrD[s - 1][j] = ws + bw + int(d["lat_b"][s - 1])
        changed = False
        for s in range(p):
            for k, (t, j, sub) in enumerate(ops[s]):
                v = end[s][k - 1] if k > 0 else 0
                if t == F:
                    if s > 0:
                        v = max(v, arrF[s][j])
                    if d["zero1"]:
                        v = max(v, int(d["t_ag"][s]))
                elif t in (D, B):
                    if s < p - 1:
                        v = max(v, arrD[s][j])
                    else:
                        v = max(v, end[s][pos[s][(F, j, 0)]])
                else:
                    v = max(v, end[s][pos[s][(D, j, 0)]])
                if v != st[s][k]:
                    st[s][k] = v
                    changed = True
                if v > horizon:
                    return {"deadlock": True, "makespan": -1, "start": st}
        if not changed:
            mk = 0
            for s in range(p):
                le = end[s][-1]
                mk = max(mk, le, le + int(d["t_dp"][s]))
                if d["zero1"]:
                    mk = max(mk, int(d["t_ag"][s]))
            return {"deadlock": False, "makespan": mk, "start": st}
    return {"deadlock": True, "makespan": -1, "start": st}


def fp_simulate_wave(d, codes):
    """Wave pattern (reading Q32) as the least fixed point of the §3.5 start-time equations.

    codes[s] = entries type | chunk << 2.  Per microbatch: F0 runs s -> s+1, turns to F1 on the
    last stage, F1 runs s -> s-1, the loss on stage 0 starts D1, D1 runs s -> s+1, turns to D0 on
    the last stage, D0 runs s -> s-1; W after the D of its chunk.  Each directed link carries its
    producer's messages in plan order through one FIFO clock (messages of both chunks share it).
    """
    p, m, ns = d["p"], d["m"], d["n_sub"]
    ops = []
    for s in range(p):
        cF, cD, cW = [0, 0], [0, 0], [0, 0]
        row = []
        for x in codes[s]:
            t, c = int(x) & 3, (int(x) >> 2) & 1
            if t == F:
                row.append((F, c, cF[c], 0)); cF[c] += 1
            elif t in (B, D):
                row.append((t, c, cD[c], 0)); cD[c] += 1
            else:
                row.append((W, c, cW[c] // ns, cW[c] % ns)); cW[c] += 1
        ops.append(row)
    pos = [{(t if t != B else D, c, j, q): k for k, (t, c, j, q) in enumerate(ops[s])} for s in range(p)]
    st = [[0] * len(ops[s]) for s in range(p)]
    horizon = 1
    for s in range(p):
        horizon += sum(_dur(d, s, t, q) for (t, c, j, q) in ops[s]) + int(d["t_ag"][s])
    for s in range(p - 1):
        horizon += 2 * m * int(d["lat_f"][s] + d["bw_f"][s] + d["lat_b"][s] + d["bw_b"][s])

    def link(end_s, s, right):
        """arrival times of the messages stage s sends right (F0, D1) or left (F1, D0)."""
        bw = int(d["bw_f"][s] if right else d["bw_b"][s - 1])
        lat = int(d["lat_f"][s] if right else d["lat_b"][s - 1])
        clk, arr = None, {}
        for k, (t, c, j, q) in enumerate(ops[s]):
            if t == W:
                continue
            goes_right = (t == F and c == 0) or (t != F and c == 1)
            if goes_right != right:
                continue
            r = end_s[k]
            ws = r if (bw == 0 or clk is None) else max(r, clk)
            if bw > 0:
                clk = ws + bw
            arr[(F if t == F else D, c, j)] = ws + bw + lat
        return arr

    for _ in range(20 * sum(len(o) for o in ops) + 10):
        end = [[st[s][k] + _dur(d, s, ops[s][k][0], ops[s][k][3]) for k in range(len(ops[s]))] for s in range(p)]
        right = [link(end[s], s, True) if s < p - 1 else {} for s in range(p)]
        left = [link(end[s], s, False) if s > 0 else {} for s in range(p)]
        changed = False
        for s in range(p):
            for k, (t, c, j, q) in enumerate(ops[s]):
                v = end[s][k - 1] if k > 0 else 0
                own = lambda key: end[s][pos[s][key]]
                # stage s hears F0 / D1 on s-1's rightward link, F1 / D0 on s+1's leftward link
                if t == F:
                    if c == 0:
                        v = max(v, right[s - 1][(F, 0, j)]) if s > 0 else v
                    else:
                        v = max(v, own((F, 0, j, 0))) if s == p - 1 else max(v, left[s + 1][(F, 1, j)])
                    if d["zero1"]:
                        v = max(v, int(d["t_ag"][s]))
                elif t in (B, D):
                    if c == 1:
                        v = max(v, own((F, 1, j, 0))) if s == 0 else max(v, right[s - 1][(D, 1, j)])
                    else:
                        v = max(v, own((D, 1, j, 0))) if s == p - 1 else max(v, left[s + 1][(D, 0, j)])
                else:
                    v = max(v, own((D, c, j, 0)))
                if v != st[s][k]:
                    st[s][k] = v
                    changed = True
                if v > horizon:
                    return {"deadlock": True, "makespan": -1, "start": st}
        if not changed:
            mk = 0
            for s in range(p):
                le = end[s][-1]
                mk = max(mk, le, le + int(d["t_dp"][s]))
                if d["zero1"]:
                    mk = max(mk, int(d["t_ag"][s]))
            return {"deadlock": False, "makespan": mk, "start": st}
    return {"deadlock": True, "makespan": -1, "start": st}


def fp_simulate_loop(d, codes):
    """Loop pattern, 2 chunks (reading Q33), as the least fixed point of the §3.5 equations.

    Per microbatch: F0 runs s -> s+1 and wraps p-1 -> 0 into F1; F1 runs s -> s+1; the loss on the
    last stage starts D1; D1 runs s -> s-1 and wraps 0 -> p-1 into D0; D0 runs s -> s-1; W after the
    D of its chunk.  Stage s sends right (its link s -> s+1, or the wrap p-1 -> 0 with boundary
    index p-1) and left (s -> s-1, or the wrap 0 -> p-1 with index p-1), one FIFO clock each.
    """
    p, m, ns = d["p"], d["m"], d["n_sub"]
    ops = []
    for s in range(p):
        cF, cD, cW = [0, 0], [0, 0], [0, 0]
        row = []
        for x in codes[s]:
            t, c = int(x) & 3, (int(x) >> 2) & 1
            if t == F:
                row.append((F, c, cF[c], 0)); cF[c] += 1
            elif t in (B, D):
                row.append((t, c, cD[c], 0)); cD[c] += 1
            else:
                row.append((W, c, cW[c] // ns, cW[c] % ns)); cW[c] += 1
        ops.append(row)
    pos = [{(t if t != B else D, c, j, q): k for k, (t, c, j, q) in enumerate(ops[s])} for s in range(p)]
    st = [[0] * len(ops[s]) for s in range(p)]
    horizon = 1
    for s in range(p):
        horizon += sum(_dur(d, s, t, q) for (t, c, j, q) in ops[s]) + int(d["t_ag"][s])
        horizon += 2 * m * int(d["lat_f"][s] + d["bw_f"][s] + d["lat_b"][s] + d["bw_b"][s])

    def link(end_s, s, right):
        if right:
            b = s                                        # s -> s+1, or the wrap p-1 -> 0
            bw, lat = int(d["bw_f"][b]), int(d["lat_f"][b])
        else:
            b = s - 1 if s > 0 else p - 1                # s -> s-1, or the wrap 0 -> p-1
            bw, lat = int(d["bw_b"][b]), int(d["lat_b"][b])
        clk, arr = None, {}
        for k, (t, c, j, q) in enumerate(ops[s]):
            if t == W:
                continue
            if right != (t == F):
                continue
            if right and s == p - 1 and c == 1:          # the last stage's F1 feeds its own D1
                continue
            if not right and s == 0 and c == 0:          # stage 0's D0 ends the chain
                continue
            r = end_s[k]
            ws = r if (bw == 0 or clk is None) else max(r, clk)
            if bw > 0:
                clk = ws + bw
            arr[(F if t == F else D, c, j)] = ws + bw + lat
        return arr

    for _ in range(20 * sum(len(o) for o in ops) + 10):
        end = [[st[s][k] + _dur(d, s, ops[s][k][0], ops[s][k][3]) for k in range(len(ops[s]))] for s in range(p)]
        right = [link(end[s], s, True) for s in range(p)]
        left = [link(end[s], s, False) for s in range(p)]
        changed = False
        for s in range(p):
            for k, (t, c, j, q) in enumerate(ops[s]):
                v = end[s][k - 1] if k > 0 else 0
                own = lambda key: end[s][pos[s][key]]
                if t == F:
                    if s > 0:
                        v = max(v, right[s - 1][(F, c, j)])
                    elif c == 1:
                        v = max(v, right[p - 1][(F, 0, j)])          # wrap p-1 -> 0
                    if d["zero1"]:
                        v = max(v, int(d["t_ag"][s]))
                elif t in (B, D):
                    if s < p - 1:
                        v = max(v, left[s + 1][(D, c, j)])
                    elif c == 1:
                        v = max(v, own((F, 1, j, 0)))                 # loss
                    else:
                        v = max(v, left[0][(D, 1, j)])                # wrap 0 -> p-1
                else:
                    v = max(v, own((D, c, j, 0)))
                if v != st[s][k]:
                    st[s][k] = v
                    changed = True
                if v > horizon:
                    return {"deadlock": True, "makespan": -1, "start": st}
        if not changed:
            mk = 0
            for s in range(p):
                le = end[s][-1]
                mk = max(mk, le, le + int(d["t_dp"][s]))
                if d["zero1"]:
                    mk = max(mk, int(d["t_ag"][s]))
            return {"deadlock": False, "makespan": mk, "start": st}
    return {"deadlock": True, "makespan": -1, "start": st}


def random_valid_plan(d, rng, p_w_first=0.3):
    """Random split plan (n_sub as in d) by a combinatorial random token game:
    uniformly pick a stage with an executable op (inputs produced, memory fits),
    then uniformly one of its executable ops.  No times involved."""
    p, m, ns = d["p"], d["m"], d["n_sub"]
    nF = [0] * p; nD = [0] * p; nW = [0] * p; mem = [0] * p
    codes = [[] for _ in range(p)]
    total = (2 + ns) * m * p
    done = 0
    while done < total:
        choices = []
        for s in range(p):
            opts = []
            if nF[s] < m and (s == 0 or nF[s - 1] > nF[s]) and mem[s] + d["m_f"][s] <= d["m_lim"][s]:
                opts.append(F)
            if nD[s] < m and ((s == p - 1 and nF[s] > nD[s]) or (s < p - 1 and nD[s + 1] > nD[s])):
                opts.append(D)
            if nW[s] < ns * nD[s]:
                opts.append(W)
            if opts:
                choices.append((s, opts))
        assert choices, "token game stuck"
        s, opts = choices[int(rng.integers(len(choices)))]
        c = opts[int(rng.integers(len(opts)))]
        codes[s].append(c)
        if c == F:
            nF[s] += 1; mem[s] += d["m_f"][s]
        elif c == D:
            nD[s] += 1; mem[s] += d["m_d"][s]
        else:
            nW[s] += 1
            if nW[s] % ns == 0:
                mem[s] += d["m_w"][s]
        done += 1
    return codes


def brute_force_opt(d):
    """min makespan over every per-stage ordering (multiset permutations of F^m D^m W^m,
    n_sub = 1), keeping those that are memory-feasible, W-after-D and deadlock-free."""
    p, m = d["p"], d["m"]
    base = [F] * m + [D] * m + [W] * m
    perms = sorted(set(itertools.permutations(base)))
    per_stage = []
    for s in range(p):
        ok = []
        for seq in perms:
            mem = peak = 0; nD = nW = 0; good = True
            for c in seq:
                if c == F:
                    mem += d["m_f"][s]
                elif c == D:
                    mem += d["m_d"][s]; nD += 1
                else:
                    mem += d["m_w"][s]; nW += 1
                    if nW > nD:
                        good = False; break
                peak = max(peak, mem)
            if good and peak <= d["m_lim"][s]:
                ok.append(seq)
        per_stage.append(ok)
    best = None
    for combo in itertools.product(*per_stage):
        r = fp_simulate(d, [list(x) for x in combo])
        if not r["deadlock"] and (best is None or r["makespan"] < best):
            best = r["makespan"]
    return best


def bubble(first, last, busy, makespan):
    """(local, global) bubble ratios of one stage (reading Q7)."""
    return 1.0 - busy / (last - first), 1.0 - busy / makespan
