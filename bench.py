#!/usr/bin/env python3
"""bench.py -- CrossPipe hot path on B200: schedule evaluations/s (+ greedy schedules/s).

Default workload (BASELINE.json configs[3], the north-star's 1e7 evals/s target):
  config 4 -- 1e6 randomly perturbed valid schedules of one 32-stage, 4-DC, 64-microbatch
  instance per GPU (weak scaling), batched makespan + peak-memory evaluation through
  cp_simulate, argmin over the batch (best_key), all_reduce(MIN) across ranks.
Secondary (same run, reported under "greedy"): config 3 -- cp_greedy on 1e5 instances.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload perturbed|greedy|sweep2|sweep5]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...  (one rank per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SCHED = 1_000_000          # config 4 schedules per GPU
N_GREEDY = 100_000           # config 3 instances
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")
# measured integer throughput (tools/int_peak.sh on a B200): one JSON line per class alu/fma/mix, with the
# SM clock block 0 observed during the best launch and nvidia-smi's clock sampled while it ran
INT_PEAK_FILE = os.path.join(ROOT, "profiles", "int_peak_r02.jsonl")
# algorithmic bytes per config-4 evaluation: plan 32 stages x 12 words x 4 B + len 32 x 2 B
# + results (makespan 8 + peak 4 + status 4); the instance record (1792 B) is read once per launch
BYTES_PER_EVAL = 32 * 12 * 4 + 32 * 2 + 16
# algorithmic integer ops per evaluation, SURVEY.md §8(d)'s per-unit figure: ~8 per block
# (start max, end add, memory add, peak max, and the dependency bookkeeping: input/order checks and
# counter updates) x 6144 blocks + ~4 per message (window max, bw add, lat add, link update) x 3968
OPS_PER_EVAL = 8 * 6144 + 4 * 3968


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def int_peak(sm_max_mhz):
    """Integer lane-ops/s peak (Tops/s) for the ALU roofline: the measured rate of the mixed class
    (independent max/add/xor chains on the ALU pipe interleaved with IMAD chains on the FMA pipe --
    the algorithmic max/add ops can issue on either); fallback = the guide's unit counts: 148 SMs x
    4 SMSP x (16 ALU + 16 FMA lanes) per clock."""
    try:
        with open(INT_PEAK_FILE) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        mix = [r for r in rows if r.get("class") == "mix"][0]
        return mix["lane_ops_per_s"] / 1e12, "measured (tools/int_peak.cu, class mix)"
    except Exception:
        return 148 * 4 * 32 * sm_max_mhz * 1e6 / 1e12, "fallback (unit counts x clock)"


def traffic_per_launch(key="simulate_config4_bytes_per_launch"):
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def issue_roofline(evals_per_s, sm_hz):
    ipe = traffic_per_launch("simulate_config4_warp_instructions_per_eval")
    if not ipe or not sm_hz:
        return None
    peak = 148 * 4 * sm_hz                       # warp-instructions/s: 148 SMs x 4 schedulers x SM clock
    ach = ipe * evals_per_s
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-instr/s", "frac": ach / peak,
            "instructions_per_eval": ipe,
            "source": "ncu smsp__inst_executed.sum (" + str(traffic_per_launch("simulate_config4_source")) + ")",
            "sm_clock_hz": sm_hz}


class Clocks:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None
        self.path = os.path.join("/tmp", f"cp_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.idx)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1])); mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        bind_gpu_local_cpus(local)
    else:
        torch.cuda.set_device(0)
    return rank, ws, local


NUMA_BOUND = False


def bind_gpu_local_cpus(dev):
    """N > 1: pin this rank to the CPUs NVML reports as local to its GPU, so the pinned host buffers
    of the e2e leg (first touch by this process) land on the GPU's NUMA node.  Best effort."""
    global NUMA_BOUND
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        n = os.cpu_count() or 64
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            NUMA_BOUND = True
    except Exception:
        pass


def barrier(ws):
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, ws):
    import torch
    import torch.distributed as dist
    if ws == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------------- oracle (CPU) arm
# The oracle (oracle/, test infrastructure) as it stands, timed on the host cores on the same seeded
# inputs as the GPU legs: the cpu_baseline of every line and the --impl reference arm.  Inputs are
# regenerated per worker from their seeds (workloads/); only the oracle calls are inside the clock.
ORACLE_KINDS = {
    "config4": "config-4 schedules (ids from 0)",
    "config4_timeline": "config-4 schedules with the full start-tick timeline (ids from 0)",
    "greedy": "config-3 greedy instances (ids from 0)",
    "wave": "Wave bench plans (ids from 0)",
    "loop": "Loop bench plans (ids from 0)",
    "config2": "config-2 sweep points (all candidates), point k*7919 mod n: spread over the grid",
    "config5": "config-5 sweep points (all candidates), point k*7919 mod n: spread over the grid",
    "e1_delay_sensitivity": "E1 sweep points (all candidates), point k*7919 mod n: spread over the grid",
}


def _oracle_items(kind, lo, hi):
    """-> (list of zero-argument oracle calls for items [lo, hi) of `kind`)."""
    from oracle import oracle as O
    from workloads import configs as K, plans as PL, unpack_plans
    if kind in ("config4", "config4_timeline"):
        b = K.perturbed_instance()
        d = b.item(0)
        ops, ln = PL.plans_host(b, hi - lo, seed=K.PERTURB_SEED, id0=lo)
        codes, lens = unpack_plans(ops, ln)
        tl = kind == "config4_timeline"
        return [lambda i=i: O.simulate(d, codes[i], lens[i], timeline=tl) for i in range(hi - lo)]
    if kind == "greedy":
        batch = K.greedy_batch(hi - lo, id0=lo)
        return [lambda i=i: O.greedy(batch.item(i)) for i in range(hi - lo)]
    if kind in ("wave", "loop"):
        from workloads.wave import unpack_wave_plans
        loop = kind == "loop"
        d = (K.loop_instance() if loop else K.wave_instance()).item(0)
        ops, ln = PL.wave_plans_host(32, 32, 1, hi - lo, seed=K.PERTURB_SEED ^ 0x3A, id0=lo, q=1, stride=32, loop=loop)
        codes, lens = unpack_wave_plans(ops, ln)
        sim = O.simulate_loop if loop else O.simulate_wave
        return [lambda i=i: sim(d, codes[i], lens[i]) for i in range(hi - lo)]
    grid = {"config2": K.gpt16_grid, "config5": K.full_sweep_grid, "e1_delay_sensitivity": K.e1_grid}[kind]()
    G = O.to_or_grid(grid)[0]
    npts = grid.n_points
    return [lambda k=k: O.sweep_point(grid, (k * 7919) % npts, G=G) for k in range(lo, hi)]


def _oracle_job(job):
    """One worker: items [lo, hi) of `kind`, or (tmax > 0) as many as fit in about tmax seconds of
    oracle time, generated 256 at a time.  Returns (items done, oracle seconds)."""
    kind, lo, hi, tmax = job
    done, busy = 0, 0.0
    step = 256 if tmax > 0 else hi - lo
    a = lo
    while a < hi and not (tmax > 0 and busy > tmax):
        calls = _oracle_items(kind, a, min(hi, a + step))
        t = time.perf_counter()
        for f in calls:
            f()
            done += 1
            if tmax > 0 and busy + (time.perf_counter() - t) > tmax:
                break
        busy += time.perf_counter() - t
        a += step
    return done, busy


def oracle_rate(kind, cores, t_one=1.0, t_all=1.5):
    """The oracle on `kind`: (i) one host core for about t_one s; (ii) `cores` processes over disjoint
    slices sized from (i) to about t_all s each.  Returns the cpu_baseline dict."""
    from multiprocessing import get_context
    n1, s1 = _oracle_job((kind, 0, 1 << 30, t_one))
    r1 = n1 / s1
    per = max(1, int(r1 * t_all))
    jobs = [(kind, k * per, (k + 1) * per, 0.0) for k in range(cores)]
    t = time.perf_counter()
    with get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_job, jobs)
    wall = time.perf_counter() - t
    n = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"value": n / busy, "cores": cores, "kind": "oracle", "value_1core": r1,
            "sample": f"{n} {ORACLE_KINDS[kind]}, {cores} processes x {per}, {busy:.1f} s (pool wall {wall:.1f} s); "
                      f"1 core: {n1} in {s1:.1f} s"}


def oracle_throughput(n_total, cores):
    """config-4 oracle rate over `cores` processes on n_total schedules (the --impl reference arm)."""
    from multiprocessing import get_context
    per = max(1, n_total // cores)
    jobs = [("config4", k * per, (k + 1) * per, 0.0) for k in range(cores)]
    t = time.perf_counter()
    with get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_job, jobs)
    wall = time.perf_counter() - t
    n = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return n / busy, wall, n


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.build()
    cores = os.cpu_count() or 1
    n_step = 300 * cores                        # bounded sample per step (~0.4 s of CPU per core)
    for _ in range(args.warmup):
        oracle_throughput(cores, cores)
    vals = []
    t0 = time.perf_counter()
    n_done = 0
    for _ in range(args.steps):
        v, wall, n = oracle_throughput(n_step, cores)
        vals.append(v)
        n_done += n
    wall_total = time.perf_counter() - t0
    value = n_done / wall_total
    line = {"impl": "reference", "metric": "schedule evaluations/sec", "value": value, "unit": "evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall_total / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": "config4: perturbed valid schedules, p=32, 4 DCs, m=64 (bounded sample)",
                       "sample_per_step": n_step},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n_step} config-4 schedules per step, first ids of the GPU batch"},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------- GPU arm
# Algorithmic integer work per unit: a fixed-plan block costs 8 ops
# (start max, end add, memory add, peak max, and the dependency bookkeeping), a message 4 (window max,
# + bw, + lat, link-clock update); a greedy decision (one F/D block or W sub-block, Alg. 1 :388-432)
# costs the block's 8 plus 6 for its selection (three eligibility tests, t* = max(t_free, min avail),
# candidate filter, priority pick).
OPS_BLOCK, OPS_MSG, OPS_DECISION = 8, 4, 14


def ops_fixed(blocks, msgs):
    return OPS_BLOCK * blocks + OPS_MSG * msgs


def ops_greedy(p, m, n_sub):
    return OPS_DECISION * (2 + n_sub) * m * p + OPS_MSG * 2 * (p - 1) * m


def sweep_ops(grid, cand_ms):
    """Algorithmic ops of one sweep: every candidate the sweep had to evaluate (cand_ms >= 0: the ones
    not statically excluded; GPipe / 1F1B combined B, 2mp blocks; ZB-H1 3mp; greedy (2+n_sub)mp
    decisions), summed over points."""
    import numpy as np
    cm = cand_ms.cpu().numpy()
    inner = grid.n_points // (len(grid.pp_vals) * len(grid.mb_vals))
    tot = 0
    for ip, p in enumerate(grid.pp_vals):
        for im, m in enumerate(grid.mb_vals):
            k0 = (ip * len(grid.mb_vals) + im) * inner
            ev = (cm[k0:k0 + inner] >= 0).sum(axis=0)
            msgs = 2 * (p - 1) * m
            per = [ops_fixed(2 * m * p, msgs), ops_fixed(2 * m * p, msgs), ops_greedy(p, m, 1),
                   ops_greedy(p, m, 2), ops_greedy(p, m, 4), ops_fixed(3 * m * p, msgs)]
            tot += int(sum(int(ev[c]) * per[c] for c in range(min(len(per), cm.shape[1]))))
    return tot


def event_times(fn, steps, stream):
    """CUDA-event time of each of `steps` back-to-back launches of fn() on `stream` (ms list)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    out = None
    for a, b in ev:
        a.record(stream)
        out = fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev], out


def tstats(ts):
    return {"mean": statistics.mean(ts), "median": statistics.median(ts), "best": min(ts)}


def alu_roofline(ops_per_launch, ms, peak, src, kernel):
    ach = ops_per_launch / (ms / 1e3) / 1e12
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Tops/s", "frac": ach / peak, "traffic": None,
            "peak_source": src, "kernel": kernel, "ops_per_launch": ops_per_launch, "kernel_ms": ms}


def run_ours(args):
    import torch

    import paper_2507_00217_b200 as cp
    from paper_2507_00217_b200 import dist as cpd
    from workloads import configs as K, plans as PL

    rank, ws, local = dist_setup(args)
    hbm_peak, sm_max, peak_src = peaks()
    alu_peak, alu_src = int_peak(sm_max)                        # Tops/s
    cores = os.cpu_count() or 1
    want_cpu = ws == 1 and not args.no_cpu and rank == 0
    b = K.perturbed_instance()
    inst = cp.Instances(b)
    n = args.n or N_SCHED
    # each rank evaluates its own n schedules (ids rank*n ...): weak scaling
    ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED, id0=rank * n)
    stream = torch.cuda.current_stream()
    # best_key carries global schedule ids (rank * n + i), so the cross-rank MIN names a traceable schedule
    out = cp.api._results(n, 32, False, False, 0, ops.device, True, index_base=rank * n)
    ws_buf = cp.api._workspace(0, inst.desc(), n, ops.device)

    def step():
        r = cp.simulate(inst, ops, ln, best=True, ws=ws_buf, out=out)
        cpd.best_schedule(r["best_key"])
        return r

    for _ in range(args.warmup):
        step()
    barrier(ws)
    clocks = Clocks(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ss = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier(ws)
    e0.record(stream)
    ss[0].record(stream)
    for i in range(args.steps):
        ks[i][0].record(stream)
        r = cp.simulate(inst, ops, ln, best=True, ws=ws_buf, out=out)
        ks[i][1].record(stream)
        cpd.best_schedule(r["best_key"])
        ss[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms_local = e0.elapsed_time(e1)
    k_ts = [a.elapsed_time(b_) for a, b_ in ks]
    s_ts = [ss[i].elapsed_time(ss[i + 1]) for i in range(args.steps)]
    kern_ms = statistics.mean(k_ts)
    clk = clocks.stop() if clocks else None
    sm_clk_hz = (clk or {}).get("sm_mhz")
    sm_clk_hz = sm_clk_hz * 1e6 if sm_clk_hz else None
    ms_tot = max_over_ranks(ms_local, ws)
    kern_ms = max_over_ranks(kern_ms, ws)
    kern_med = max_over_ranks(statistics.median(k_ts), ws)
    kern_best = max_over_ranks(min(k_ts), ws)
    step_med = max_over_ranks(statistics.median(s_ts), ws)
    step_best = max_over_ranks(min(s_ts), ws)
    value = ws * n * args.steps / (ms_tot / 1e3)
    best = int(out[0]["best_key"][0].item())
    status_ok = bool((out[0]["status"] == 0).all().item())
    del out

    # ---------------- secondary: timeline mode (full start-tick timelines requested,
    # 24.6 KB/eval, the HBM-bound variant): the same config-4 step with every entry's start tick written
    timeline = None
    if not args.no_timeline:
        tl_out = cp.api._results(n, 32, False, True, 16 * ops.shape[1], ops.device, True, index_base=rank * n)
        for _ in range(3):
            cp.simulate(inst, ops, ln, best=True, timeline=True, ws=ws_buf, out=tl_out)
        barrier(ws)
        ts, r_tl = event_times(lambda: cp.simulate(inst, ops, ln, best=True, timeline=True, ws=ws_buf, out=tl_out),
                               max(3, min(args.steps, 5)), stream)
        t = tstats(ts)
        t = {k: max_over_ranks(v, ws) for k, v in t.items()}
        tl_bytes = BYTES_PER_EVAL + 4 * 32 * 16 * ops.shape[1]      # + the 32 x 192 int32 start ticks
        ach = tl_bytes * n / (t["median"] / 1e3) / 1e9
        timeline = {"value": ws * n / (t["median"] / 1e3), "unit": "evals/s",
                    "workload": "config4 with the full timeline (t_start, 32 x 192 int32 per schedule)",
                    "ms_per_launch": t, "status_ok": bool((r_tl["status"] == 0).all().item()),
                    "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": ach / hbm_peak, "traffic": traffic_per_launch("simulate_timeline_bytes_per_launch"),
                                 "peak_source": peak_src, "bytes_per_eval": tl_bytes,
                                 "kernel": "k_chunk32f<UD, timeline> (start ticks staged in smem, 32 B per lane store)"}}
        del tl_out, r_tl
        torch.cuda.empty_cache()

    # ---------------- e2e: same metric through the public API with HOST buffers (pinned):
    # cp.HostPipeline overlaps each chunk's H2D copy with the previous chunk's kernel and streams
    # results back (D2H) -- the copies are inside the timed region every step
    ops_h = torch.empty(ops.shape, dtype=ops.dtype, pin_memory=True)
    ln_h = torch.empty(ln.shape, dtype=ln.dtype, pin_memory=True)
    ops_h.copy_(ops); ln_h.copy_(ln)
    ms_h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    pk_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    st_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    del ops, ln, ws_buf
    torch.cuda.empty_cache()
    pipe = cp.HostPipeline(inst, n, ops_h.shape[1], ops_h.shape[2], chunks=args.chunks, index_base=rank * n)
    for _ in range(2):
        pipe.run(ops_h, ln_h, ms_h, pk_h, st_h)
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5))
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        bk = pipe.run(ops_h, ln_h, ms_h, pk_h, st_h)
        cpd.best_schedule(bk)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, ws)
    e2e_val = ws * n * e2e_steps / e2e_s
    e2e_ok = int(bk[0].item()) == best and bool((st_h == 0).all().item())
    h2d = ops_h.numel() * 4 + ln_h.numel() * 2
    d2h = n * (8 + 4 + 4)
    del pipe
    # the e2e leg's ceiling: a plain pinned -> device copy of the same plan bytes on this box (PCIe;
    # each rank measures its own copy alone)
    dst = torch.empty(ops_h.shape, dtype=ops_h.dtype, device="cuda")
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst.copy_(ops_h, non_blocking=True)
    c0.record()
    for _ in range(3):
        dst.copy_(ops_h, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_peak = 3 * ops_h.numel() * 4 / (c0.elapsed_time(c1) / 1e3) / 1e9
    h2d_achieved = h2d * e2e_steps / e2e_s / 1e9                 # per GPU: one rank's bytes / step time
    del dst, ops_h, ln_h

    # ---------------- secondary: config 3 greedy schedules/s (same run)
    greedy = None
    if not args.no_greedy:
        gb = K.greedy_batch(args.n_greedy or N_GREEDY, seed=K.SEED + rank)
        ginst = cp.Instances(gb)
        gws = cp.api._workspace(1, ginst.desc(), ginst.n, "cuda")
        for _ in range(3):
            g = cp.greedy(ginst, ws=gws)
        barrier(ws)
        ts, g = event_times(lambda: cp.greedy(ginst, ws=gws), max(3, min(args.steps, 5)), stream)
        t = {k: max_over_ranks(v, ws) for k, v in tstats(ts).items()}
        g_ops = sum(ops_greedy(int(gb.p[i]), int(gb.m[i]), int(gb.n_sub[i])) for i in range(len(gb)))
        greedy = {"value": ws * ginst.n / (t["median"] / 1e3), "unit": "greedy schedules/s",
                  "workload": "config3: 1e5 instances/GPU, p=16, 2 DCs, m=32, n_sub 1/2/4, memory x DP x ZeRO-1 grid",
                  "ms_per_launch": t, "status_ok": bool((g["status"] == 0).all().item()),
                  "roofline": alu_roofline(g_ops, t["median"], alu_peak, alu_src, "k_greedy_fast<16> (cp_greedy)")}
        if want_cpu:
            greedy["cpu_baseline"] = dict(oracle_rate("greedy", cores), unit="greedy schedules/s")
        del gws, g

    # ---------------- secondary: two-chunk patterns (NEXT 1): Wave (reading Q32) and Loop (Q33), 2e5
    # random valid plans per GPU of one p=32 / 4-DC / m=32 instance (192 entries per stage, as config 4)
    wave = loop = None
    if not args.no_wave:
        for name, b_, is_loop in (("wave", K.wave_instance(), False), ("loop", K.loop_instance(), True)):
            winst = cp.Instances(b_)
            nw = args.n_wave or 200_000
            wops, wln = PL.wave_plans_device(32, 32, 1, nw, seed=K.PERTURB_SEED ^ 0x3A, id0=rank * nw, q=1, stride=32,
                                             loop=is_loop)
            kw = {"loop": True} if is_loop else {"wave": True}
            for _ in range(3):
                wr = cp.simulate(winst, wops, wln, best=True, index_base=rank * nw, **kw)
            barrier(ws)
            ts, wr = event_times(lambda: cp.simulate(winst, wops, wln, best=True, index_base=rank * nw, **kw),
                                 max(3, min(args.steps, 5)), stream)
            t = {k: max_over_ranks(v, ws) for k, v in tstats(ts).items()}
            # per plan: 6 m p blocks (F, D, W of two chunks); 4(p-1)m messages (+ 2m over Loop's wraps)
            w_ops = nw * ops_fixed(6 * 32 * 32, 4 * 31 * 32 + (2 * 32 if is_loop else 0))
            line_w = {"value": ws * nw / (t["median"] / 1e3), "unit": "evals/s",
                      "workload": ("Loop (2 chunks, wrap-around links)" if is_loop else "Wave (2 chunks, V)") +
                                  ": 2e5 random valid plans/GPU of one p=32, 4-DC, m=32 instance (L=T_F, T_bw=T_F/2), "
                                  "makespan + peak memory + argmin",
                      "ms_per_launch": t, "status_ok": bool((wr["status"] == 0).all().item()),
                      "roofline": alu_roofline(w_ops, t["median"], alu_peak, alu_src, "k_chunk32f<Wave|Loop> (cp_simulate first pass, two-chunk)")}
            if want_cpu:
                line_w["cpu_baseline"] = dict(oracle_rate(name, cores), unit="evals/s")
            if is_loop:
                loop = line_w
            else:
                wave = line_w
            del wops, wln, wr

    # ---------------- secondary: sweeps (config 2 on one GPU's shard, config 5 sharded over all
    # ranks with one all_reduce(MIN) of the packed keys inside the timed region)
    sweeps = None
    if not args.no_sweep:
        sweeps = {}
        for name, grid, ncand in (("config2", K.gpt16_grid(), 3), ("config5", K.full_sweep_grid(), 5),
                                  ("e1_delay_sensitivity", K.e1_grid(), 6)):
            # blocked ownership (cp_sweep_shard_rank): every rank evaluates its slice of every (p, m)
            # block, then one all_reduce(MIN) of the keys inside the timed region
            for _ in range(3):
                keys, _ = cpd.sweep(grid)
            barrier(ws)
            ts, (keys, _) = event_times(lambda: cpd.sweep(grid), 5, stream)
            t = {k: max_over_ranks(v, ws) for k, v in tstats(ts).items()}
            feas = int((keys < cp.KEY_OVER).sum().item())
            _, cm = cp.sweep_shard(grid, cand=True)             # untimed: which candidates were evaluated
            s_ops = sweep_ops(grid, cm)
            sweeps[name] = {"points": grid.n_points, "candidates_per_point": ncand, "ms_per_sweep": t,
                            "points_per_s": grid.n_points / (t["median"] / 1e3),
                            "candidate_evals_per_s": grid.n_points * ncand / (t["median"] / 1e3),
                            "feasible_points": feas, "workload": grid.name,
                            "roofline": alu_roofline(s_ops, t["median"], alu_peak, alu_src,
                                                     "k_greedy_fast<W, grid> + k_engine<SWEEP> (cp_sweep_shard)")}
            if want_cpu:
                sweeps[name]["cpu_baseline"] = dict(oracle_rate(name, cores), unit="points/s")

    if rank == 0:
        achieved = BYTES_PER_EVAL * n / (kern_med / 1e3) / 1e9
        alu_ach = OPS_PER_EVAL * n / (kern_med / 1e3) / 1e12
        line = {
            "metric": "schedule evaluations/sec", "value": value, "unit": "evals/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_tot / args.steps,
            "ms_per_step_median": step_med, "ms_per_step_best": step_best,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": "config4: 1e6 randomly perturbed valid schedules/GPU of one p=32, 4-DC, m=64 "
                                   "instance (L=T_F, T_bw=T_F/2, M_L=1.5x 1F1B), makespan + peak memory + argmin",
                       "schedules_per_gpu": n, "parallelism": f"dp{ws} (shard schedules, all_reduce MIN)",
                       "l2": "inputs 1.6 GB/GPU > 126 MB L2 (no flush needed)"},
            # the binding roofline: integer arithmetic; HBM reported beside it; fractions
            # from the median launch
            "roofline": {"bound": "alu", "achieved": alu_ach, "peak": alu_peak, "unit": "Tops/s",
                         "frac": alu_ach / alu_peak, "traffic": traffic_per_launch(),
                         "peak_source": alu_src,
                         "kernel": traffic_per_launch("simulate_config4_kernel") or "cp_simulate first pass",
                         "kernel_ms": kern_ms, "kernel_ms_median": kern_med, "kernel_ms_best": kern_best,
                         "ops_per_eval": OPS_PER_EVAL, "evals_per_launch": n},
            # the integer-issue ceiling SURVEY.md §8(d) names: 4 warp-instructions per clock per SM; the
            # instructions per evaluation come from the committed ncu capture (profiles/traffic.json)
            "roofline_issue": issue_roofline(n / (kern_med / 1e3), sm_clk_hz),       # per GPU
            "roofline_hbm": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                             "frac": achieved / hbm_peak, "traffic": traffic_per_launch(),
                             "peak_source": peak_src, "bytes_per_eval": BYTES_PER_EVAL},
            "cpu_baseline": None,
            "e2e": {"value": e2e_val, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": f"cp.HostPipeline ({args.chunks} chunks, copy/compute overlap)", "matches_device_run": e2e_ok,
                    "host_cpus_bound_to_gpu_numa_node": NUMA_BOUND,
                    "h2d_GBps_per_gpu": round(h2d_achieved, 2),
                    "h2d_copy_ceiling_GBps_per_gpu": round(h2d_peak, 2)},
            "gpu_launches": 2 * args.steps,
            "clocks": clk,
            "timeline": timeline,
            "greedy": greedy,
            "wave": wave,
            "loop": loop,
            "sweep": sweeps,
            "best_schedule": {"makespan_ticks": best >> 32, "index": best & 0xFFFFFFFF, "all_status_ok": status_ok},
        }
        if want_cpu:
            line["cpu_baseline"] = dict(oracle_rate("config4", cores, t_one=1.0, t_all=2.0), unit="evals/s")
            if timeline is not None:
                timeline["cpu_baseline"] = dict(oracle_rate("config4_timeline", cores), unit="evals/s")
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="schedules per GPU (default 1e6)")
    ap.add_argument("--n-greedy", type=int, default=0)
    ap.add_argument("--no-greedy", action="store_true")
    ap.add_argument("--n-wave", type=int, default=0, help="Wave plans per GPU (default 2e5)")
    ap.add_argument("--no-wave", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-timeline", action="store_true")
    ap.add_argument("--chunks", type=int, default=32, help="e2e host pipeline chunks (32: 33.5 M vs 8: 31.8 M evals/s, the H2D copy ceiling is ~34.7 M)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
