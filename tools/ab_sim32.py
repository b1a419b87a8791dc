"""A/B of k_sim32 launch variants in one process (environment switches are read per call):
config-4 cp_simulate over n resident plans, CUDA events around each launch, median and best.
usage: python tools/ab_sim32.py [n] [VAR=VAL,VAR=VAL ...]   (each argument after n is one variant;
"base" = no switches).  Also times the timeline mode when TL=1 is part of a variant."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_00217_b200 as cp  # noqa: E402
from workloads import configs as K, plans as PL  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
variants = sys.argv[2:] or ["base"]
b = K.perturbed_instance()
inst = cp.Instances(b)
ops, ln = PL.plans_device(b, n, seed=K.PERTURB_SEED)
ref = None
for rep in range(2):
    for v in variants:
        env = {} if v == "base" else dict(x.split("=", 1) for x in v.split(","))
        tl = env.pop("TL", "0") == "1"
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        out = cp.api._results(n, 32, False, tl, 16 * ops.shape[1], ops.device, True)
        ws = cp.api._workspace(0, inst.desc(), n, ops.device)
        for _ in range(3):
            out[0]["best_key"].fill_(cp.KEY_NONE)
            r = cp.simulate(inst, ops, ln, best=True, timeline=tl, ws=ws, out=out)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = cp.simulate(inst, ops, ln, best=True, timeline=tl, ws=ws, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = r["makespan"].clone()
        if ref is None:
            ref = ms
        ok = torch.equal(ms, ref)
        med, best = statistics.median(ts), min(ts)
        print(f"{v:40s} tl={int(tl)} median {med:.3f} ms ({n / med / 1e3:.2f} M/s)  best {best:.3f} ms "
              f"({n / best / 1e3:.2f} M/s) same={ok}", flush=True)
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val
        del out, ws, r
        torch.cuda.empty_cache()
