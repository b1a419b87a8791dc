"""Debug-build repro: run greedy / simulate on small cases with libcrosspipe_dbg.so and print
the first bounds violation recorded by the engine (tag, idx, lim, item, thread, block)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CROSSPIPE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "paper_2507_00217_b200", "libcrosspipe_dbg.so")
import torch
import paper_2507_00217_b200 as cp
from paper_2507_00217_b200 import _lib
from workloads import configs as K
L = _lib.load()
buf = (ctypes.c_int * 8)()
print("start", flush=True)
for name, b in [("tiny", K.tiny(1.0, 0.5)), ("rand32", K.random_instances(50, seed=11, max_p=32, max_m=20))]:
    g = cp.greedy(cp.Instances(b), stats=True)
    torch.cuda.synchronize()
    L.cp_debug_read(buf)
    print(name, "dbg:", list(buf), "ms:", g["makespan"][:4].tolist(), "st:", g["status"][:4].tolist(), flush=True)
