"""Greedy occupancy-ring cap A/B: config-3 greedy time + fix-up count, config-5 sweep time + fix-up count.
usage: CP_GRING_CAP=16 python tools/gring_ab.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from paper_2507_00217_b200 import _lib as L
from workloads import configs as K

cap = os.environ.get("CP_GRING_CAP", "default")
gi = cp.Instances(K.greedy_batch(100_000))
for _ in range(2):
    r = cp.greedy(gi)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    r = cp.greedy(gi)
e1.record(); torch.cuda.synchronize()
ok = bool((r["status"] == 0).all().item()) if isinstance(r, dict) else None
print(f"cap {cap} config3 greedy {e0.elapsed_time(e1) / 5:.3f} ms status_ok {ok}")

grid = K.full_sweep_grid()
g = cp.to_cp_grid(grid)
npts = grid.n_points
ws = torch.empty(int(L.load().cp_workspace_bytes(2, C.byref(g), 0)), dtype=torch.uint8, device="cuda")
keys = torch.full((npts,), cp.KEY_NONE, dtype=torch.int64, device="cuda")
def run():
    L.check(L.load().cp_sweep_shard(C.byref(g), 0, npts, C.c_void_p(keys.data_ptr()), None,
                                    C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)), "sweep")
for _ in range(2):
    run()
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    run()
e1.record(); torch.cuda.synchronize()
nfix = int(ws[128:132].view(torch.int32).item())
ref_keys, _ = cp.sweep_shard(grid)
print(f"cap {cap} config5 sweep {e0.elapsed_time(e1) / 5:.3f} ms fixups {nfix} keys_equal_default_call {bool(torch.equal(keys, ref_keys))}")
