"""A/B of cp_greedy (config 3) between library builds whose cp_greedy ABI is identical:
python tools/greedy_ab_lib.py lib1.so lib2.so ..."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from paper_2507_00217_b200 import _lib as L, api
from workloads import configs as K

gi = cp.Instances(K.greedy_batch(100_000))
ref = cp.greedy(gi)                                # allocate outputs / workspace with the current lib
n, stride = gi.n, gi.max_pp
words = ref["ops"].shape[1]
d = gi.desc(None)
ws = api._workspace(1, d, n, gi.dev.device)
P = C.POINTER
for path in sys.argv[1:]:
    lib = C.CDLL(path)
    lib.cp_greedy.restype = C.c_int32
    lib.cp_greedy.argtypes = [P(L.CpInstances), P(L.CpSchedules), P(L.CpResults), C.c_void_p, C.c_size_t, C.c_void_p]
    r, cres = api._results(n, stride, False, False, 16 * words, gi.dev.device, False)
    ops = torch.empty((n, words, stride), dtype=torch.int32, device="cuda")
    ln = torch.empty((n, stride), dtype=torch.int16, device="cuda")
    sc = L.CpSchedules(n, stride, words, 0, None, ops.data_ptr(), ln.data_ptr())
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    call = lambda: lib.cp_greedy(C.byref(d), C.byref(sc), C.byref(cres), C.c_void_p(ws.data_ptr()), ws.numel(), st)
    for _ in range(3):
        assert call() == 0
    torch.cuda.synchronize()
    best = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            call()
        e1.record(); torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / 10)
    same = torch.equal(r["makespan"], ref["makespan"])
    print(os.path.basename(path), "ms per launch", [round(x, 3) for x in best], "makespans equal current", same)
