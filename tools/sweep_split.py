"""Time the config-5 sweep by candidate subset (static GPipe/1F1B vs greedy n_sub 1/2/4)."""
import os, sys, copy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_00217_b200 as cp
from workloads import configs as K

for name, grid in (("config5", K.full_sweep_grid()), ("config2", K.gpt16_grid())):
    for label, mask in (("all", grid.cand_mask), ("static", grid.cand_mask & 0b00011), ("greedy", grid.cand_mask & 0b11100),
                        ("g1", grid.cand_mask & 0b00100), ("g2", grid.cand_mask & 0b01000), ("g4", grid.cand_mask & 0b10000)):
        if mask == 0:
            continue
        g = copy.copy(grid); g.cand_mask = mask
        for _ in range(2):
            cp.sweep_shard(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            cp.sweep_shard(g)
        e1.record(); torch.cuda.synchronize()
        print(name, label, f"{e0.elapsed_time(e1) / 5:.3f} ms")
