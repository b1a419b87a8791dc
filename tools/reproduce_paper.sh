#!/bin/bash
# Regenerate every paper-analysis artifact under profiles/ on one B200 (a few minutes):
#   E1 delay-sensitivity grid relative to ZBV (§5.1), greedy vs exact on E1 replicas (m = 3, 4),
#   the exact optimum of the paper's 4 x 8 E1 setup by the GPU branch and bound, greedy vs exact on
#   2000 random tiny instances, E2 PP vs DP for Llama-3-405B (§5.2, App. E).
# usage (from the repo root, via gpurun): bash tools/reproduce_paper.sh [out_dir]
set -e
out=${1:-profiles}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/e1_grid.py "$out/e1_delay_sensitivity_r02.json" > /dev/null
python tools/e1_exact.py 3 "$out/e1_exact_m3_r02.json"
python tools/e1_exact.py 4 "$out/e1_exact_m4_r02.json"
python tools/bnb_gpu.py "$out/bnb_gpu_r02.json"
python tools/greedy_gap.py 2000 "$out/greedy_gap_r02.json" > /dev/null
python tools/e2_ppdp.py "$out/e2_pp_vs_dp_r02.json" > /dev/null
echo "paper artifacts written to $out"
