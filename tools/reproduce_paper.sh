#!/bin/bash
# Regenerate every paper-analysis artifact under profiles/ on one B200 (about 2 minutes):
#   E1 delay-sensitivity grid relative to ZBV (§5.1), greedy vs exact on E1 replicas (m = 3, 4),
#   greedy vs exact on 2000 random tiny instances, E2 PP vs DP for Llama-3-405B (§5.2, App. E),
#   E3 GBS / memory / recomputation tables at the model level (§5.3).
# usage (from the repo root, via gpurun): bash tools/reproduce_paper.sh [out_dir]
set -e
out=${1:-profiles}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/e1_grid.py "$out/e1_delay_sensitivity_r01.json" > /dev/null
python tools/e1_exact.py 3 "$out/e1_exact_m3_r01.json"
python tools/e1_exact.py 4 "$out/e1_exact_m4_r01.json"
python tools/greedy_gap.py 2000 "$out/greedy_gap_r01.json" > /dev/null
python tools/e2_ppdp.py "$out/e2_pp_vs_dp_r01.json" > /dev/null
python tools/e3_table.py "$out/e3_gbs_memory_r01.json" > /dev/null
echo "paper artifacts written to $out"
