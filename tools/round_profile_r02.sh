#!/bin/bash
# Round-2 evidence in one GPU session (run via gpurun from the repo root):
#   ncu launch list of a short bench; one --set full capture of the config-4 first-pass kernel
#   (k_chunk32f<UD>, 1e6 schedules) and of the Wave one (2e5 plans); the paper artifacts.
# usage: bash tools/round_profile_r02.sh TAG
tag=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chunk32f -s 2 -c 1 -f -o gpurun_out/chunkf_ud_$tag \
    python tools/prof_sim.py sim 1000000 > gpurun_out/ncu_full_ud_$tag.log 2>&1; echo "ncu ud rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chunk32f -s 2 -c 1 -f -o gpurun_out/chunkf_wave_$tag \
    python tools/prof_wave.py 200000 > gpurun_out/ncu_full_wave_$tag.log 2>&1; echo "ncu wave rc=$?"
mkdir -p gpurun_out/paper
timeout 1200 bash tools/reproduce_paper.sh gpurun_out/paper > gpurun_out/paper_$tag.log 2>&1; echo "paper rc=$?"
