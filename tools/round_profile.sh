#!/bin/bash
# One GPU session of round-end evidence (run via gpurun from the repo root):
#   bench N=1 (default args, with the CPU baseline) and the reference arm; the ncu launch list of a
#   short bench; one --set full capture of k_sim32 at the bench launch size (1e6 config-4 schedules).
# usage: bash tools/round_profile.sh TAG
tag=${1:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; tail -1 gpurun_out/bench_n1_$tag.json | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; tail -1 gpurun_out/bench_ref_$tag.json | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sim32 -s 2 -c 1 -f -o gpurun_out/sim32_$tag \
    python tools/prof_sim.py sim 1000000 > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu full rc=$?"
