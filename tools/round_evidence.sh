#!/bin/bash
# Round-end evidence on one B200 (run via gpurun from the repo root): the default bench line (with the
# CPU baseline), the oracle arm, the ncu launch list of a short bench, and --set full captures of the
# bench kernel k_chunk32f<UD> (1e6 config-4 schedules) and of k_chunk32f<Wave> (2e5 plans).
# usage: bash tools/round_evidence.sh TAG
tag=${1:-r02}
python bench.py > gpurun_out/bench_n1_$tag.json 2> gpurun_out/bench_n1_$tag.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chunk32f -s 2 -c 1 -f -o gpurun_out/chunkf_ud_$tag \
    python tools/prof_sim.py sim 1000000 > gpurun_out/ncu_full_ud_$tag.log 2>&1; echo "ncu ud rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_chunk32f -s 2 -c 1 -f -o gpurun_out/chunkf_wave_$tag \
    python tools/prof_wave.py 200000 > gpurun_out/ncu_full_wave_$tag.log 2>&1; echo "ncu wave rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_greedy_fast -s 2 -c 1 -f -o gpurun_out/greedy_c3_$tag \
    python tools/prof_sim.py greedy 100000 > gpurun_out/ncu_full_greedy_$tag.log 2>&1; echo "ncu greedy rc=$?"
python tools/shard8.py > gpurun_out/shard8_$tag.txt 2>&1; echo "shard8 rc=$?"
