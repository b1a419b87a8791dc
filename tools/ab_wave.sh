#!/bin/bash
# A/B of library variants x ring caps on the Wave / Loop lines: tools/ab_wave.sh "base w6" "8 4"
for rep in 1 2; do
for v in $1; do for cap in $2; do
  if [ "$v" = "base" ]; then unset CROSSPIPE_LIB; else export CROSSPIPE_LIB=$PWD/paper_2507_00217_b200/libcrosspipe_$v.so; fi
  CP_RING_CAP=$cap python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep --no-greedy --no-timeline > gpurun_out/abw_${v}_$cap.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/abw_${v}_$cap.log').read().strip().splitlines()[-1])
print('$v cap $cap', round(d['value']/1e6,2), 'M evals/s wave', round(d['wave']['value']/1e6,2), 'loop', round(d['loop']['value']/1e6,2))"
done; done; done
