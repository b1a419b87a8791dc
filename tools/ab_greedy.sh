#!/bin/bash
# A/B of library variants on the greedy line and the sweeps: tools/ab_greedy.sh base name1 ...
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = "base" ]; then unset CROSSPIPE_LIB; else export CROSSPIPE_LIB=$PWD/paper_2507_00217_b200/libcrosspipe_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/abg_${v}_$rep.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/abg_${v}_$rep.log').read().strip().splitlines()[-1])
s=d['sweep']
print('$v', round(d['value']/1e6,2), 'M evals/s', round(d['greedy']['value']/1e6,2), 'M greedy/s', 'c2', round(s['config2']['ms_per_sweep']['median'],3), 'c5', round(s['config5']['ms_per_sweep']['median'],3), 'ms')"
done
done
