#!/bin/bash
# A/B bench of library variants in one GPU session: tools/ab.sh name1 name2 ...  ("base" = libcrosspipe.so)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset CROSSPIPE_LIB; else export CROSSPIPE_LIB=$PWD/paper_2507_00217_b200/libcrosspipe_$v.so; fi
  for rep in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_${v}_$rep.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$rep.log').read().strip().splitlines()[-1]);print('$v', round(d['value']/1e6,3), 'M evals/s', round(d['greedy']['value']/1e6,2), 'M greedy/s', 'kern_ms', round(d['roofline']['kernel_ms'],2))"
  done
done
