#!/bin/bash
# A/B of the SMSP-balanced block count (CP_NO_SMSP_BALANCE=1 restores the occupancy maximum)
for rep in 1 2; do
  for v in off on; do
    if [ $v = off ]; then export CP_NO_SMSP_BALANCE=1; else unset CP_NO_SMSP_BALANCE; fi
    python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), 'greedy', round(d['greedy']['value']/1e6,2), 'wave', round(d['wave']['value']/1e6,2), 'loop', round(d['loop']['value']/1e6,2), 'sweep5', round(d['sweep']['config5']['ms_per_sweep'],3), 'e2e', round(d['e2e']['value']/1e6,2))"
  done
done
