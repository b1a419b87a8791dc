#!/bin/bash
# A/B of the fast-path ring cap (CP_RING_CAP) on the bench (config 4 + config 3 greedy)
for cap in "$@"; do
  CP_RING_CAP=$cap python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep > gpurun_out/abr_$cap.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abr_$cap.log').read().strip().splitlines()[-1]);print('cap $cap', round(d['value']/1e6,3), 'M evals/s', round(d['greedy']['value']/1e6,2), 'M greedy/s', 'kern_ms', round(d['roofline']['kernel_ms'],2), 'ok', d['best_schedule']['all_status_ok'], d['greedy']['status_ok'])"
done
