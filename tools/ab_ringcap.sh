for cap in 4 8 16 32; do
  CP_RING_CAP=$cap python bench.py --steps 10 --warmup 3 --no-cpu --no-greedy --no-sweep > gpurun_out/ring_$cap.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ring_$cap.log').read().strip().splitlines()[-1]);print('cap $cap', round(d['value']/1e6,3), 'kern_ms', round(d['roofline']['kernel_ms'],2))"
done
