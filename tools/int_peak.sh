#!/bin/bash
# Integer-pipe peak (tools/int_peak.cu) with the SM clock sampled by nvidia-smi while it runs.
# usage (on a B200 box): bash tools/int_peak.sh > profiles/int_peak_rNN.jsonl
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peak tools/int_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 -i 0 \
  > /tmp/int_peak_clocks.csv 2>/dev/null &
SMI=$!
sleep 0.3
./tools/int_peak
kill $SMI 2>/dev/null || true
python3 - <<'PY'
import json, statistics
rows = [l.split(",") for l in open("/tmp/int_peak_clocks.csv") if l.strip()]
sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
print(json.dumps({"class": "clocks", "nvidia_smi_sm_mhz_median": statistics.median(sm) if sm else None,
                  "nvidia_smi_sm_mhz_min": min(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                  "samples": len(sm), "reasons_active": sorted({r[2].strip() for r in rows if len(r) > 2})}))
PY
