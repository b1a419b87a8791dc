"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.
usage: python tools/launch_summary.py launches.csv "header line" > summary.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v = v / 1e3 if r[iu] in ("ns", "nsecond") else (v * 1e3 if r[iu] in ("ms", "msecond") else v)   # -> us
    tot[r[ik]] += v
    cnt[r[ik]] += 1
all_us = sum(tot.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print()
print("kernel | launches | total us | mean us | share of listed GPU time")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:90]} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {100 * tot[k] / all_us:.1f}%")
