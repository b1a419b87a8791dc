"""Per-instruction execution counts from an ncu report's SASS source page, grouped into
regions of (nearly) equal execution count.  usage: python tools/sass_hist.py REP [n_items]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n_items = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex, ism = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ins = [(r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ism] or 0)) for r in rows[2:] if len(r) > iex]
tot = sum(x[2] for x in ins)
print(f"total warp-instr {tot:.4g}  per item {tot / n_items:.1f}")
# regions: consecutive instructions whose counts are within 2x of the region's first
reg = []
for a, s, c, sm in ins:
    if reg and c > 0 and reg[-1][1] > 0 and 0.5 < c / reg[-1][1] < 2:
        reg[-1][2] += c; reg[-1][3] += 1; reg[-1][5] += sm
    else:
        reg.append([a, c, c, 1, s, sm])
for a, c0, c, k, s, sm in sorted(reg, key=lambda r: -r[2])[:int(sys.argv[3]) if len(sys.argv) > 3 else 14]:
    print(f"{a[-5:]} n={k:4d} per-item {c / n_items:9.1f} ({100 * c / tot:5.1f}%) samples {sm:6d}  first: {s[:60]}")
