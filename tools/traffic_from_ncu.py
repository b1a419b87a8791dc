"""Write profiles/traffic.json from one `ncu --set full` capture of the bench kernel (1e6 config-4
schedules): DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) and warp-instructions
per evaluation (smsp__inst_executed.sum / evaluations).  bench.py reads both (roofline.traffic,
roofline_issue).  usage: python tools/traffic_from_ncu.py REP.ncu-rep SUMMARY.txt KERNEL_LABEL [evals]"""
import csv
import json
import os
import subprocess
import sys

rep, summary, label = sys.argv[1], sys.argv[2], sys.argv[3]
evals = int(sys.argv[4]) if len(sys.argv) > 4 else 1_000_000
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
v = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(k):
    return float(v[k].replace(",", "")) * scale[u[k]]


rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
inst = float(v["smsp__inst_executed.sum"].replace(",", ""))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "traffic.json")
try:
    cur = json.load(open(path))
except Exception:
    cur = {}
cur.update({
    "_comment": f"dram__bytes_read.sum + dram__bytes_write.sum of {label} from one ncu --set full capture of the bench "
                f"launch size ({summary}: {evals:,} config-4 schedules, {rd / 1e9:.3f} GB read + {wr / 1e6:.2f} MB written). "
                "Algorithmic bytes: 1616 B per evaluation.",
    "simulate_config4_kernel": label,
    "simulate_config4_source": summary,
    "simulate_config4_bytes_per_eval": round((rd + wr) / evals, 1),
    "simulate_config4_bytes_per_launch": int(rd + wr),
    "simulate_config4_warp_instructions_per_eval": round(inst / evals, 1),
    "_comment_instructions": f"smsp__inst_executed.sum of the {label} capture {summary}: {int(inst):,} warp-instructions "
                             f"for {evals:,} config-4 evaluations",
})
json.dump(cur, open(path, "w"), indent=1)
print(json.dumps(cur, indent=1))
