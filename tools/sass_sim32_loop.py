"""Static SASS inspection of k_sim32's n_sub == 1 round: prints the loop body between the branch
target before the entry-code funnel shift (SHF.R.W) and the backward branch after its VOTE.ANY."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2507_00217_b200/libcrosspipe.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "k_sim32ILb0E"
verbose = "-v" in sys.argv
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for b in out.split("Function : ")[1:]:
    name = b.split("\n")[0]
    if pat not in name:
        continue
    ins = [(int(a, 16), t) for a, t in re.findall(r'/\*([0-9a-f]{4})\*/\s+(.*?)\s*;', b)]
    for i, (a, t) in enumerate(ins):
        if "SHF.R.W" not in t:
            continue
        # the backward branch that closes this loop
        j = next(k for k in range(i, len(ins)) if "BRA" in ins[k][1] and
                 int(ins[k][1].split("0x")[-1], 16) < a and "@P" in ins[k][1])
        top = int(ins[j][1].split("0x")[-1], 16)
        body = [(x, s) for x, s in ins if top <= x <= ins[j][0]]
        print(name, "loop", hex(top), "->", hex(ins[j][0]), len(body), "instructions")
        if verbose:
            for x, s in body:
                print(" ", hex(x), s)
        break
