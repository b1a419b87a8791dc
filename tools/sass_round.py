"""Static SASS inspection of the engine's round loop: prints its span (instruction slots between
the count-exchange SHFL.UP and the round-end VOTE) and the branches inside it."""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2507_00217_b200/libcrosspipe.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "ILi0ELb0ELb0E"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for b in out.split("Function : ")[1:]:
    name = b.split("\n")[0]
    if pat not in name:
        continue
    ins = [(int(a, 16), t) for a, t in re.findall(r'/\*([0-9a-f]{4})\*/\s+(.*?)\s*;', b)]
    ups = [a for a, t in ins if t.startswith('SHFL.UP') and ', 0x1,' in t]
    up = ups[-1]
    v = [a for a, t in ins if 'VOTE.ANY' in t and a > up]
    print(name, "round span", hex(up), "->", hex(v[0]), (v[0] - up) // 16, "slots; total", len(ins))
    print([(hex(a), t) for a, t in ins if up - 0x100 < a < v[0] + 0x40 and ('BRA' in t or 'BSSY' in t)])
