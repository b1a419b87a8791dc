"""List the small loops (SHFL.UP ... VOTE.ANY spans) of a kernel with an opcode histogram:
python tools/sass_loops.py [lib] [kernel-substring] [--dump ADDR]"""
import collections, re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2507_00217_b200/libcrosspipe.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "k_sim32"
dump = int(sys.argv[4], 16) if len(sys.argv) > 4 and sys.argv[3] == "--dump" else None
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
ALU = {"ISETP", "SEL", "LOP3", "PLOP3", "VIMNMX", "VIMNMX3", "SHF", "IADD3", "LEA", "PRMT", "FLO", "POPC", "IABS", "P2R", "R2P"}
for b in out.split("Function : ")[1:]:
    name = b.split("\n")[0]
    if pat not in name:
        continue
    ins = [(int(a, 16), t) for a, t in re.findall(r'/\*([0-9a-f]{4})\*/\s+(.*?)\s*;', b)]
    votes = [a for a, t in ins if "VOTE.ANY" in t]
    for u in [a for a, t in ins if t.startswith("SHFL.UP")]:
        v = [x for x in votes if x > u]
        if not v:
            continue
        seg = [t for a, t in ins if u <= a <= v[0] + 0x30]
        if len(seg) > 200:
            continue
        ops = [re.sub(r"^@!?U?P[T0-9]\s+", "", t).split()[0].split(".")[0] for t in seg]
        c = collections.Counter(ops)
        print(name[:40], hex(u), "instr", len(seg), "alu", sum(c[k] for k in ALU), sorted(c.items(), key=lambda x: -x[1]))
        if dump == u:
            for a, t in ins:
                if u <= a <= v[0] + 0x30:
                    print(hex(a), t)
