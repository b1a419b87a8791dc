"""List the loops (backward branches) of a kernel with an opcode histogram and ALU-pipe count:
python tools/sass_loops.py [lib] [kernel-substring] [--dump HEAD_ADDR] [--min N] [--max N]"""
import collections, re, subprocess, sys
args = sys.argv[1:]
opt = {}
while len(args) >= 2 and args[-2].startswith("--"):
    opt[args[-2][2:]] = args[-1]; args = args[:-2]
lib = args[0] if args else "paper_2507_00217_b200/libcrosspipe.so"
pat = args[1] if len(args) > 1 else "k_sim32"
dump = int(opt["dump"], 16) if "dump" in opt else None
lo, hi = int(opt.get("min", 30)), int(opt.get("max", 400))
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
ALU = {"ISETP", "SEL", "LOP3", "PLOP3", "VIMNMX", "VIMNMX3", "SHF", "IADD3", "LEA", "PRMT", "FLO", "POPC", "IABS", "P2R", "R2P"}
for b in out.split("Function : ")[1:]:
    name = b.split("\n")[0]
    if pat not in name:
        continue
    ins = [(int(a, 16), t) for a, t in re.findall(r'/\*([0-9a-f]{4})\*/\s+(.*?)\s*;', b)]
    for a, t in ins:
        m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        if not m or not m.group(1):
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a:
            continue
        seg = [x for y, x in ins if tgt <= y <= a]
        if not lo <= len(seg) <= hi:
            continue
        ops = [re.sub(r"^@!?U?P[T0-9]\s+", "", x).split()[0].split(".")[0] for x in seg]
        c = collections.Counter(ops)
        print(name[:40], hex(tgt), "instr", len(seg), "alu", sum(c[k] for k in ALU), sorted(c.items(), key=lambda x: -x[1]))
        if dump == tgt:
            for y, x in ins:
                if tgt <= y <= a:
                    print(hex(y), x)
