"""List the short backward-branch loops of one kernel's SASS (dev tool).
usage: python tools/sass_loops.py LIB.so MANGLED_NAME [dump_from_hex dump_to_hex]"""
import re, subprocess, sys
lib, fn = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s+Function : ", txt)
body = next(b for b in blocks if b.startswith(fn))
ins = []
for l in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for addr, t in ins:
    mm = re.search(r"BRA.*0x([0-9a-f]+)", t)
    if mm:
        tgt = int(mm.group(1), 16)
        if tgt < addr and addr - tgt < 0x1000:
            b = [x for a, x in ins if tgt <= a <= addr]
            cnt = lambda k: sum(k in x for x in b)
            print(hex(tgt), hex(addr), len(b), "F2I", cnt("F2I"), "DADD", cnt("DADD"), "LDS", cnt("LDS"),
                  "STS", cnt("STS"), "ATOMS", cnt("ATOMS"), "RED", cnt("RED"), "VOTE", cnt("VOTE"))
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    for a, t in ins:
        if lo <= a <= hi:
            print(hex(a), t)
