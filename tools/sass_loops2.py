"""Backward-branch loops of one kernel's SASS with their size and marker-op counts (dev tool).
usage: python tools/sass_loops2.py LIB.so MANGLED_NAME [marker ...]"""
import re, subprocess, sys
so, name = sys.argv[1], sys.argv[2]
marks = sys.argv[3:] or ["FFMA2"]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
body, on = [], False
for ln in out.splitlines():
    if "Function : " in ln:
        on = ln.strip().endswith(name)
        continue
    if on:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(body)}
for i, (a, ins) in enumerate(body):
    m = re.search(r"BRA (?:`\(.*?\))?\s*0x([0-9a-f]+)", ins)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            seg = body[addr[tgt]:i + 1]
            cnt = {k: sum(1 for _, x in seg if k in x) for k in marks}
            if any(cnt.values()):
                print(f"loop {hex(tgt)}..{hex(a)}: {len(seg)} instrs {cnt}")
