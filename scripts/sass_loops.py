#!/usr/bin/env python
"""usage: sass_loops.py OBJ KERNEL_SUBSTR [min_body]  -- static opcode mix of every loop (backward branch)
of a kernel's SASS with at least `min_body` instructions, and of the whole kernel."""
import collections, re, subprocess, sys
obj, key = sys.argv[1], sys.argv[2]
min_body = int(sys.argv[3]) if len(sys.argv) > 3 else 200
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
ins, on = [], False
for line in txt.splitlines():
    if "Function :" in line:
        on = key in line
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
def opc(s):
    s = re.sub(r"^@!?U?P[0-9T]+\s+", "", s)
    return re.split(r"[ .]", s)[0]
def mix(lo, hi):
    c = collections.Counter(opc(s) for a, s in ins if lo <= a <= hi)
    n = sum(c.values())
    fp = c["DFMA"] + c["DADD"] + c["DMUL"]
    return n, fp, " ".join(f"{k}={v}" for k, v in c.most_common(16))
n, fp, m = mix(0, 1 << 40)
print(f"kernel: {n} instr, fp64 {fp}: {m}")
for a, s in ins:
    mm = re.search(r"BRA(?:\.\w+)*\s+(?:\w+,\s*)?0x([0-9a-f]+)", s)
    if mm and "BRA" in opc(s):
        t = int(mm.group(1), 16)
        if t < a:
            n, fp, m = mix(t, a)
            if n >= min_body:
                print(f"loop {t:#x}..{a:#x}: {n} instr, fp64 {fp}: {m}")
