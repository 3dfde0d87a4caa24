#!/usr/bin/env python
"""usage: sass_ctrl.py OBJ KERNEL_SUBSTR LO HI -- SASS between two addresses (hex) with the decoded
scheduling control word: stall count, yield, write / read barrier, wait mask."""
import re, subprocess, sys
obj, key, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3], 16), int(sys.argv[4], 16)
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
on, pend = False, None
tot = 0
for line in txt.splitlines():
    if "Function :" in line:
        on = key in line
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* 0x([0-9a-f]+) \*/", line)
    if m:
        pend = (int(m.group(1), 16), m.group(2).strip())
        continue
    m = re.match(r"\s+/\* 0x([0-9a-f]+) \*/", line)
    if m and pend:
        w = int(m.group(1), 16)
        stall, yld, wb, rb, wm = (w >> 41) & 0xf, (w >> 45) & 1, (w >> 46) & 7, (w >> 49) & 7, (w >> 52) & 0x3f
        if lo <= pend[0] <= hi:
            tot += stall
            print(f"{pend[0]:05x} st={stall:2d} y={yld} wb={wb if wb != 7 else '-'} rb={rb if rb != 7 else '-'} wait={wm:02x}  {pend[1]}")
        pend = None
print("sum of stall counts", tot)
