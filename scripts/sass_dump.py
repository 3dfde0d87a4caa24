#!/usr/bin/env python
"""usage: sass_dump.py OBJ KERNEL_SUBSTR LO HI -- SASS of a kernel between two addresses (hex)."""
import re, subprocess, sys
obj, key, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3], 16), int(sys.argv[4], 16)
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
on = False
for line in txt.splitlines():
    if "Function :" in line:
        on = key in line
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and lo <= int(m.group(1), 16) <= hi:
        print(f"{m.group(1)}  {m.group(2).strip()}")
