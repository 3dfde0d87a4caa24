#!/usr/bin/env python
"""Per-instruction view of an `ncu --page source --csv` dump: executed counts by opcode class and the
hottest instructions by stall samples."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iN, iSm = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('# Samples')
ops = collections.Counter(); samp = collections.Counter(); tot = 0; tsm = 0
lines = []
for r in rows[2:]:
    if len(r) <= iN: continue
    src = r[iS].strip()
    m = re.match(r'(@!?U?P\d+\s+)?([A-Z0-9_.]+)', src)
    op = m.group(2).split('.')[0] if m else '?'
    n = int(r[iN] or 0); s = int(r[iSm] or 0)
    ops[op] += n; samp[op] += s; tot += n; tsm += s
    lines.append((s, n, src))
print(f"total warp-instructions {tot}, samples {tsm}")
for op, n in ops.most_common(28):
    print(f"  {op:10s} {n:12d} {100*n/tot:5.1f}%   samples {100*samp[op]/max(tsm,1):5.1f}%")
if len(sys.argv) > 2:
    print('-- hottest instructions by samples')
    for s, n, src in sorted(lines, reverse=True)[:int(sys.argv[2])]:
        print(f"  {s:6d} {n:10d}  {src[:100]}")
