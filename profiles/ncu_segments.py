#!/usr/bin/env python
"""usage: ncu_segments.py REPORT.ncu-rep [min_samples] -- warp-stall samples of the (single) captured kernel,
grouped into runs of SASS instructions with the same execution count (= prologue / loop / epilogue
segments), plus the hottest instructions.  Needs a capture taken with --set full --import-source on."""
import csv, io, re, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iN, iSm = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('# Samples')
data = [(i, r[iS].strip(), int(r[iN] or 0), int(r[iSm] or 0)) for i, r in enumerate(rows[2:]) if len(r) > iN]
tot = sum(d[3] for d in data)
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 300
seg, cur = [], None
for i, s, n, sm in data:
    if cur is None or abs(n - cur[0]) > 0.02 * max(n, cur[0], 1):
        cur = [n, i, i, 0, 0]
        seg.append(cur)
    cur[2] = i; cur[3] += sm; cur[4] += 1
print(f"total samples {tot}, warp instructions {sum(d[2] for d in data)}")
for k, a, b, sm, cnt in seg:
    if sm > thr:
        print(f"exec={k:9d} idx {a:5d}-{b:5d} ninstr={cnt:4d} samples={sm:6d} {100 * sm / tot:5.1f}%")
print("-- hottest instructions")
for i, s, n, sm in sorted(data, key=lambda d: -d[3])[:25]:
    print(f"  {sm:6d} {100 * sm / tot:4.1f}% exec={n:9d} idx={i:5d}  {s[:90]}")
