#!/usr/bin/env python
"""One line per captured launch from an .ncu-rep: duration, DRAM bytes, DRAM %, occupancy, top stalls."""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
def g(r, k):
    return r[hdr.index(k)] if k in hdr else ''
for r in rows[2:]:
    st = sorted([(float(r[i] or 0), h.split('issue_stalled_')[1].replace('_per_issue_active.ratio', ''))
                 for i, h in enumerate(hdr) if 'issue_stalled' in h and h.endswith('per_issue_active.ratio')], reverse=True)[:4]
    rd = float(g(r, 'dram__bytes_read.sum') or 0); wr = float(g(r, 'dram__bytes_write.sum') or 0)
    ru = rows[1][hdr.index('dram__bytes_read.sum')]; wu = rows[1][hdr.index('dram__bytes_write.sum')]
    print(f"{g(r,'Kernel Name')[:48]:48s} grid={g(r,'Grid Size'):>16s} t={float(g(r,'gpu__time_duration.sum')):8.1f}us "
          f"rd={rd:8.1f}{ru} wr={wr:8.1f}{wu} dram%={float(g(r,'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):5.1f} "
          f"regs={g(r,'launch__registers_per_thread')} warps%={float(g(r,'sm__warps_active.avg.pct_of_peak_sustained_active')):5.1f} "
          f"issue%={float(g(r,'smsp__issue_active.avg.pct_of_peak_sustained_active')):5.1f} "
          f"L1hit={float(g(r,'l1tex__t_sector_hit_rate.pct') or 0):5.1f} L2hit={float(g(r,'lts__t_sector_hit_rate.pct') or 0):5.1f} "
          + ' '.join(f"{n}={v:.2f}" for v, n in st))
