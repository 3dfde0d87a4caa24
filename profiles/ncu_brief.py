#!/usr/bin/env python
"""One line per captured launch from an .ncu-rep: duration, DRAM GB/s (and bytes when the capture has them),
DRAM %, registers, occupancy, issue %, cache hit rates, top stalls.  Optional argv[2]: minimum grid.y to list."""
import csv, subprocess, sys, io, re
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
min_gy = int(sys.argv[2]) if len(sys.argv) > 2 else 0
def g(r, k):
    return r[hdr.index(k)] if k in hdr else ''
def f(r, k):
    try:
        return float(g(r, k).replace(',', '') or 0)
    except ValueError:
        return 0.0
def scaled(r, k, table):
    return f(r, k) * table.get(units[hdr.index(k)], 1.0) if k in hdr else None
BY = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12}
BPS = {'byte/s': 1, 'Kbyte/s': 1e3, 'Mbyte/s': 1e6, 'Gbyte/s': 1e9, 'Tbyte/s': 1e12}
T = {'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 's': 1e6}
for r in rows[2:]:
    m = re.search(r'\((\d+), (\d+), (\d+)\)', g(r, 'Grid Size'))
    if m and int(m.group(2)) < min_gy:
        continue
    st = sorted([(float(r[i] or 0), h.split('issue_stalled_')[1].replace('_per_issue_active.ratio', ''))
                 for i, h in enumerate(hdr) if 'issue_stalled' in h and h.endswith('per_issue_active.ratio')], reverse=True)[:4]
    t_us = f(r, 'gpu__time_duration.sum') * T.get(units[hdr.index('gpu__time_duration.sum')], 1.0)
    rd, wr = scaled(r, 'dram__bytes_read.sum', BY), scaled(r, 'dram__bytes_write.sum', BY)
    bps = scaled(r, 'dram__bytes.sum.per_second', BPS)
    if rd is not None:
        mem = f"rd={rd / 1e6:8.1f}MB wr={wr / 1e6:8.1f}MB dram={((rd + wr) / 1e9) / (t_us * 1e-6) if t_us else 0:6.0f}GB/s"
    else:
        mem = f"dram={bps / 1e9 if bps else 0:6.0f}GB/s"
    print(f"{g(r, 'Kernel Name').replace('void ', '')[:44]:44s} grid={g(r, 'Grid Size'):>15s} t={t_us:8.1f}us {mem} "
          f"dram%={f(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
          f"regs={g(r, 'launch__registers_per_thread')} warps%={f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} "
          f"issue%={f(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f} "
          f"L1hit={f(r, 'l1tex__t_sector_hit_rate.pct'):5.1f} L2hit={f(r, 'lts__t_sector_hit_rate.pct'):5.1f} "
          + ' '.join(f"{n}={v:.2f}" for v, n in st))
