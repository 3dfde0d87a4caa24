#!/usr/bin/env python
"""Per-kernel / per-grid summary of one solve from an ncu launch list
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X)."""
import csv, collections, re, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
iK, iG, iM, iV, iID = (hdr.index(n) for n in ('Kernel Name', 'Grid Size', 'Metric Name', 'Metric Value', 'ID'))
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[iID], {'k': r[iK].replace('b200p::', '').replace('void ', ''), 'g': r[iG]})
    d[r[iM]] = float(r[iV].replace(',', ''))
ids = list(L)
starts = [i for i, k in enumerate(ids) if L[k]['k'].startswith('pack_block_masks') and i + 1 < len(ids)
          and L[ids[i + 1]]['k'].startswith('downsample_mask') and (i == 0 or L[ids[i - 1]]['k'].startswith('pack_reports'))]
a = starts[-1]
b = len(ids)
agg = collections.OrderedDict()
tot = 0.0
for k in ids[a:b]:
    d = L[k]
    name = re.sub(r'\(.*', '', d['k'])[:46]
    e = agg.setdefault((name, d['g']), [0, 0.0, 0.0, 0.0])
    t = d['gpu__time_duration.sum']
    e[0] += 1; e[1] += t; e[2] += d.get('dram__bytes_read.sum', 0); e[3] += d.get('dram__bytes_write.sum', 0); tot += t
print(f'# one solve: {b - a} launches, {tot / 1e6:.3f} ms in kernels (ncu: serialised, cold cache -- compare shares)')
byname = collections.Counter()
for (n, g), e in agg.items():
    byname[n] += e[1]
print('# by kernel')
for n, t in byname.most_common():
    print(f'{n:48s} {t / 1e3:9.1f} us {100 * t / tot:5.1f}%')
print('# by kernel and grid')
for (n, g), e in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 45]:
    print(f'{n:48s} {g:18s} n={e[0]:3d} t={e[1] / 1e3:9.1f}us {100 * e[1] / tot:5.1f}%  rd={e[2] / e[0] / 1e6:8.1f}MB wr={e[3] / e[0] / 1e6:8.1f}MB per launch')
