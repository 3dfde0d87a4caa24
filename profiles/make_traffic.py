#!/usr/bin/env python
"""Reads an ncu launch list (gpu__time_duration, dram bytes per launch; CSV written by
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`) and writes
(1) a per-kernel summary (launches, time share, DRAM bytes per launch) and (2) traffic.json with the
measured DRAM bytes per launch of the ORAS sweep (K2 + K2b), which bench.py reports as roofline.traffic."""
import collections, csv, json, sys
src, out_txt, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [l for l in open(src) if not l.startswith('==')]
rows = list(csv.DictReader(lines))
launch = collections.OrderedDict()
for r in rows:
    d = launch.setdefault(r['ID'], {'name': r['Kernel Name'].split('(')[0].replace('b200p::', '').replace('void ', ''),
                                    'grid': r['Grid Size']})
    v = float(r['Metric Value'].replace(',', ''))
    unit = r['Metric Unit']
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1, 'us': 1e3, 'ms': 1e6}.get(unit, 1)
    d[r['Metric Name']] = v * scale
agg = collections.OrderedDict()
for d in launch.values():
    a = agg.setdefault(d['name'], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get('gpu__time_duration.sum', 0.0)
    a[2] += d.get('dram__bytes_read.sum', 0.0)
    a[3] += d.get('dram__bytes_write.sum', 0.0)
tot = sum(a[1] for a in agg.values())
with open(out_txt, 'w') as f:
    f.write(f"# {len(launch)} launches, {tot/1e6:.3f} ms total (ncu: serialised, cold cache -- compare shares)\n")
    f.write(f"{'kernel':58s} {'n':>4s} {'ms':>9s} {'share':>6s} {'rd MB/launch':>13s} {'wr MB/launch':>13s}\n")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{k[:58]:58s} {a[0]:4d} {a[1]/1e6:9.3f} {a[1]/tot:6.3f} {a[2]/a[0]/1e6:13.2f} {a[3]/a[0]/1e6:13.2f}\n")
sweep = [a for k, a in agg.items() if 'oras_sweep' in k or 'oras_combine' in k]
n_sweeps = sum(a[0] for k, a in agg.items() if 'oras_sweep' in k)
traffic = {'oras_sweep': {'dram_bytes_per_launch': sum(a[2] + a[3] for a in sweep) / max(n_sweeps, 1),
                          'sweeps': n_sweeps, 'source': src.split('/')[-1],
                          'note': 'dram__bytes_read.sum + dram__bytes_write.sum of K2 + K2b, averaged over the '
                                  'sweeps of one step (all levels), like roofline.alg_bytes_per_launch',
                          # frames per step of the profiled command (scripts/profile_round.sh: --frames 4)
                          'frames': int(sys.argv[4]) if len(sys.argv) > 4 else 4}}
json.dump(traffic, open(out_json, 'w'), indent=1)
print(open(out_txt).read())
print(traffic)
