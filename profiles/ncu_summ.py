#!/usr/bin/env python
"""Summarise an `ncu --page raw --csv` dump: key metrics, top stall reasons, pipe mix."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
want = ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'smsp__inst_executed.sum',
        'lts__t_bytes.sum', 'l1tex__t_bytes.sum', 'smsp__cycles_active.avg', 'sm__cycles_elapsed.max']
for r in rows[2:]:
    print('=' * 60)
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:75s} {r[i]:>20s} {units[i]}")
    names = [h for h in hdr if 'warp_issue_stalled' in h and h.endswith('_per_warp_active.pct')]
    vals = sorted([(float(r[hdr.index(n)] or 0), n) for n in names], reverse=True)[:8]
    print('-- top stall reasons (% of warp-active cycles)')
    for v, n in vals:
        print(f"   {v:8.2f}  {n.replace('smsp__average_warp_latency_issue_stalled_', '').replace('smsp__average_warps_issue_stalled_', '')}")
    print('-- pipe instruction mix')
    for n in [h for h in hdr if h.startswith('sm__inst_executed_pipe_') and h.endswith('.sum')]:
        v = r[hdr.index(n)]
        if v not in ('0', '', 'n/a'):
            print(f"   {n:55s} {v}")
