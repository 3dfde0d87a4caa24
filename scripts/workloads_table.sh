#!/bin/bash
# Regenerates profiles/workloads_r1.txt's rows on a B200: every BASELINE workload through bench.py.
run() { python bench.py --workload $1 --frames $2 --steps 6 --lanes 4 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); e=d['e2e']
print('%-28s %3d %14.1f %9.3f    %-10s %8.1f %8.1f   %.3f' % (d['config']['workload'], d['config']['frames_per_step_per_gpu'], d['value'], d['ms_per_frame'], str(d['config']['v_cycles']).replace(' ',''), e['value'], e['u8_value'], d['frame_roofline']['frac']))"; }
echo "# bench.py --workload W --frames F --steps 6 --lanes 4 on one B200 (round 1), frames/s"
echo "# workload              frames/step  device-resident  ms/frame  V-cycles   e2e fp64  e2e u8   frame alg. bytes / HBM peak"
run 256_gray_5pct_b16o2 64
run 1080p_rgb_4pct_b16o2 8
run 4k_rgb_2pct_b32o6 8
run 4k_rgb_0.5pct_b32o6 8
run 8k_rgb_2pct_b32o6 2
