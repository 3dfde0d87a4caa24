#!/bin/bash
# Every BASELINE configuration through bench.py on one B200 -> gpurun_out/workloads_r2.txt (summarised into profiles/)
out=gpurun_out/workloads_r2.txt
echo "# bench.py --workload W --frames F --steps 6 on one B200 (round 2, final build), frames/s" > $out
echo "# workload              frames/step  device-resident  ms/frame  V-cycles   e2e fp64  e2e image-u8   frame alg. bytes / HBM peak" >> $out
run() {  # workload frames
  python bench.py --workload $1 --frames $2 --steps 6 --warmup 3 --no-cpu-baseline --no-parity --no-traffic > gpurun_out/wl.json 2> gpurun_out/wl.err
  python - $1 $2 >> $out <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/wl.json").read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"{sys.argv[1]:28s} {int(sys.argv[2]):4d} {d['value']:14.1f} {d['ms_per_frame']:9.3f}    {str(d['config']['v_cycles']).replace(' ', ''):10s} "
          f"{e.get('value', float('nan')):9.1f} {e.get('image_u8_value', float('nan')):9.1f}   {d['frame_roofline']['frac']:.3f}")
except Exception as ex:
    print(sys.argv[1], "FAILED", ex, open("gpurun_out/wl.err").read()[-300:].replace("\n", " | "))
PY
}
run 256_gray_5pct_b16o2 64
run 1080p_rgb_4pct_b16o2 8
run 4k_rgb_2pct_b32o6 8
run 4k_rgb_0.5pct_b32o6 8
run 8k_rgb_2pct_b32o6 2
cat $out
