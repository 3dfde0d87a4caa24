#!/bin/bash
# device-resident frames/s against frames per step (plan batch size)
for f in "$@"; do
  python bench.py --steps 6 --warmup 3 --frames $f --no-e2e --no-cpu-baseline --no-parity --no-traffic > gpurun_out/abf.json 2>gpurun_out/abf.err
  python - $f <<'PY'
import json,sys
try:
    d=json.load(open("gpurun_out/abf.json")); print("frames", sys.argv[1], "fps=%.1f"%d["value"], "plan GB=%.1f"%(d["plan_device_bytes"]/1e9))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/abf.err").read()[-300:])
PY
done
