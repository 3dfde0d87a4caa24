#!/bin/bash
# usage: scripts/ab.sh "ENV=.. ENV=.." ... -> one line per variant (8 frames of 4K RGB per step, device-resident)
for v in "$@"; do
  env $v python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$v" <<'PY'
import json,sys
try:
    d=json.load(open("gpurun_out/ab.json"))
    k=d["kernels"]
    print(sys.argv[1], "fps=%.1f"%d["value"], " ".join("%s=%.2f"%(n[:14],x["ms_per_step"]) for n,x in k.items() if x["ms_per_step"]>0.3))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/ab.err").read()[-300:])
PY
done
