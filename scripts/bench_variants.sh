#!/bin/bash
# usage: scripts/bench_variants.sh "ENV1=.. ENV2=.." ...   -> one summary line per variant
for v in "$@"; do
  env $v python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/variant.err | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernels']
print('$v', 'fps=%.1f'%d['value'], 'ms/frame=%.2f'%d['ms_per_frame'], ' '.join('%s=%.2f'%(n[:14],v['ms_per_step']) for n,v in k.items() if v['ms_per_step']>0.3))
"
  grep stats gpurun_out/variant.err
done
