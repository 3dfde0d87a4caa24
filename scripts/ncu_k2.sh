#!/bin/bash
# usage: scripts/ncu_k2.sh NAME "ENV=.." -> gpurun_out/NAME.ncu-rep : ncu --set full of the first level-0 K2 launch
name=$1; shift
env "$@" ncu --set full --clock-control none --import-source on -k regex:oras_sweep_ --launch-skip 6 --launch-count 1 \
  -f -o gpurun_out/$name python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log | cut -c1-300
