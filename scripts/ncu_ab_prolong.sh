#!/bin/bash
# ncu --set full of the prolongation kernels of one step for two builds (A/B of load orderings)
for tag in orig mb6; do
  B200P_LIB=/root/repo/ab_lib_$tag.so ncu --set full --clock-control none -k regex:'prolongate_kernel' --launch-skip 0 --launch-count 21 \
    -f -o gpurun_out/prolong_$tag python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity --no-traffic > gpurun_out/prolong_$tag.log 2>&1
done
