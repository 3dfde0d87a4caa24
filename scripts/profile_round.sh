#!/bin/bash
# Regenerates the raw material of profiles/ on a B200 (run through gpurun):
#   launch list of one bench step (gpu time + DRAM bytes per launch), ncu --set full of the
#   level-0 block-solve kernel and of the streaming kernels.  Summaries are made on the CPU side
#   (profiles/make_traffic.py, launch_summary.py, ncu_summ.py, ncu_brief.py).
set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --frames 4 --no-e2e --no-cpu-baseline --no-parity \
    > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oras_sweep_lean --launch-skip 6 --launch-count 1 \
    -f -o gpurun_out/k2_lean python bench.py --steps 1 --warmup 0 --frames 4 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/k2_lean.log 2>&1
ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section LaunchStats --section SchedulerStats \
    --clock-control none -k regex:'residual_|oras_combine|prolongate|downsample_values' --launch-skip 0 --launch-count 120 \
    -f -o gpurun_out/stream python bench.py --steps 1 --warmup 0 --frames 4 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/stream.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
