#!/bin/bash
# ncu sections of every streaming kernel of one solve (4 frames of 4K RGB) -> gpurun_out/stream.ncu-rep
ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section LaunchStats --section SchedulerStats \
    --clock-control none -k regex:'residual_|oras_combine|prolongate|downsample_values' --launch-skip 0 --launch-count 120 \
    -f -o gpurun_out/stream python bench.py --steps 1 --warmup 0 --frames 4 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/stream.log 2>&1
ls -la gpurun_out/
