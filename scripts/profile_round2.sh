#!/bin/bash
# Round-2 raw material for profiles/ (run on a B200 through gpurun; summaries are made on the CPU side with
# profiles/make_traffic.py, launch_summary.py, ncu_brief.py, ncu_summ.py, ncu_segments.py):
#   1. ncu launch list of the bench command (gpu time + DRAM bytes per launch)
#   2. ncu --set full of the level-0 block-solve kernel (K2W) with source / SASS sampling
#   3. ncu sections of every streaming kernel of one solve
#   4. the bench line itself and the reference arm (NOT under a profiler)
set -x
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_arm_r2.json 2>> gpurun_out/bench_r2.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1400 --csv \
    --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity --no-traffic \
    > gpurun_out/launches_r2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oras_sweep_warp --launch-skip 6 --launch-count 1 \
    -f -o gpurun_out/k2w_r2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity --no-traffic > gpurun_out/k2w_r2.log 2>&1
ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section LaunchStats --section SchedulerStats \
    --clock-control none -k regex:'residual_|oras_combine|prolongate|downsample_|pack_block' --launch-skip 0 --launch-count 140 \
    -f -o gpurun_out/stream_r2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity --no-traffic > gpurun_out/stream_r2.log 2>&1
ls -la gpurun_out/
