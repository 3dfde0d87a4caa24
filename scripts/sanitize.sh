#!/bin/bash
# compute-sanitizer passes over the small GPU tests (run through gpurun); all three were clean in round 1:
#   memcheck + initcheck on the stage tests and the small solves, racecheck on the K2 variants.
set -e
S="compute-sanitizer --error-exitcode 9"
$S --tool memcheck  python -m pytest tests/test_gpu_stages.py -m gpu -q -x
$S --tool memcheck  python -m pytest tests/test_gpu_solve.py -m gpu -q -x -k "small_cases or cg_pipelines or ml_oras or single_level or frame_pipeline or graph_and_eager or u8 or fused_and or sparse_ingest or mask_residual or callback"
$S --tool racecheck python -m pytest tests/test_gpu_stages.py -m gpu -q -x -k "tile32 or sweeps_match or general_start"
$S --tool racecheck python -m pytest tests/test_gpu_solve.py -m gpu -q -x -k "config1 or cg_pipelines"
$S --tool initcheck python -m pytest tests/test_gpu_solve.py tests/test_gpu_stages.py -m gpu -q -x -k "config1 or ml_oras or cg_pipelines or single_level or tile32 or build_hierarchy or small_cases"
