#!/bin/bash
# compute-sanitizer passes over the small GPU tests (run through gpurun):
#   memcheck + initcheck on the stage tests, the known-answer tests, the 8-bit image path and the small solves;
#   racecheck on the block-solve kernels (K2W keeps its tables / weight rows in shared memory) and the coarse kernel.
# racecheck runs with the TMA tile pipelines switched off (B200P_ROWS_TMA=0 B200P_PROLONG_TMA=0): compute-sanitizer 12.9's
# racecheck segfaults on the host as soon as a kernel with a CUtensorMap parameter is launched (reproduced on the
# smallest solve; memcheck and initcheck run those kernels fine).  Their shared-memory protocol is one mbarrier
# phase per stage fill and one __syncthreads per tile before the refill.
# Output: gpurun_out/sanitize.log (one summary line per pass).
S="compute-sanitizer --error-exitcode 9"
run() {   # name, tool, pytest args...
  name=$1; tool=$2; shift 2
  timeout 1500 $S --tool $tool python -m pytest "$@" -m gpu -q -x > gpurun_out/sanitize_$name.log 2>&1
  echo "$name ($tool): rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$name.log | tail -1) | $(tail -1 gpurun_out/sanitize_$name.log)" | tee -a gpurun_out/sanitize.log
}
mkdir -p gpurun_out; : > gpurun_out/sanitize.log
run stages_mem memcheck tests/test_gpu_stages.py tests/test_gpu_kats.py tests/test_gpu_images.py   # incl. the tile pipelines on ragged levels
run solve_mem memcheck tests/test_gpu_solve.py tests/test_gpu_regressions.py -k "small_cases or cg_pipelines or ml_oras or single_level or frame_pipeline or graph_and_eager or u8 or sparse_ingest or mask_residual or callback or pinned or element_counts or cache_eviction or host_gather"
run strip_mem memcheck tests/test_gpu_strip.py -k "native or matches_single_plan"
export B200P_ROWS_TMA=0 B200P_PROLONG_TMA=0
run sweeps_race racecheck tests/test_gpu_stages.py tests/test_gpu_kats.py -k "tile32 or sweeps_match or general_start or identity or single_level_v"
run solve_race racecheck tests/test_gpu_solve.py -k "config1 or cg_pipelines"
unset B200P_ROWS_TMA B200P_PROLONG_TMA
run init initcheck tests/test_gpu_solve.py tests/test_gpu_stages.py tests/test_gpu_images.py -k "config1 or ml_oras or cg_pipelines or single_level or tile32 or build_hierarchy or small_cases or decode_matches"
cat gpurun_out/sanitize.log
