"""paper_2401_06744_b200 -- B200-native (sm_100a) drop-in for the reference's
``mg-oras`` path: full-multigrid homogeneous-diffusion inpainting with the
Robin-optimised restricted-additive-Schwarz block smoother (arXiv 2401.06744).

Same Python vocabulary as the reference package ``diffpaint`` for this path;
the arithmetic runs in ``libb200paint.so`` (hand-written CUDA, C-ABI in
``include/b200paint.h``).  No CPU fallback.
"""

from . import _lib, fileio, strip, suites
from .core import (EmptyMaskError, InpaintingProblem, Metrics, StencilOperator, apply_operator,
                   as_field, as_mask, compute_metrics, mask_density, residual)
from .multigrid import (Level, LevelHierarchy, MultigridConfig, Plan, build_hierarchy, cached_plan,
                        cascadic_init, clear_plan_cache, downsample_mask, downsample_values_modified,
                        downsample_values_naive, fmg_solve, prolongate_correction,
                        prolongate_solution, restrict_residual, v_cycle)
from .partition import (BlockPartition, BlockRect, BlockWeights, build_partition, build_weights,
                        extend_add_weighted, restrict_to_block)
from .pipeline import FramePipeline
from .fileio import ImageFile, image_from_fields, pack_mask_raster, unpack_mask_raster
from .pipelines import (SOLVER_NAMES, SolveResult, inpaint_image_u8, join_solver_name, solve_channel,
                        solve_frames, solve_image, split_solver_name)
from .solvers import BlockSolver, SolveReport, SolverConfig, oras_sweeps

__version__ = "0.1.0"

build = _lib.build

__all__ = [
    "EmptyMaskError", "InpaintingProblem", "Metrics", "StencilOperator", "apply_operator", "as_field",
    "as_mask", "compute_metrics", "mask_density", "residual",
    "Level", "LevelHierarchy", "MultigridConfig", "Plan", "build_hierarchy", "cached_plan",
    "cascadic_init", "clear_plan_cache", "downsample_mask", "downsample_values_modified",
    "downsample_values_naive", "fmg_solve", "prolongate_correction", "prolongate_solution",
    "restrict_residual", "v_cycle",
    "BlockPartition", "BlockRect", "BlockWeights", "build_partition", "build_weights",
    "extend_add_weighted", "restrict_to_block",
    "SOLVER_NAMES", "SolveResult", "join_solver_name", "solve_channel", "solve_frames", "solve_image",
    "split_solver_name", "inpaint_image_u8", "ImageFile", "image_from_fields", "pack_mask_raster",
    "unpack_mask_raster", "fileio",
    "BlockSolver", "SolveReport", "SolverConfig", "oras_sweeps", "FramePipeline", "suites", "strip",
]
