"""Solver configuration, report record and the ORAS smoother entry points.

Interface of the reference's ``diffpaint.solvers`` for the ORAS half
(solvers.py:43-94, :255-424); the sweeps run in libb200paint's K1/K2/K2b
kernels through ``b200p_plan_oras_sweeps``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _dev
from .partition import BlockPartition, BlockWeights, build_partition, build_weights


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:43-69 (same fields, defaults and validation)."""

    tol_rel: float = 1e-3
    max_outer_iters: int = 10_000
    alpha: float = 0.5
    local_tol_fraction: float = 1e-5
    local_max_iters: int | None = None
    smoother_cg_iters: int = 10

    def __post_init__(self):
        if not 0.0 < self.tol_rel < 1.0:
            raise ValueError(f"tol_rel must be in (0, 1), got {self.tol_rel}")
        if self.alpha <= 0.0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")
        if self.local_tol_fraction <= 0.0:
            raise ValueError(f"local_tol_fraction must be positive, got {self.local_tol_fraction}")


@dataclass
class SolveReport:
    """solvers.py:72-94."""

    solver: str
    iterations: int
    final_rel_residual: float
    wall_time: float
    history: list = field(default_factory=list)
    converged: bool = True
    baseline_residual: float = 0.0
    init_residual: float = 0.0
    fine_smoother_iterations: int = 0


class BlockSolver:
    """Descriptor of the batched Robin block solves (solvers.py:255-301).

    The reference precomputes gather indices and per-block diagonals; the GPU
    kernels derive both analytically, so this object only validates and carries
    the geometry.  ``solve_blocks`` / ``gather`` / ``scatter_weighted`` are
    provided for A/B tests.
    """

    def __init__(self, mask, spacing: float, part: BlockPartition, weights: BlockWeights, alpha: float):
        if alpha <= 0.0:
            raise ValueError(f"alpha must be positive, got {alpha}")
        mask = np.asarray(mask).astype(bool)
        h, w = mask.shape
        if (w, h) != (part.width, part.height):
            raise ValueError("partition does not match the mask dimensions")
        self.mask, self.spacing, self.part, self.weights, self.alpha = mask, float(spacing), part, weights, float(alpha)
        self.shape = (h, w)

    def _plan(self, eta=1e-5, local_max_iters=None):
        from .multigrid import _stage_plan
        return _stage_plan(self.mask, self.spacing, self.part.block_size, self.part.overlap,
                           self.alpha, eta, local_max_iters)

    def solve_blocks(self, rhs_field, target_sq: float, max_iters: int, workers: int = 1) -> np.ndarray:
        """gather + solve_blocks on a global residual FIELD (solvers.py:303-305, :372-390)."""
        plan = self._plan(local_max_iters=max_iters)
        r = _dev.to_device_f64(rhs_field)
        p = self.part
        v = _dev.empty_f64((p.nblocks, p.block_h, p.block_w))
        _dev.call("b200p_plan_solve_blocks", plan.handle, 0, _dev.ptr(r), float(target_sq),
                  _dev.ptr(v), _dev.stream())
        return _dev.to_host(v)


def oras_sweeps(op, blocks: BlockSolver, b, u, *, max_sweeps: int, stop_norm: float, eta: float,
                local_max_iters: int, workers: int = 1, on_state=None, path: int = 0):
    """Schwarz sweeps on u in place until ||b - A u|| <= stop_norm (solvers.py:393-424).

    ``workers`` is accepted for signature compatibility (block parallelism is
    the CUDA grid).  ``on_state(u, rn, sweeps)`` is called at every residual
    evaluation like the reference's (solvers.py:418-419); with a hook the sweeps
    are enqueued one at a time so that the iterate can be handed out in between.
    Returns (sweeps, final residual norm).
    """
    u_arr = np.asarray(u)
    if u_arr.dtype != np.float64 or u_arr.shape != blocks.shape:
        raise ValueError("u must be a float64 field of the mask's shape")
    plan = blocks._plan(eta, local_max_iters)
    du, db = _dev.to_device_f64(u_arr), _dev.to_device_f64(b)
    sweeps = np.zeros(1, dtype=np.int32)
    rn = np.zeros(1)

    def run(k):
        _dev.call("b200p_plan_oras_sweeps", plan.handle, 0, _dev.ptr(db), _dev.ptr(du), int(k),
                  float(stop_norm), int(path), sweeps.ctypes.data, rn.ctypes.data, _dev.stream())
        return int(sweeps[0]), float(rn[0])

    if on_state is None:
        done, norm = run(max_sweeps)
    else:
        done, (_, norm) = 0, run(0)                      # the residual of the start iterate
        while True:
            u_arr[...] = _dev.to_host(du)
            on_state(u_arr, norm, done)
            if norm == 0.0 or norm <= stop_norm or done >= max_sweeps:   # solvers.py:420-421
                break
            step, norm = run(1)
            if step == 0:
                break
            done += step
    u_arr[...] = _dev.to_host(du)
    return done, norm


__all__ = ["SolverConfig", "SolveReport", "BlockSolver", "oras_sweeps",
           "BlockPartition", "BlockWeights", "build_partition", "build_weights"]
