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
    the geometry.  ``gather`` / ``solve_blocks`` / ``scatter_weighted`` are the
    reference's stage calls for A/B tests: the block solve runs the generic
    shared-memory kernel on its own, the scatter runs the sweeps' combine
    kernel (K2b) on its own.
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

    def gather(self, r) -> np.ndarray:
        """R_i r for every block: (h, w) -> (nblocks, bh, bw) (solvers.py:303-305).  Host-side indexing with
        the library's block starts; inside the sweeps the gather is fused into the block-solve kernel."""
        r = np.asarray(r, dtype=np.float64)
        if r.shape != self.shape:
            raise ValueError(f"field shape {r.shape} does not match the mask {self.shape}")
        p = self.part
        return np.stack([r[y:y + p.block_h, x:x + p.block_w] for y in p.ys for x in p.xs])

    def _field_of(self, tiles) -> np.ndarray:
        """The field whose gather is `tiles` (the device entry point takes a field)."""
        p = self.part
        if tiles.shape != (p.nblocks, p.block_h, p.block_w):
            raise ValueError(f"expected gathered blocks {(p.nblocks, p.block_h, p.block_w)}, got {tiles.shape}")
        f = np.zeros(self.shape)
        for t, (y, x) in zip(tiles, ((y, x) for y in p.ys for x in p.xs)):
            f[y:y + p.block_h, x:x + p.block_w] = t
        if not np.array_equal(self.gather(f), tiles):
            raise ValueError("blocks disagree on their overlaps: not the gather of a field")
        return f

    def scatter_weighted(self, v) -> np.ndarray:
        """sum_i R_i^T (wy_i (x) wx_i * v_i) in block order (solvers.py:307-314): the combine kernel alone."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        p = self.part
        if v.shape != (p.nblocks, p.block_h, p.block_w):
            raise ValueError(f"expected local corrections {(p.nblocks, p.block_h, p.block_w)}, got {v.shape}")
        plan = self._plan()
        d_v = _dev.to_device_f64(v)
        d_f = _dev.empty_f64(self.shape)
        _dev.call("b200p_plan_scatter_weighted", plan.handle, 0, _dev.ptr(d_v), _dev.ptr(d_f), _dev.stream())
        return _dev.to_host(d_f)

    def solve_blocks(self, rhs, target_sq: float, max_iters: int, workers: int = 1) -> np.ndarray:
        """Local Robin solves of all blocks (solvers.py:372-390) to `target_sq`.  `rhs` is the reference's
        gathered residual (nblocks, bh, bw) -- `bs.solve_blocks(bs.gather(r), ...)` -- or the global residual
        field itself (gather fused, as in the sweeps)."""
        rhs_field = np.asarray(rhs, dtype=np.float64)
        if rhs_field.ndim == 3:
            rhs_field = self._field_of(rhs_field)
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
