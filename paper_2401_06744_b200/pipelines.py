"""Named-pipeline front end: the drop-in boundary of the path.

``solve_image(problem, "mg-oras", cfg)`` has the reference's signature, result
type and error behaviour (pipelines.py:20-114).  All six names run on the CUDA
path: "mg-oras" (the hot path), "ml-oras" (cascadic multilevel) and "oras"
(single-level Schwarz iteration) on the same kernels, and the CG-smoothed
comparison set "mg-cg", "ml-cg", "cg" on flat global-CG kernels.
``solve_frames`` is the batched entry (frames x channels in one plan).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from .core import EmptyMaskError, InpaintingProblem
from .multigrid import LevelHierarchy, MultigridConfig, build_hierarchy, cached_plan, fmg_solve
from .solvers import SolveReport

SOLVER_NAMES = ("cg", "oras", "ml-cg", "ml-oras", "mg-cg", "mg-oras")
BUILT = SOLVER_NAMES  # all six pipelines of the reference run on the CUDA path


def split_solver_name(name: str):
    """pipelines.py:23-31: name -> (smoother, mode)."""
    if name not in SOLVER_NAMES:
        raise ValueError(f"unknown solver {name!r}, expected one of {SOLVER_NAMES}")
    head, sep, tail = name.partition("-")
    if not sep:
        return name, "single"
    return tail, {"ml": "multilevel", "mg": "full_multigrid"}[head]


def join_solver_name(base: str, mode: str) -> str:
    name = {"single": "", "multilevel": "ml-", "full_multigrid": "mg-"}[mode] + base
    if name not in SOLVER_NAMES:
        raise ValueError(f"no solver for base {base!r} in mode {mode!r}")
    return name


def _require_built(name: str):
    split_solver_name(name)
    if name not in BUILT:
        raise NotImplementedError(
            f"pipeline {name!r} is outside the B200 hot path; only {BUILT} are built")


HBM_PEAK_GBS = 6546.0   # measured copy bandwidth of the B200s this was built on (MEASURED_PEAKS.json)


def algorithmic_bytes(width: int, height: int, channels: int, v_cycles: int) -> float:
    """Compulsory HBM traffic of one mg-oras solve: every array of a fused stage touched once,
    B = (6.67 + 15.33 V) C s N0 + (4.67 + 9.33 V) m N0 with s = 8 (fp64), m = 1 (mask byte), V = V-cycles."""
    n0 = float(width) * float(height)
    return (6.67 + 15.33 * v_cycles) * channels * 8.0 * n0 + (4.67 + 9.33 * v_cycles) * n0


@dataclass
class SolveResult:
    """pipelines.py:75-93, plus the throughput view of the call: frames/s, algorithmic HBM GB/s and
    its fraction of the measured HBM peak -- of the whole host-to-host call, copies included."""

    fields: np.ndarray
    reports: list
    elapsed: float

    @property
    def frames_per_s(self) -> float:
        return 1.0 / self.elapsed if self.elapsed > 0 else float("inf")

    @property
    def hbm_gbs(self) -> float:
        c, h, w = self.fields.shape
        return algorithmic_bytes(w, h, c, self.iterations) / 1e9 / self.elapsed if self.elapsed > 0 else float("inf")

    @property
    def roofline_fraction(self) -> float:
        return self.hbm_gbs / HBM_PEAK_GBS

    @property
    def converged(self) -> bool:
        return all(r.converged for r in self.reports)

    @property
    def iterations(self) -> int:
        return max(r.iterations for r in self.reports)

    @property
    def final_rel_residual(self) -> float:
        return max(r.final_rel_residual for r in self.reports)


def solve_channel(problem: InpaintingProblem, name: str, cfg: MultigridConfig | None = None,
                  channel: int = 0, hierarchy: LevelHierarchy | None = None, callback=None):
    """pipelines.py:42-72 for "mg-oras"."""
    _require_built(name)
    base, mode = split_solver_name(name)
    if mode == "single":
        if callback is not None:
            if base != "oras":
                from .multigrid import _cg_solve_with_step_hook
                if not problem.mask.any():
                    raise EmptyMaskError("cannot solve without known pixels")
                return _cg_solve_with_step_hook(problem, replace(cfg or MultigridConfig(), smoother=base), channel,
                                                callback, single_level=True)
            return _oras_solve_stepwise(problem, (cfg or MultigridConfig()), channel, callback)
        sub = InpaintingProblem(problem.mask, problem.known[channel], problem.spacing)
        res = solve_image(sub, name, cfg)
        return res.fields[0], res.reports[0]
    cfg = replace(cfg or MultigridConfig(), smoother=base, mode=mode)
    if hierarchy is None:
        hierarchy = build_hierarchy(problem, cfg)
    return fmg_solve(hierarchy, cfg, channel, callback=callback)


def _oras_solve_stepwise(problem: InpaintingProblem, cfg: MultigridConfig, channel: int, callback):
    """oras_solve with `callback(u)` after every sweep (solvers.py:427-485): the reference's own structure -- the
    sweeps are driven one at a time through `oras_sweeps(..., on_state=)` (same kernels as the one-call solve), the
    history is the relative residual at every residual evaluation."""
    from .partition import build_partition, build_weights
    from .solvers import BlockSolver, oras_sweeps
    t0 = time.perf_counter()
    s = cfg.solver
    h, w = problem.shape
    part = build_partition(w, h, cfg.block_size, cfg.overlap)
    op = problem.operator()
    blocks = BlockSolver(problem.mask, problem.spacing, part, build_weights(part), s.alpha)
    b = problem.rhs(channel)
    u = problem.flat_init(channel)
    r0 = float(np.linalg.norm(op.residual(b, u)))
    if r0 == 0.0:
        return u, SolveReport(solver="oras", iterations=0, final_rel_residual=0.0, wall_time=time.perf_counter() - t0,
                              history=[0.0], converged=True, baseline_residual=r0, init_residual=r0,
                              fine_smoother_iterations=0)
    history = []

    def on_state(uu, rn_now, sweeps_done):
        history.append(rn_now / r0)
        if sweeps_done > 0:
            callback(uu)

    sweeps, rn = oras_sweeps(op, blocks, b, u, max_sweeps=s.max_outer_iters, stop_norm=s.tol_rel * r0,
                             eta=s.local_tol_fraction, local_max_iters=s.local_max_iters or 4 * part.block_h * part.block_w,
                             on_state=on_state)
    rel = rn / r0
    return u, SolveReport(solver="oras", iterations=sweeps, final_rel_residual=rel, wall_time=time.perf_counter() - t0,
                          history=history, converged=rel <= s.tol_rel, baseline_residual=r0, init_residual=r0,
                          fine_smoother_iterations=sweeps)


def solve_image(problem: InpaintingProblem, name: str = "mg-oras",
                cfg: MultigridConfig | None = None) -> SolveResult:
    """All channels of one frame, batched in one plan (pipelines.py:96-114).

    Host arrays in, host arrays out; ``elapsed`` covers H2D, hierarchy build,
    the solve and D2H.
    """
    _require_built(name)
    base, mode = split_solver_name(name)
    single = mode == "single"  # "oras": oras_solve on the finest level (solvers.py:427-485)
    cfg = cfg or MultigridConfig()
    cfg = replace(cfg, smoother=base) if single else replace(cfg, smoother=base, mode=mode)
    if not problem.mask.any():
        raise EmptyMaskError("cannot solve without known pixels")
    t0 = time.perf_counter()
    h, w = problem.shape
    plan = cached_plan(w, h, problem.channels, 1, cfg, problem.spacing, single_level=single)
    out, reports = plan.solve_host(problem.mask.view(np.uint8)[None], problem.known[None])
    elapsed = time.perf_counter() - t0
    for r in reports:
        r.wall_time = elapsed
    return SolveResult(fields=out[0], reports=reports, elapsed=elapsed)


def inpaint_image_u8(pixels, mask, name: str = "mg-oras", cfg: MultigridConfig | None = None,
                     spacing: float = 1.0, packed: bool = False):
    """8-bit decode of one image, the body of the reference's `inpaint` command (cli.py:80-95):

        image_from_fields(solve_image(InpaintingProblem(mask, image.channel_fields()), name, cfg).fields).pixels

    `pixels` is ImageFile.pixels -- (H,W) or (H,W,3) uint8 -- and `mask` the boolean known-pixel mask, or with
    packed=True its P4 raster (H, ceil(W/8)) as read_mask / write_mask hold it on disk (fileio.py:181-230).
    Returns (pixels_out uint8 of the same shape, reports): unpacking, channel_fields, rounding, clipping and
    the interleave run on the device (fileio.py:51-65), only 8-bit data crosses PCIe."""
    _require_built(name)
    base, mode = split_solver_name(name)
    single = mode == "single"
    cfg = cfg or MultigridConfig()
    cfg = replace(cfg, smoother=base) if single else replace(cfg, smoother=base, mode=mode)
    px = np.asarray(pixels)
    if px.dtype != np.uint8 or px.ndim not in (2, 3) or (px.ndim == 3 and px.shape[2] != 3):
        raise ValueError("pixels must be uint8 with shape (h, w) or (h, w, 3)")     # fileio.py:34-37
    h, w = px.shape[:2]
    c = 1 if px.ndim == 2 else 3
    if packed:
        bits = np.ascontiguousarray(mask, dtype=np.uint8)
        if bits.shape != (h, (w + 7) // 8):
            raise ValueError(f"packed mask must be ({h}, {(w + 7) // 8}), got {bits.shape}")
    else:
        m = np.asarray(mask)
        if m.shape != (h, w):
            raise ValueError(f"mask shape {m.shape} does not match the image {(h, w)}")
        bits = np.packbits(m.astype(bool), axis=1)
    if not np.unpackbits(bits, axis=1)[:, :w].any():
        raise EmptyMaskError("cannot solve without known pixels")
    plan = cached_plan(w, h, c, 1, cfg, spacing, single_level=single)
    out, reports = plan.solve_host_image_u8(bits[None], np.ascontiguousarray(px)[None])
    return out[0], reports


def solve_frames(masks, known, cfg: MultigridConfig | None = None, spacing: float = 1.0):
    """Batch of independent frames: masks (F,H,W), known (F,C,H,W) -> (fields, reports[F][C], elapsed)."""
    cfg = cfg or MultigridConfig()
    masks = np.asarray(masks)
    known = np.asarray(known, dtype=np.float64)
    if known.ndim == 3:
        known = known[:, None]
    if masks.ndim != 3 or known.ndim != 4 or known.shape[0] != masks.shape[0] or known.shape[2:] != masks.shape[1:]:
        raise ValueError(f"need masks (F,H,W) and known (F,C,H,W), got {masks.shape} and {known.shape}")
    if not np.isfinite(known).all():
        raise ValueError("known values contain non-finite entries")
    f, c, h, w = known.shape
    t0 = time.perf_counter()
    plan = cached_plan(w, h, c, f, cfg, spacing)
    out, reports = plan.solve_host(masks.astype(bool).view(np.uint8), known)
    elapsed = time.perf_counter() - t0
    return out, [reports[i * c:(i + 1) * c] for i in range(f)], elapsed
