"""CPU oracle for the mg-oras path -- TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/fmg_oracle.c`` (a plain-C restatement of the
reference's FMG + ORAS algorithm; each C function cites the reference file:line
it follows).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product package ``paper_2401_06744_b200`` never does.

Pinning: ``tests/test_oracle_vs_reference.py`` compares every function here
with the live reference (``/root/reference/pkg/src/diffpaint``) where that is
mounted, and ``tests/test_oracle_golden.py`` with vectors the reference wrote
(``tests/golden/``), so the oracle is pinned on the GPU box as well.

The function names and argument meanings follow the reference's Python API so
that the parity tests read like the reference's own tests.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
MAX_HIST = 256


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    src = os.path.join(_HERE, "fmg_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-B", "liboracle.so"], check=True, capture_output=True)
    return _LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [
        ("nu_pre", C.c_int), ("nu_post", C.c_int), ("v_cycles_max", C.c_int),
        ("modified", C.c_int), ("multilevel", C.c_int),
        ("block_size", C.c_int), ("overlap", C.c_int),
        ("coarse_tol", C.c_double), ("coarse_max_iters", C.c_int),
        ("tol_rel", C.c_double), ("max_outer_iters", C.c_int),
        ("alpha", C.c_double), ("eta", C.c_double),
        ("local_max_iters", C.c_int), ("threads", C.c_int),
        ("smoother", C.c_int), ("smoother_cg_iters", C.c_int),
    ]


class _Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("converged", C.c_int), ("fine_units", C.c_int),
        ("history_len", C.c_int),
        ("final_rel", C.c_double), ("baseline", C.c_double), ("init_res", C.c_double),
        ("history", C.c_double * MAX_HIST),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_axis_starts.restype = C.c_int
        L.orc_oras_sweeps.restype = C.c_int
        L.orc_hier_build.restype = C.c_void_p
        L.orc_hier_nlevels.restype = C.c_int
        L.orc_hier_level_mask.restype = C.c_void_p
        L.orc_hier_level_rhs.restype = C.c_void_p
        L.orc_hier_level_wx.restype = C.c_void_p
        L.orc_hier_level_wy.restype = C.c_void_p
        L.orc_hier_level_xs.restype = C.c_void_p
        L.orc_hier_level_ys.restype = C.c_void_p
        L.orc_fmg_solve.restype = C.c_int
        L.orc_solve_image.restype = C.c_int
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(np.asarray(a).astype(bool), dtype=np.uint8)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ----------------------------------------------------------------- configs

@dataclass(frozen=True)
class SolverConfig:
    """Same fields/defaults as the reference's SolverConfig (solvers.py:43-69)."""

    tol_rel: float = 1e-3
    max_outer_iters: int = 10_000
    alpha: float = 0.5
    local_tol_fraction: float = 1e-5
    local_max_iters: int | None = None
    smoother_cg_iters: int = 10


@dataclass(frozen=True)
class MultigridConfig:
    """Same fields/defaults as the reference's MultigridConfig (multigrid.py:50-82)."""

    nu_pre: int = 1
    nu_post: int = 1
    v_cycles_max: int = 100
    smoother: str = "oras"
    value_downsampling: str = "modified"
    mode: str = "full_multigrid"
    block_size: int = 32
    overlap: int = 6
    coarse_tol: float = 1e-8
    coarse_max_iters: int = 20_000
    solver: SolverConfig = field(default_factory=SolverConfig)


@dataclass
class SolveReport:
    solver: str
    iterations: int
    final_rel_residual: float
    history: list
    converged: bool
    baseline_residual: float
    init_residual: float
    fine_smoother_iterations: int


def _cfg(cfg, threads: int = 0) -> _Cfg:
    """Accepts this module's configs or the reference's own (duck-typed)."""
    cfg = cfg or MultigridConfig()
    if cfg.smoother not in ("oras", "cg"):
        raise ValueError(f"unknown smoother {cfg.smoother!r}")
    s = cfg.solver
    return _Cfg(
        cfg.nu_pre, cfg.nu_post, cfg.v_cycles_max,
        1 if cfg.value_downsampling == "modified" else 0,
        1 if cfg.mode == "multilevel" else 0,
        cfg.block_size, cfg.overlap, cfg.coarse_tol, cfg.coarse_max_iters,
        s.tol_rel, s.max_outer_iters, s.alpha, s.local_tol_fraction,
        int(s.local_max_iters or 0), threads,
        1 if cfg.smoother == "cg" else 0, int(s.smoother_cg_iters),
    )


def _report(r: _Report, name: str) -> SolveReport:
    return SolveReport(
        solver=name, iterations=r.iterations, final_rel_residual=r.final_rel,
        history=list(r.history[: r.history_len]), converged=bool(r.converged),
        baseline_residual=r.baseline, init_residual=r.init_res,
        fine_smoother_iterations=r.fine_units,
    )


# -------------------------------------------------------------------- core

def apply_operator(mask, spacing, u):
    """core.py:113-115 / StencilOperator.apply :100-107."""
    m, u = _u8(mask), _f64(u)
    out = np.empty_like(u)
    lib().orc_apply(_p(m), C.c_int(m.shape[0]), C.c_int(m.shape[1]), C.c_double(spacing), _p(u), _p(out))
    return out


def residual(mask, spacing, b, u):
    """StencilOperator.residual, core.py:109-110."""
    m, b, u = _u8(mask), _f64(b), _f64(u)
    out = np.empty_like(u)
    lib().orc_residual(_p(m), C.c_int(m.shape[0]), C.c_int(m.shape[1]), C.c_double(spacing), _p(b), _p(u), _p(out))
    return out


# --------------------------------------------------------------- partition

def axis_starts(dim, block, stride):
    """partition.py:84-90."""
    n = lib().orc_axis_starts(C.c_int(dim), C.c_int(block), C.c_int(stride), None, C.c_int(0))
    out = np.zeros(n, dtype=np.int64)
    lib().orc_axis_starts(C.c_int(dim), C.c_int(block), C.c_int(stride), _p(out), C.c_int(n))
    return out


def axis_weights(starts, block, dim, overlap):
    """partition.py:137-154."""
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    w = np.empty((len(starts), block))
    lib().orc_axis_weights(_p(starts), C.c_int(len(starts)), C.c_int(block), C.c_int(dim), C.c_int(overlap), _p(w))
    return w


@dataclass(frozen=True)
class Partition:
    width: int
    height: int
    block_size: int
    overlap: int
    xs: np.ndarray
    ys: np.ndarray
    block_w: int
    block_h: int

    @property
    def nx(self):
        return len(self.xs)

    @property
    def ny(self):
        return len(self.ys)

    @property
    def nblocks(self):
        return self.nx * self.ny


def build_partition(width, height, block_size=32, overlap=6) -> Partition:
    """partition.py:93-116."""
    if width < 1 or height < 1:
        raise ValueError("image dimensions must be >= 1")
    if overlap < 0 or block_size <= overlap:
        raise ValueError("need block_size > overlap >= 0")
    stride = block_size - overlap
    return Partition(width, height, block_size, overlap,
                     axis_starts(width, block_size, stride), axis_starts(height, block_size, stride),
                     min(block_size, width), min(block_size, height))


def build_weights(part: Partition):
    """partition.py:157-168; returns (wx, wy)."""
    return (axis_weights(part.xs, part.block_w, part.width, part.overlap),
            axis_weights(part.ys, part.block_h, part.height, part.overlap))


# ----------------------------------------------------------------- solvers

def solve_blocks(mask, spacing, block, overlap, alpha, r, target_sq, max_iters, threads=0):
    """BlockSolver.gather + solve_blocks (solvers.py:303-305, :372-390)."""
    m, r = _u8(mask), _f64(r)
    h, w = m.shape
    part = build_partition(w, h, block, overlap)
    v = np.empty((part.nblocks, part.block_h, part.block_w))
    lib().orc_solve_blocks(_p(m), C.c_int(h), C.c_int(w), C.c_double(spacing), C.c_int(block),
                           C.c_int(overlap), C.c_double(alpha), _p(r), C.c_double(target_sq),
                           C.c_int(max_iters), C.c_int(threads), _p(v))
    return v


def scatter_weighted(shape, block, overlap, v):
    """BlockSolver.scatter_weighted (solvers.py:307-314)."""
    h, w = shape
    v = _f64(v)
    out = np.empty((h, w))
    lib().orc_scatter_weighted(C.c_int(h), C.c_int(w), C.c_int(block), C.c_int(overlap), _p(v), _p(out))
    return out


def oras_sweeps(mask, spacing, block, overlap, alpha, b, u, *, max_sweeps, stop_norm=0.0,
                eta=1e-5, local_max_iters=None, threads=0):
    """oras_sweeps (solvers.py:393-424); u is updated in place. Returns (sweeps, rn)."""
    m, b = _u8(mask), _f64(b)
    assert u.dtype == np.float64 and u.flags.c_contiguous
    rn = C.c_double(0.0)
    s = lib().orc_oras_sweeps(_p(m), C.c_int(m.shape[0]), C.c_int(m.shape[1]), C.c_double(spacing),
                              C.c_int(block), C.c_int(overlap), C.c_double(alpha), _p(b), _p(u),
                              C.c_int(max_sweeps), C.c_double(stop_norm), C.c_double(eta),
                              C.c_int(int(local_max_iters or 0)), C.c_int(threads), C.byref(rn))
    return int(s), float(rn.value)


def oras_solve(mask, known, spacing=1.0, block=32, overlap=6, cfg=None):
    """oras_solve (solvers.py:427-485) from the flat initialisation, one channel: `known` (h,w).
    Built from orc_oras_sweeps one sweep per call (each call ends with the residual evaluation
    whose norm is the next history entry), so the iterates are those of one long call.
    Returns (u, report dict with the SolveReport fields)."""
    cfg = cfg or SolverConfig()
    m = np.asarray(mask, dtype=bool)
    b = np.where(m, np.asarray(known, dtype=np.float64), 0.0)
    u = b.copy()
    r0 = float(np.linalg.norm(residual(m, spacing, b, u)))
    rep = dict(solver="oras", iterations=0, final_rel_residual=0.0, history=[0.0], converged=True,
               baseline_residual=r0, init_residual=r0, fine_smoother_iterations=0)
    if r0 == 0.0:
        return u, rep
    stop = cfg.tol_rel * r0
    history, sweeps, rn = [1.0], 0, r0
    while not (rn <= stop or sweeps >= cfg.max_outer_iters):
        done, rn = oras_sweeps(m, spacing, block, overlap, cfg.alpha, b, u, max_sweeps=1, stop_norm=0.0,
                               eta=cfg.local_tol_fraction, local_max_iters=cfg.local_max_iters)
        if done == 0:  # rs == 0
            break
        sweeps += done
        history.append(rn / r0)
    rel = rn / r0
    rep.update(iterations=sweeps, final_rel_residual=rel, history=history, converged=rel <= cfg.tol_rel,
               fine_smoother_iterations=sweeps)
    return u, rep


# --------------------------------------------------------------- multigrid

def downsample_mask(fine):
    """multigrid.py:98-101."""
    f = _u8(fine)
    h, w = f.shape
    out = np.empty(((h + 1) // 2, (w + 1) // 2), dtype=np.uint8)
    lib().orc_downsample_mask(_p(f), C.c_int(h), C.c_int(w), _p(out))
    return out.astype(bool)


def downsample_values_naive(fine_mask, fine_rhs):
    """multigrid.py:104-109."""
    f, r = _u8(fine_mask), _f64(fine_rhs)
    h, w = f.shape
    out = np.empty(((h + 1) // 2, (w + 1) // 2))
    lib().orc_downsample_values_naive(_p(f), _p(r), C.c_int(h), C.c_int(w), _p(out))
    return out


def downsample_values_modified(fine_mask, coarse_mask, fine_rhs):
    """multigrid.py:112-146."""
    f, cm, r = _u8(fine_mask), _u8(coarse_mask), _f64(fine_rhs)
    h, w = f.shape
    out = np.empty(((h + 1) // 2, (w + 1) // 2))
    lib().orc_downsample_values_modified(_p(f), _p(cm), _p(r), C.c_int(h), C.c_int(w), _p(out))
    return out


def restrict_residual(fine_r, coarse_mask):
    """multigrid.py:149-154."""
    r, cm = _f64(fine_r), _u8(coarse_mask)
    h, w = r.shape
    out = np.empty(((h + 1) // 2, (w + 1) // 2))
    lib().orc_restrict_residual(_p(r), C.c_int(h), C.c_int(w), _p(cm), _p(out))
    return out


def _check_halves(coarse, fine_shape):
    hf, wf = fine_shape
    if coarse.shape != ((hf + 1) // 2, (wf + 1) // 2):
        raise ValueError(f"coarse shape {coarse.shape} does not halve fine shape {fine_shape}")


def prolongate_correction(coarse_e, fine_mask):
    """multigrid.py:175-177."""
    c, fm = _f64(coarse_e), _u8(fine_mask)
    _check_halves(c, fm.shape)
    out = np.empty(fm.shape)
    lib().orc_prolongate_correction(_p(c), _p(fm), C.c_int(fm.shape[0]), C.c_int(fm.shape[1]), _p(out))
    return out


def prolongate_solution(coarse_u, fine_mask, fine_rhs):
    """multigrid.py:180-186."""
    c, fm, fr = _f64(coarse_u), _u8(fine_mask), _f64(fine_rhs)
    _check_halves(c, fm.shape)
    out = np.empty(fm.shape)
    lib().orc_prolongate_solution(_p(c), _p(fm), _p(fr), C.c_int(fm.shape[0]), C.c_int(fm.shape[1]), _p(out))
    return out


class Level:
    def __init__(self, h, w, nx, ny, bw, bh, spacing, mask, rhs, xs, ys, wx, wy):
        self.shape = (h, w)
        self.nx, self.ny, self.block_w, self.block_h = nx, ny, bw, bh
        self.spacing = spacing
        self.mask, self.rhs, self.xs, self.ys, self.wx, self.wy = mask, rhs, xs, ys, wx, wy


class Hierarchy:
    """build_hierarchy (multigrid.py:236-261); owns the C-side level arrays."""

    def __init__(self, mask, known, spacing=1.0, cfg=None, threads=0):
        m = _u8(mask)
        k = _f64(known)
        if k.ndim == 2:
            k = k[None]
        self.channels = k.shape[0]
        self.cfg = cfg or MultigridConfig()
        self._c = _cfg(self.cfg, threads)
        h, w = m.shape
        self._h = C.c_void_p(lib().orc_hier_build(_p(m), _p(k), C.c_int(h), C.c_int(w), C.c_int(self.channels),
                                                  C.c_double(spacing), C.byref(self._c)))
        self.levels = []
        L = lib()
        for l in range(L.orc_hier_nlevels(self._h)):
            info = (C.c_int * 6)()
            sp = C.c_double()
            L.orc_hier_level_info(self._h, C.c_int(l), info, C.byref(sp))
            hh, ww, nx, ny, bw, bh = list(info)

            def arr(ptr, shape, dt):
                n = int(np.prod(shape))
                buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
                return np.frombuffer(buf, dtype=dt).reshape(shape).copy()

            self.levels.append(Level(
                hh, ww, nx, ny, bw, bh, sp.value,
                arr(L.orc_hier_level_mask(self._h, C.c_int(l)), (hh, ww), np.uint8).astype(bool),
                arr(L.orc_hier_level_rhs(self._h, C.c_int(l)), (self.channels, hh, ww), np.float64),
                arr(L.orc_hier_level_xs(self._h, C.c_int(l)), (nx,), np.int64),
                arr(L.orc_hier_level_ys(self._h, C.c_int(l)), (ny,), np.int64),
                arr(L.orc_hier_level_wx(self._h, C.c_int(l)), (nx, bw), np.float64),
                arr(L.orc_hier_level_wy(self._h, C.c_int(l)), (ny, bh), np.float64),
            ))

    def __len__(self):
        return len(self.levels)

    def __del__(self):
        try:
            if self._h:
                lib().orc_hier_free(self._h)
                self._h = None
        except Exception:
            pass


def build_hierarchy(mask, known, spacing=1.0, cfg=None, threads=0) -> Hierarchy:
    return Hierarchy(mask, known, spacing, cfg, threads)


def v_cycle(hier: Hierarchy, level, u, rhs, cfg=None, threads=0):
    """multigrid.py:335-371; u in place; returns finest-level smoother units used."""
    c = _cfg(cfg or hier.cfg, threads)
    rhs = _f64(rhs)
    assert u.dtype == np.float64 and u.flags.c_contiguous
    fu = C.c_int(0)
    lib().orc_v_cycle(hier._h, C.c_int(level), _p(u), _p(rhs), C.byref(c), C.byref(fu))
    return int(fu.value)


def cascadic_init(hier: Hierarchy, cfg=None, channel=0, threads=0):
    """multigrid.py:374-386."""
    c = _cfg(cfg or hier.cfg, threads)
    u = np.empty(hier.levels[0].shape)
    lib().orc_cascadic_init(hier._h, C.byref(c), C.c_int(channel), _p(u))
    return u


def fmg_solve(hier: Hierarchy, cfg=None, channel=0, threads=0):
    """multigrid.py:425-487; returns (u, SolveReport)."""
    cfg = cfg or hier.cfg
    c = _cfg(cfg, threads)
    u = np.empty(hier.levels[0].shape)
    rep = _Report()
    rc = lib().orc_fmg_solve(hier._h, C.byref(c), C.c_int(channel), _p(u), C.byref(rep))
    if rc != 0:
        raise ValueError("cannot solve without known pixels")
    return u, _report(rep, ("ml-" if cfg.mode == "multilevel" else "mg-") + cfg.smoother)


def solve_image(mask, known, spacing=1.0, cfg=None, threads=0):
    """pipelines.py:96-114 for "mg-oras"/"ml-oras"; returns (fields (C,h,w), reports)."""
    cfg = cfg or MultigridConfig()
    m, k = _u8(mask), _f64(known)
    if k.ndim == 2:
        k = k[None]
    c = _cfg(cfg, threads)
    out = np.empty_like(k)
    reps = (_Report * k.shape[0])()
    rc = lib().orc_solve_image(_p(m), _p(k), C.c_int(m.shape[0]), C.c_int(m.shape[1]), C.c_int(k.shape[0]),
                               C.c_double(spacing), C.byref(c), _p(out), reps)
    if rc != 0:
        raise ValueError("cannot solve without known pixels")
    name = ("ml-" if cfg.mode == "multilevel" else "mg-") + cfg.smoother
    return out, [_report(r, name) for r in reps]


def cg_solve(mask, known, spacing=1.0, cfg=None):
    """cg_solve (solvers.py:140-186) from the flat initialisation, one channel: known (h,w).
    Returns (u, SolveReport)."""
    cfg = cfg or SolverConfig()
    m, k = _u8(mask), _f64(known)
    u = np.empty_like(k)
    rep = _Report()
    rc = lib().orc_cg_solve(_p(m), _p(k), C.c_int(m.shape[0]), C.c_int(m.shape[1]), C.c_double(spacing),
                            C.c_double(cfg.tol_rel), C.c_int(cfg.max_outer_iters), _p(u), C.byref(rep))
    if rc != 0:
        raise ValueError("cannot solve without known pixels")
    return u, _report(rep, "cg")


def counters_reset():
    lib().orc_counters_reset()


def counters():
    """(block-CG iterations, block solves, sweeps) since the last reset."""
    out = (C.c_longlong * 3)()
    lib().orc_counters_get(out)
    return tuple(int(x) for x in out)


# ------------------------------------------------ synthetic inputs (masks.py)
# The reference's benchmark recipe (masks.py:13-25, :50-67; tests/conftest.py:7-12)
# restated with the same Generator calls, hence the same bits (pinned by
# tests/test_oracle_vs_reference.py::test_input_generators_are_bit_identical).

def random_mask(width, height, density, seed=0):
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    total = width * height
    wanted = int(round(density * total))
    if wanted < 1:
        raise ValueError("density selects zero pixels")
    chosen = np.random.default_rng(seed).choice(total, size=wanted, replace=False)
    flat = np.zeros(total, dtype=bool)
    flat[chosen] = True
    return flat.reshape(height, width)


def _lattice_axis(n_nodes, n_px):
    pos = np.linspace(0.0, n_nodes - 1.0, n_px)
    cell = np.clip(pos.astype(int), 0, n_nodes - 2)
    return cell, pos - cell


def synthetic_image(width, height, seed=0):
    gx, gy = max(2, width // 24 + 2), max(2, height // 24 + 2)
    nodes = np.random.default_rng(seed).uniform(0.0, 255.0, size=(gy, gx))
    cy, fy = _lattice_axis(gy, height)
    cx, fx = _lattice_axis(gx, width)
    hi = nodes[cy][:, cx] * (1 - fx) + nodes[cy][:, cx + 1] * fx
    lo = nodes[cy + 1][:, cx] * (1 - fx) + nodes[cy + 1][:, cx + 1] * fx
    return np.ascontiguousarray(np.rint(hi * (1 - fy)[:, None] + lo * fy[:, None]), dtype=np.float64)


def seeded_problem(width, height, density, seed, channels=1):
    """(mask, known (C,h,w)) of the reference's tests/conftest.py:7-12 recipe."""
    mask = random_mask(width, height, density, seed)
    known = np.stack([synthetic_image(width, height, seed + 1000 + c) for c in range(channels)])
    return mask, known
