"""Full-multigrid driver of the mg-oras path, device-backed.

Interface of the reference's ``diffpaint.multigrid`` (multigrid.py:50-487) for
``mode="full_multigrid"``, ``smoother="oras"``: MultigridConfig, the transfer
operators, build_hierarchy, cascadic_init, v_cycle and fmg_solve.  Everything
numeric runs in libb200paint (CUDA graphs of the K1-K7 kernels); this module
validates arguments, owns plans and converts reports.
"""

from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _dev, _lib
from .core import EmptyMaskError, InpaintingProblem, StencilOperator, as_mask
from .partition import BlockPartition, BlockWeights, build_partition, build_weights
from .solvers import SolveReport, SolverConfig

SMOOTHERS = ("oras", "cg")
MODES = ("multilevel", "full_multigrid")
DOWNSAMPLINGS = ("naive", "modified")


@dataclass(frozen=True)
class MultigridConfig:
    """multigrid.py:50-82 (same fields, defaults and validation)."""

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

    def __post_init__(self):
        if self.nu_pre + self.nu_post < 1:
            raise ValueError("need at least one smoothing iteration per cycle")
        if self.smoother not in SMOOTHERS:
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.value_downsampling not in DOWNSAMPLINGS:
            raise ValueError(f"unknown value downsampling {self.value_downsampling!r}")


def _require_hot_path(cfg) -> None:
    if cfg.smoother not in ("oras", "cg"):
        raise NotImplementedError(f"unknown smoother {cfg.smoother!r}")


# --------------------------------------------------------------------- plan

class Plan:
    """RAII wrapper of a ``b200p_plan`` (geometry, scratch, CUDA graphs)."""

    def __init__(self, width, height, channels=1, frames=1, cfg=None, spacing=1.0,
                 use_graphs=True, single_level=False):
        cfg = cfg or MultigridConfig()
        _require_hot_path(cfg)
        _dev.require_cuda()
        s = cfg.solver
        c = _lib.Config()
        _lib.lib().b200p_config_default(C.byref(c), int(width), int(height), int(channels))
        c.frames = int(frames)
        c.spacing = float(spacing)
        c.block_size, c.overlap = int(cfg.block_size), int(cfg.overlap)
        c.nu_pre, c.nu_post, c.v_cycles_max = int(cfg.nu_pre), int(cfg.nu_post), int(cfg.v_cycles_max)
        c.value_downsampling = 1 if cfg.value_downsampling == "modified" else 0
        c.coarse_tol, c.coarse_max_iters = float(cfg.coarse_tol), int(cfg.coarse_max_iters)
        c.tol_rel, c.alpha, c.eta = float(s.tol_rel), float(s.alpha), float(s.local_tol_fraction)
        c.local_max_iters = int(s.local_max_iters or 0)
        c.use_graphs = 1 if use_graphs else 0
        # single_level: oras_solve on the finest level only (the "oras" pipeline, solvers.py:427-485)
        c.mode = 2 if single_level else (1 if cfg.mode == "multilevel" else 0)
        self.single_level = bool(single_level)
        c.smoother = 1 if cfg.smoother == "cg" else 0
        c.smoother_cg_iters = int(s.smoother_cg_iters)
        c.max_outer_iters = int(s.max_outer_iters)
        self.config = c
        self.cfg = cfg
        self.width, self.height, self.channels, self.frames = int(width), int(height), int(channels), int(frames)
        self.problems = self.channels * self.frames
        h = C.c_void_p()
        _lib.check(_lib.lib().b200p_plan_create(C.byref(c), C.byref(h)))
        self.handle = h
        self.num_levels = _lib.lib().b200p_plan_num_levels(h)

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib().b200p_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- information
    def level_info(self, level) -> _lib.LevelInfo:
        info = _lib.LevelInfo()
        _lib.check(_lib.lib().b200p_plan_level_info(self.handle, int(level), C.byref(info)))
        return info

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().b200p_plan_device_bytes(self.handle))

    @property
    def launch_count(self) -> int:
        return int(_lib.lib().b200p_plan_launch_count(self.handle))

    def set_ingest(self, dense: bool = False, host_gather: bool = False):
        """Host f64 entry points: default = sparse ingest when the mask is sparse (from a pinned source the device
        fetches the values itself; lowest latency of a single solve); dense = always DMA the planes;
        host_gather = sparse, with the (index, values) list always gathered by the library's host threads
        (12 MB instead of 207 MB per 4K RGB frame on the link, and no device reads of host memory)."""
        if dense and host_gather:
            raise ValueError("dense and host_gather exclude each other")
        _lib.check(_lib.lib().b200p_plan_set_ingest(self.handle, 1 if dense else (2 if host_gather else 0)))

    def last_transfer_bytes(self):
        """(H2D, D2H) bytes copied by the last host entry point (the f64 ingest is sparse when the mask is)."""
        a, b = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().b200p_plan_last_transfer_bytes(self.handle, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def profile(self, enable: bool):
        _lib.check(_lib.lib().b200p_plan_profile(self.handle, 1 if enable else 0))

    def profile_summary(self) -> dict:
        """{kernel kind: (total ms, launches, algorithmic bytes)} since profile(True)."""
        L = _lib.lib()
        out = {}
        for k in range(L.b200p_plan_profile_kinds()):
            ms, n, by = C.c_double(), C.c_int64(), C.c_double()
            _lib.check(L.b200p_plan_profile_get(self.handle, k, C.byref(ms), C.byref(n), C.byref(by)))
            if n.value:
                out[L.b200p_plan_profile_name(k).decode()] = (ms.value, n.value, by.value)
        return out

    # -- solves
    def _reports(self, raw, wall):
        reps = []
        base = self.cfg.smoother
        name = base if self.single_level else ("ml-" if self.cfg.mode == "multilevel" else "mg-") + base
        for p, r in enumerate(raw):
            reps.append(SolveReport(
                solver=name, iterations=r.iterations, final_rel_residual=r.final_rel_residual,
                wall_time=wall, history=self._history(r, p),
                converged=bool(r.converged),
                baseline_residual=r.baseline_residual, init_residual=r.init_residual,
                fine_smoother_iterations=r.fine_smoother_iterations))
        return reps

    def _history(self, r, p):
        """The report record stores the first B200P_MAX_HISTORY values; a longer history (comparison pipelines
        that record per sweep / step, v_cycles_max > 127) is fetched whole from the plan's device buffer, which
        is sized from the config's iteration caps (`b200p_plan_history`): never truncated, like the reference's
        list.  Only a history past even that buffer (more than 2^22 values) is cut, loudly."""
        cap = len(r.history)
        if r.history_len <= cap:
            return list(r.history[: r.history_len]) or [r.final_rel_residual]
        full = np.empty(r.history_len)
        got = _lib.lib().b200p_plan_history(self.handle, int(p), full.ctypes.data, int(r.history_len))
        if got < 0:
            _lib.check(got)
        if got >= r.history_len:
            return full.tolist()
        import warnings
        warnings.warn(f"residual history truncated: {r.history_len} values recorded, the first {got} and the "
                      f"last are kept", RuntimeWarning, stacklevel=3)
        return full[:got].tolist() + [r.final_rel_residual]

    def solve_device(self, d_mask, d_known, d_out=None, want_reports=True):
        """Device-resident solve: mask (F,H,W) uint8, known (F,C,H,W) float64 CUDA tensors."""
        if d_out is None:
            d_out = _dev.empty_f64((self.frames, self.channels, self.height, self.width))
        n = self.height * self.width
        _dev.check_tensor(d_mask, "mask", "uint8", self.frames * n)
        _dev.check_tensor(d_known, "known", "float64", self.problems * n)
        _dev.check_tensor(d_out, "out", "float64", self.problems * n)
        raw = (_lib.Report * self.problems)() if want_reports else None
        t0 = time.perf_counter()
        _dev.call("b200p_solve", self.handle, _dev.ptr(d_mask), _dev.ptr(d_known), _dev.ptr(d_out),
                  C.cast(raw, C.c_void_p) if raw is not None else None, _dev.stream())
        wall = time.perf_counter() - t0
        return d_out, (self._reports(raw, wall) if raw is not None else None)

    def _check_host(self, mask, known, out, dtype, packed_mask=False):
        """The C side reads F*H*W mask bytes (F*H*ceil(W/8) for a bit-packed raster) and P*H*W values and
        writes P*H*W values through raw host pointers: element counts, dtypes and contiguity are checked
        here (the device path has _dev.check_tensor for the same reason)."""
        n = self.height * self.width
        mask_count = self.frames * (self.height * ((self.width + 7) // 8) if packed_mask else n)
        for a, name, dt, count in ((mask, "mask", np.uint8, mask_count),
                                   (known, "known", dtype, self.problems * n),
                                   (out, "out", dtype, self.problems * n)):
            if not isinstance(a, np.ndarray) or a.dtype != dt or not a.flags.c_contiguous:
                raise ValueError(f"{name} must be a C-contiguous {np.dtype(dt)} array")
            if a.size != count:
                raise ValueError(f"{name} has {a.size} elements, this plan needs {count} "
                                 f"({self.frames} frame(s) x {self.channels} channel(s) x {self.height} x {self.width})")
            if name == "out" and not a.flags.writeable:
                raise ValueError("out must be writeable")

    def solve_host(self, mask, known, out=None):
        """Host buffers in and out (H2D + solve + D2H inside the call)."""
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        known = np.ascontiguousarray(known, dtype=np.float64)
        if out is None:
            out = _dev.empty_host((self.frames, self.channels, self.height, self.width))
        self._check_host(mask, known, out, np.float64)
        raw = (_lib.Report * self.problems)()
        t0 = time.perf_counter()
        _dev.call("b200p_solve_host", self.handle, mask.ctypes.data, known.ctypes.data, out.ctypes.data,
                  C.cast(raw, C.c_void_p))
        wall = time.perf_counter() - t0
        return out, self._reports(raw, wall)

    def solve_host_async(self, mask, known, out, u8: bool = False, image: bool = False):
        """Enqueue H2D + solve + D2H on the plan's stream and return; `wait()` completes it.
        The arrays must be C-contiguous, of the exact dtypes, and stay alive until `wait()`.
        image=True: the 8-bit file layouts -- mask = P4 raster bits (F,H,ceil(W/8)), known / out =
        interleaved pixels (F,H,W,C) (see solve_host_image_u8)."""
        u8 = u8 or image
        self._check_host(mask, known, out, np.uint8 if u8 else np.float64, packed_mask=image)
        self._t0 = time.perf_counter()
        entry = "b200p_solve_host_image_u8_async" if image else (
            "b200p_solve_host_u8_async" if u8 else "b200p_solve_host_async")
        _dev.call(entry, self.handle, mask.ctypes.data, known.ctypes.data, out.ctypes.data)
        self._keep = (mask, known, out)

    def wait(self):
        """Complete the pending asynchronous solve; returns its SolveReports."""
        raw = (_lib.Report * self.problems)()
        _dev.call("b200p_solve_wait", self.handle, C.cast(raw, C.c_void_p))
        self._keep = None
        return self._reports(raw, time.perf_counter() - self._t0)

    def solve_host_u8(self, mask, known_u8, out=None):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        known_u8 = np.ascontiguousarray(known_u8, dtype=np.uint8)
        if out is None:
            out = _dev.empty_host((self.frames, self.channels, self.height, self.width), np.uint8)
        self._check_host(mask, known_u8, out, np.uint8)
        raw = (_lib.Report * self.problems)()
        t0 = time.perf_counter()
        _dev.call("b200p_solve_host_u8", self.handle, mask.ctypes.data, known_u8.ctypes.data,
                  out.ctypes.data, C.cast(raw, C.c_void_p))
        wall = time.perf_counter() - t0
        return out, self._reports(raw, wall)


    def solve_host_image_u8(self, mask_bits, pixels, out=None):
        """8-bit images as they are on disk: `pixels` (F,H,W,C) uint8 interleaved (ImageFile.pixels,
        fileio.py:27-37; C = 1 may be (F,H,W)), `mask_bits` (F,H,ceil(W/8)) the P4 raster of
        read_mask / write_mask (fileio.py:181-230, = np.packbits(mask, axis=-1)).  Returns
        (image_from_fields(fields).pixels per frame, reports): channel_fields, the rounding, the clip and
        the interleave run on the device (fileio.py:51-65)."""
        mask_bits = np.ascontiguousarray(mask_bits, dtype=np.uint8)
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
        if out is None:
            out = _dev.empty_host(pixels.shape, np.uint8)
        self._check_host(mask_bits, pixels, out, np.uint8, packed_mask=True)
        raw = (_lib.Report * self.problems)()
        t0 = time.perf_counter()
        _dev.call("b200p_solve_host_image_u8", self.handle, mask_bits.ctypes.data, pixels.ctypes.data,
                  out.ctypes.data, C.cast(raw, C.c_void_p))
        wall = time.perf_counter() - t0
        return out, self._reports(raw, wall)


_PLAN_CACHE: dict = {}
_PLAN_CACHE_MAX = 4
_PLAN_CACHE_LOCK = threading.Lock()


def _cfg_key(cfg):
    s = cfg.solver
    return (cfg.nu_pre, cfg.nu_post, cfg.v_cycles_max, cfg.value_downsampling, cfg.block_size,
            cfg.overlap, cfg.coarse_tol, cfg.coarse_max_iters, s.tol_rel, s.alpha,
            s.local_tol_fraction, s.local_max_iters, cfg.mode, s.max_outer_iters, cfg.smoother,
            s.smoother_cg_iters)


def cached_plan(width, height, channels, frames, cfg, spacing=1.0, single_level=False) -> Plan:
    """Plans are expensive (device scratch + graph capture); reuse by configuration."""
    key = (width, height, channels, frames, float(spacing), _cfg_key(cfg), bool(single_level))
    with _PLAN_CACHE_LOCK:
        plan = _PLAN_CACHE.pop(key, None)
        if plan is None or not plan.handle:
            # Eviction only drops the cache's reference: a LevelHierarchy (or any caller) may still hold the
            # plan, so it is never closed here -- Plan.__del__ frees it with the last reference.
            while len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
                _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
            plan = Plan(width, height, channels, frames, cfg, spacing, single_level=single_level)
        _PLAN_CACHE[key] = plan
        return plan


def clear_plan_cache():
    """Drop the cache's references (plans still held elsewhere stay valid)."""
    with _PLAN_CACHE_LOCK:
        _PLAN_CACHE.clear()


def _stage_plan(mask, spacing, block_size, overlap, alpha, eta, local_max_iters) -> Plan:
    """Single-field plan with its level-0 mask bound, for the stage-level calls."""
    mask = np.asarray(mask).astype(bool)
    h, w = mask.shape
    cfg = MultigridConfig(block_size=block_size, overlap=overlap,
                          solver=SolverConfig(alpha=alpha, local_tol_fraction=eta,
                                              local_max_iters=local_max_iters))
    plan = cached_plan(w, h, 1, 1, cfg, spacing)
    d_mask = _dev.to_device_u8(mask)
    d_known = _dev.empty_f64((1, h, w)).zero_()
    _dev.call("b200p_plan_build_hierarchy", plan.handle, _dev.ptr(d_mask), _dev.ptr(d_known), _dev.stream())
    plan._stage_keep = (d_mask, d_known)
    return plan


# ---------------------------------------------------------------- transfers

def _coarse_shape(shape):
    return ((shape[0] + 1) // 2, (shape[1] + 1) // 2)


def downsample_mask(fine) -> np.ndarray:
    """2x2 max pooling with ceil dims (multigrid.py:98-101)."""
    f = as_mask(fine)
    h, w = f.shape
    d_f = _dev.to_device_u8(f)
    d_c = _dev.empty_u8(_coarse_shape(f.shape))
    _dev.call("b200p_downsample_mask", _dev.ptr(d_f), h, w, _dev.ptr(d_c), _dev.stream())
    return _dev.to_host(d_c).astype(bool)


def _downsample_values(fine_mask, coarse_mask, fine_rhs, modified):
    fm = as_mask(fine_mask)
    h, w = fm.shape
    cm = as_mask(coarse_mask) if coarse_mask is not None else downsample_mask(fm)
    if cm.shape != _coarse_shape(fm.shape):
        raise ValueError(f"coarse mask shape {cm.shape} does not halve {fm.shape}")
    d_fm, d_cm = _dev.to_device_u8(fm), _dev.to_device_u8(cm)
    d_r = _dev.to_device_f64(fine_rhs)
    d_o = _dev.empty_f64(cm.shape)
    _dev.call("b200p_downsample_values", _dev.ptr(d_fm), _dev.ptr(d_cm), _dev.ptr(d_r), h, w,
              1 if modified else 0, _dev.ptr(d_o), _dev.stream())
    return _dev.to_host(d_o)


def downsample_values_naive(fine_mask, fine_rhs) -> np.ndarray:
    """multigrid.py:104-109."""
    return _downsample_values(fine_mask, None, fine_rhs, False)


def downsample_values_modified(fine_mask, coarse_mask, fine_rhs) -> np.ndarray:
    """multigrid.py:112-146."""
    return _downsample_values(fine_mask, coarse_mask, fine_rhs, True)


def restrict_residual(fine_r, coarse_mask) -> np.ndarray:
    """multigrid.py:149-154."""
    r = np.asarray(fine_r, dtype=np.float64)
    cm = as_mask(coarse_mask)
    if cm.shape != _coarse_shape(r.shape):
        raise ValueError(f"coarse mask shape {cm.shape} does not halve {r.shape}")
    d_r, d_cm = _dev.to_device_f64(r), _dev.to_device_u8(cm)
    d_o = _dev.empty_f64(cm.shape)
    _dev.call("b200p_restrict_residual", _dev.ptr(d_r), _dev.ptr(d_cm), r.shape[0], r.shape[1],
              _dev.ptr(d_o), _dev.stream())
    return _dev.to_host(d_o)


def prolongate_correction(coarse_e, fine_mask) -> np.ndarray:
    """multigrid.py:175-177 (returned as a field; the fused kernel adds it to u = 0)."""
    fm = as_mask(fine_mask)
    e = np.asarray(coarse_e, dtype=np.float64)
    if e.shape != _coarse_shape(fm.shape):
        raise ValueError(f"coarse shape {e.shape} does not halve fine shape {fm.shape}")
    d_e, d_fm = _dev.to_device_f64(e), _dev.to_device_u8(fm)
    d_u = _dev.empty_f64(fm.shape).zero_()
    _dev.call("b200p_prolongate_correct", _dev.ptr(d_e), _dev.ptr(d_fm), fm.shape[0], fm.shape[1],
              _dev.ptr(d_u), _dev.stream())
    return _dev.to_host(d_u)


def prolongate_solution(coarse_u, fine_mask, fine_rhs) -> np.ndarray:
    """multigrid.py:180-186."""
    fm = as_mask(fine_mask)
    c = np.asarray(coarse_u, dtype=np.float64)
    if c.shape != _coarse_shape(fm.shape):
        raise ValueError(f"coarse shape {c.shape} does not halve fine shape {fm.shape}")
    d_c, d_fm, d_b = _dev.to_device_f64(c), _dev.to_device_u8(fm), _dev.to_device_f64(fine_rhs)
    d_u = _dev.empty_f64(fm.shape)
    _dev.call("b200p_prolongate_solution", _dev.ptr(d_c), _dev.ptr(d_fm), _dev.ptr(d_b), fm.shape[0],
              fm.shape[1], _dev.ptr(d_u), _dev.stream())
    return _dev.to_host(d_u)


# ---------------------------------------------------------------- hierarchy

class Level:
    """One resolution level (multigrid.py:189-225); arrays are copies of device data."""

    def __init__(self, mask, rhs, spacing, block_size, overlap):
        self.mask = mask
        self.rhs = rhs
        self.spacing = spacing
        self.op = StencilOperator(mask, spacing)
        h, w = mask.shape
        self.part: BlockPartition = build_partition(w, h, block_size, overlap)
        self.weights: BlockWeights = build_weights(self.part)

    @property
    def shape(self):
        return self.mask.shape

    def flat_init(self, channel):
        return self.rhs[channel].copy()


class LevelHierarchy:
    """Fine-to-coarse levels (multigrid.py:228-261), built on the device."""

    def __init__(self, problem: InpaintingProblem, cfg: MultigridConfig):
        self.problem = problem
        self.cfg = cfg
        self.value_downsampling = cfg.value_downsampling
        h, w = problem.shape
        # the data half runs on the GPU; smoother/mode do not affect the levels
        hot = replace(cfg, smoother="oras", mode="full_multigrid")
        self.plan = cached_plan(w, h, problem.channels, 1, hot, problem.spacing)
        self._d_mask = _dev.to_device_u8(problem.mask)
        self._d_known = _dev.to_device_f64(problem.known)
        self._bind()
        self._levels = None

    def _bind(self):
        _dev.call("b200p_plan_build_hierarchy", self.plan.handle, _dev.ptr(self._d_mask),
                  _dev.ptr(self._d_known), _dev.stream())

    def _fetch(self, level):
        import torch
        info = self.plan.level_info(level)
        h, w = info.height, info.width
        if level == 0:
            return self.problem.mask, np.where(self.problem.mask[None], self.problem.known, 0.0)
        pm, pr = C.c_void_p(), C.c_void_p()
        _lib.check(_lib.lib().b200p_plan_level_ptrs(self.plan.handle, level, C.byref(pm), C.byref(pr)))
        m = np.empty((h, w), dtype=np.uint8)
        r = np.empty((self.problem.channels, h, w))
        torch.cuda.synchronize()
        _dev.call("b200p_memcpy_d2h", m.ctypes.data, pm, m.nbytes)
        _dev.call("b200p_memcpy_d2h", r.ctypes.data, pr, r.nbytes)
        return m.astype(bool), r

    @property
    def levels(self):
        if self._levels is None:
            self._bind()  # the cached plan may have served another problem since
            out = []
            for l in range(self.plan.num_levels):
                info = self.plan.level_info(l)
                m, r = self._fetch(l)
                out.append(Level(m, r, info.spacing, self.cfg.block_size, self.cfg.overlap))
            self._levels = out
        return self._levels

    def __len__(self):
        return self.plan.num_levels


def build_hierarchy(problem: InpaintingProblem, cfg: MultigridConfig | None = None) -> LevelHierarchy:
    """multigrid.py:236-261."""
    return LevelHierarchy(problem, cfg or MultigridConfig())


def _channel_plan(hier: LevelHierarchy, cfg: MultigridConfig, channel: int):
    """Single-channel plan with the hierarchy of `channel` built on the device."""
    p = hier.problem
    if not 0 <= channel < p.channels:
        raise IndexError(f"channel {channel} out of range")
    h, w = p.shape
    plan = cached_plan(w, h, 1, 1, cfg, p.spacing)
    d_mask = hier._d_mask
    d_known = hier._d_known[channel:channel + 1].contiguous()
    _dev.call("b200p_plan_build_hierarchy", plan.handle, _dev.ptr(d_mask), _dev.ptr(d_known), _dev.stream())
    plan._stage_keep = (d_mask, d_known)
    return plan, d_mask, d_known


def cascadic_init(hier: LevelHierarchy, cfg: MultigridConfig | None = None, channel: int = 0) -> np.ndarray:
    """multigrid.py:374-386."""
    cfg = cfg or hier.cfg
    _require_hot_path(cfg)
    plan, _, _ = _channel_plan(hier, cfg, channel)
    d_u = _dev.empty_f64(hier.problem.shape)
    _dev.call("b200p_plan_cascade", plan.handle, _dev.ptr(d_u), _dev.stream())
    return _dev.to_host(d_u)


def v_cycle(hier: LevelHierarchy, level: int, u, rhs, cfg: MultigridConfig | None = None,
            counters: dict | None = None):
    """One V-cycle at `level`, in place on u (multigrid.py:335-371)."""
    cfg = cfg or hier.cfg
    _require_hot_path(cfg)
    plan, _, _ = _channel_plan(hier, cfg, 0)
    info = plan.level_info(level)
    u_arr = np.asarray(u)
    if u_arr.dtype != np.float64 or u_arr.shape != (info.height, info.width):
        raise ValueError(f"u must be a float64 field of shape {(info.height, info.width)}")
    d_u, d_b = _dev.to_device_f64(u_arr), _dev.to_device_f64(rhs)
    units = np.zeros(1, dtype=np.int32)
    _dev.call("b200p_plan_vcycle", plan.handle, int(level), _dev.ptr(d_u), _dev.ptr(d_b),
              units.ctypes.data, _dev.stream())
    u_arr[...] = _dev.to_host(d_u)
    if counters is not None and level == 0:
        counters["fine_units"] = counters.get("fine_units", 0) + int(units[0])
    return u


_STEP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int)


def _cg_solve_with_step_hook(problem: InpaintingProblem, cfg: MultigridConfig, channel: int, callback,
                             single_level: bool):
    """`cg` / `ml-cg` with `callback(u)` after every CG step of the finest level (solvers.py:171-174,
    multigrid.py:316-321, 449-464): the solve itself is the library's (same kernels and report as without a
    callback); `b200p_plan_set_step_callback` makes it check the step counters on the host after every update
    and call back with the device iterate, which is copied out here."""
    if not 0 <= channel < problem.channels:
        raise IndexError(f"channel {channel} out of range")
    h, w = problem.shape
    plan = cached_plan(w, h, 1, 1, cfg, problem.spacing, single_level=single_level)
    u = np.empty((h, w))
    raised = []

    def hook(_user, d_u, hh, ww):
        try:
            assert (hh, ww) == (h, w)
            _dev.call("b200p_memcpy_d2h", u.ctypes.data, d_u, u.nbytes)
            callback(u)
            return 0
        except BaseException as exc:  # noqa: BLE001 -- carried across the C frame and re-raised below
            raised.append(exc)
            return 1

    fn = _STEP_FN(hook)
    _dev.call("b200p_plan_set_step_callback", plan.handle, C.cast(fn, C.c_void_p), None)
    try:
        out, reports = plan.solve_host(problem.mask.view(np.uint8)[None], np.ascontiguousarray(problem.known[channel], dtype=np.float64)[None, None])
    except Exception:
        if raised:
            raise raised[0]
        raise
    finally:
        _dev.call("b200p_plan_set_step_callback", plan.handle, None, None)
    return out[0, 0], reports[0]


def _ml_oras_solve_stepwise(hier: LevelHierarchy, cfg: MultigridConfig, channel: int, callback):
    """fmg_solve in "multilevel" mode with the ORAS smoother and a `callback(u)` after every finest-level
    sweep (multigrid.py:449-464, on_fine_state): the levels below the finest ARE the multilevel solve of the
    level-1 problem (the hierarchy is recursive: multigrid.py:236-261), which runs on the fast path; its
    result is prolongated (multigrid.py:407-410) and the finest level is smoothed to tolerance one sweep at a
    time through `oras_sweeps(..., on_state=)` (_smooth_to_tol, multigrid.py:282-322)."""
    from .pipelines import solve_image
    from .solvers import BlockSolver, oras_sweeps
    t0 = time.perf_counter()
    s = cfg.solver
    levels = hier.levels
    fine = levels[0]
    b = fine.rhs[channel]
    baseline = float(np.linalg.norm(b - fine.op.apply(fine.flat_init(channel))))
    if len(levels) == 1:
        u = fine.flat_init(channel)
        tol, max_units, denom = min(cfg.coarse_tol, s.tol_rel), cfg.coarse_max_iters, 0.0
    else:
        below = levels[1]
        sub = InpaintingProblem(below.mask, below.rhs[channel], below.spacing)
        u = prolongate_solution(solve_image(sub, "ml-oras", cfg).fields[0], fine.mask, b)
        tol, max_units, denom = s.tol_rel, s.max_outer_iters, baseline
    if denom == 0.0:
        denom = float(np.linalg.norm(b - fine.op.apply(u)))
    history, units, rel = [], 0, 0.0
    if denom > 0.0:
        def on_state(uu, rn_now, sweeps_done):
            history.append(rn_now / denom)
            if sweeps_done > 0:
                callback(uu)

        blocks = BlockSolver(fine.mask, fine.spacing, fine.part, fine.weights, s.alpha)
        cap = s.local_max_iters or 4 * fine.part.block_h * fine.part.block_w
        units, rn = oras_sweeps(fine.op, blocks, b, u, max_sweeps=max_units, stop_norm=tol * denom,
                                eta=s.local_tol_fraction, local_max_iters=cap, on_state=on_state)
        rel = rn / denom
    return u, SolveReport(
        solver="ml-oras", iterations=units, final_rel_residual=rel, wall_time=time.perf_counter() - t0,
        history=history or [rel], converged=rel <= s.tol_rel, baseline_residual=baseline,
        init_residual=baseline, fine_smoother_iterations=units)


def _fmg_solve_stepwise(hier: LevelHierarchy, cfg: MultigridConfig, channel: int, callback):
    """fmg_solve with a per-cycle `callback(u)` (multigrid.py:466-481): the reference's own loop, driven from
    the host over the stage entry points (cascade, V-cycle, residual norm) instead of the one-graph solve,
    so that the iterate can be handed out after every cycle.  Same kernels, same cycle counts."""
    if cfg.mode == "multilevel" and cfg.smoother == "oras":
        return _ml_oras_solve_stepwise(hier, cfg, channel, callback)
    if cfg.mode == "multilevel":
        return _cg_solve_with_step_hook(hier.problem, cfg, channel, callback, single_level=False)
    t0 = time.perf_counter()
    p = hier.problem
    h, w = p.shape
    plan, d_mask, _ = _channel_plan(hier, cfg, channel)
    d_b = _dev.to_device_f64(np.where(p.mask, p.known[channel], 0.0))
    sq = np.zeros(1)

    def norm(d_u):
        _dev.call("b200p_residual_sqnorm", _dev.ptr(d_mask), h, w, float(p.spacing), _dev.ptr(d_b),
                  _dev.ptr(d_u), 1, sq.ctypes.data, _dev.stream())
        return float(np.sqrt(sq[0]))

    baseline = norm(d_b)                                    # flat initialisation = rhs (multigrid.py:446)
    d_u = _dev.empty_f64((h, w))
    _dev.call("b200p_plan_cascade", plan.handle, _dev.ptr(d_u), _dev.stream())
    rn = norm(d_u)
    denom = baseline if baseline > 0.0 else (rn if rn > 0.0 else 1.0)
    rel = rn / denom
    history, cycles, fine_units = [rel], 0, 0
    units = np.zeros(1, dtype=np.int32)
    while rel > cfg.solver.tol_rel and cycles < cfg.v_cycles_max:
        _dev.call("b200p_plan_vcycle", plan.handle, 0, _dev.ptr(d_u), _dev.ptr(d_b), units.ctypes.data,
                  _dev.stream())
        fine_units += int(units[0])
        cycles += 1
        rel = norm(d_u) / denom
        history.append(rel)
        callback(_dev.to_host(d_u))
    name = "mg-" + cfg.smoother
    return _dev.to_host(d_u), SolveReport(
        solver=name, iterations=cycles, final_rel_residual=rel, wall_time=time.perf_counter() - t0,
        history=history, converged=rel <= cfg.solver.tol_rel, baseline_residual=baseline,
        init_residual=baseline, fine_smoother_iterations=fine_units)


def fmg_solve(hier: LevelHierarchy, cfg: MultigridConfig | None = None, channel: int = 0, callback=None):
    """Full-multigrid solve of one channel (multigrid.py:425-487) -> (u, SolveReport)."""
    cfg = cfg or hier.cfg
    _require_hot_path(cfg)
    p = hier.problem
    if not p.mask.any():
        raise EmptyMaskError("cannot solve without known pixels")
    if callback is not None:
        return _fmg_solve_stepwise(hier, cfg, channel, callback)
    h, w = p.shape
    plan = cached_plan(w, h, 1, 1, cfg, p.spacing)
    d_known = hier._d_known[channel:channel + 1].contiguous()
    d_out, reps = plan.solve_device(hier._d_mask, d_known)
    return _dev.to_host(d_out)[0, 0], reps[0]
