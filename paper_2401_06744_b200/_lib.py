"""ctypes binding of ``libb200paint.so`` (include/b200paint.h).

The library is the product: there is no Python/NumPy/CPU fallback.  Importing
this module without the built library raises, and every compute entry point
fails with the CUDA error when no device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B200P_LIB") or os.path.join(_HERE, "libb200paint.so")  # override: A/B builds
CSRC = os.path.join(_HERE, "csrc")

MAX_LEVELS = 32
MAX_HISTORY = 128
MAX_BLOCK = 64

ERR_ARG, ERR_EMPTY_MASK, ERR_UNSUPPORTED, ERR_STATE = -1, -2, -3, -4


class Config(C.Structure):
    """b200p_config"""

    _fields_ = [
        ("width", C.c_int), ("height", C.c_int), ("channels", C.c_int), ("frames", C.c_int),
        ("spacing", C.c_double),
        ("block_size", C.c_int), ("overlap", C.c_int),
        ("nu_pre", C.c_int), ("nu_post", C.c_int), ("v_cycles_max", C.c_int),
        ("value_downsampling", C.c_int),
        ("coarse_tol", C.c_double), ("coarse_max_iters", C.c_int),
        ("tol_rel", C.c_double), ("alpha", C.c_double), ("eta", C.c_double),
        ("local_max_iters", C.c_int), ("use_graphs", C.c_int),
        ("mode", C.c_int), ("max_outer_iters", C.c_int),
        ("smoother", C.c_int), ("smoother_cg_iters", C.c_int),
    ]


class Report(C.Structure):
    """b200p_report"""

    _fields_ = [
        ("iterations", C.c_int), ("converged", C.c_int),
        ("fine_smoother_iterations", C.c_int), ("history_len", C.c_int),
        ("final_rel_residual", C.c_double), ("baseline_residual", C.c_double),
        ("init_residual", C.c_double),
        ("history", C.c_double * MAX_HISTORY),
    ]


class LevelInfo(C.Structure):
    """b200p_level_info"""

    _fields_ = [
        ("height", C.c_int), ("width", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("block_w", C.c_int), ("block_h", C.c_int),
        ("spacing", C.c_double),
    ]


class B200PaintError(RuntimeError):
    """A CUDA runtime error reported by libb200paint."""


def build(force: bool = False) -> str:
    """Compile libb200paint.so for sm_100a with the committed Makefile."""
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(_HERE, "..", "include", "b200paint.h")]
    stale = (not os.path.exists(LIB_PATH)
             or os.path.getmtime(LIB_PATH) < max(os.path.getmtime(s) for s in srcs))
    if force or stale:
        r = subprocess.run(["make", "-C", CSRC] + (["-B"] if force else []),
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("building libb200paint.so failed:\n" + r.stdout + r.stderr)
    return LIB_PATH


_lib = None

_VP, _I, _D, _I64 = C.c_void_p, C.c_int, C.c_double, C.c_int64

# name -> (restype, argtypes); every symbol include/b200paint.h declares
SIGNATURES = {
    "b200p_last_error": (C.c_char_p, []),
    "b200p_device_count": (_I, []),
    "b200p_set_device": (_I, [_I]),
    "b200p_get_device": (_I, [C.POINTER(_I)]),
    "b200p_config_default": (None, [C.POINTER(Config), _I, _I, _I]),
    "b200p_axis_starts": (_I, [_I, _I, _I, _VP, _I]),
    "b200p_axis_weights": (_I, [_I, _I, _I, _VP, _I]),
    "b200p_level_shapes": (_I, [_I, _I, _D, _I, _I, C.POINTER(LevelInfo), _I]),
    "b200p_plan_create": (_I, [C.POINTER(Config), C.POINTER(_VP)]),
    "b200p_plan_destroy": (None, [_VP]),
    "b200p_plan_num_levels": (_I, [_VP]),
    "b200p_plan_level_info": (_I, [_VP, _I, C.POINTER(LevelInfo)]),
    "b200p_plan_set_strip_nccl": (_I, [_VP, _I, _VP, _I, _I, _VP]),
    "b200p_nccl_unique_id": (_I, [_VP]),
    "b200p_nccl_comm_create": (_I, [_VP, _I, _I, C.POINTER(_VP)]),
    "b200p_nccl_comm_destroy": (_I, [_VP]),
    "b200p_strip_halo_plan": (_I, [_VP, _I, _I, _I, _I, _VP, _VP, _I]),
    "b200p_plan_strip_ranges": (_I, [_VP, _I, _I, _I, _VP]),
    "b200p_strip_ranges": (_I, [_I, _I, _I, _I, _I, _I, _VP]),
    "b200p_plan_set_strip": (_I, [_VP, _I, _VP, _VP, _VP]),
    "b200p_plan_set_step_callback": (_I, [_VP, _VP, _VP]),
    "b200p_plan_history": (_I, [_VP, _I, _VP, _I]),
    "b200p_plan_level_rc": (_I, [_VP, _I, C.POINTER(_VP)]),
    "b200p_plan_device_bytes": (_I64, [_VP]),
    "b200p_plan_launch_count": (_I64, [_VP]),
    "b200p_plan_set_ingest": (_I, [_VP, _I]),
    "b200p_plan_last_transfer_bytes": (_I, [_VP, C.POINTER(_I64), C.POINTER(_I64)]),
    "b200p_plan_profile": (_I, [_VP, _I]),
    "b200p_plan_profile_kinds": (_I, []),
    "b200p_plan_profile_name": (C.c_char_p, [_I]),
    "b200p_plan_profile_get": (_I, [_VP, _I, C.POINTER(_D), C.POINTER(_I64), C.POINTER(_D)]),
    "b200p_solve": (_I, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "b200p_solve_async": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "b200p_solve_wait": (_I, [_VP, _VP]),
    "b200p_solve_host": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "b200p_solve_host_async": (_I, [_VP, _VP, _VP, _VP]),
    "b200p_solve_host_u8_async": (_I, [_VP, _VP, _VP, _VP]),
    "b200p_solve_host_u8": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "b200p_solve_host_image_u8_async": (_I, [_VP, _VP, _VP, _VP]),
    "b200p_solve_host_image_u8": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "b200p_plan_build_hierarchy": (_I, [_VP, _VP, _VP, _VP]),
    "b200p_plan_level_ptrs": (_I, [_VP, _I, C.POINTER(_VP), C.POINTER(_VP)]),
    "b200p_plan_cascade": (_I, [_VP, _VP, _VP]),
    "b200p_plan_vcycle": (_I, [_VP, _I, _VP, _VP, _VP, _VP]),
    "b200p_plan_oras_sweeps": (_I, [_VP, _I, _VP, _VP, _I, _D, _I, _VP, _VP, _VP]),
    "b200p_plan_scatter_weighted": (_I, [_VP, _I, _VP, _VP, _VP]),
    "b200p_plan_solve_blocks": (_I, [_VP, _I, _VP, _D, _VP, _VP]),
    "b200p_apply": (_I, [_VP, _I, _I, _D, _VP, _VP, _VP]),
    "b200p_residual": (_I, [_VP, _I, _I, _D, _VP, _VP, _VP, _VP]),
    "b200p_residual_sqnorm": (_I, [_VP, _I, _I, _D, _VP, _VP, _I, _VP, _VP]),
    "b200p_downsample_mask": (_I, [_VP, _I, _I, _VP, _VP]),
    "b200p_image_from_fields": (_I, [_VP, _I, _I, _I, _I, _VP, _VP]),
    "b200p_unpack_mask_bits": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "b200p_downsample_values": (_I, [_VP, _VP, _VP, _I, _I, _I, _VP, _VP]),
    "b200p_residual_restrict": (_I, [_VP, _VP, _I, _I, _D, _VP, _VP, _VP, _VP]),
    "b200p_restrict_residual": (_I, [_VP, _VP, _I, _I, _VP, _VP]),
    "b200p_prolongate_correct": (_I, [_VP, _VP, _I, _I, _VP, _VP]),
    "b200p_prolongate_solution": (_I, [_VP, _VP, _VP, _I, _I, _VP, _VP]),
    "b200p_malloc": (_I, [C.POINTER(_VP), _I64]),
    "b200p_free": (_I, [_VP]),
    "b200p_ipc_export": (_I, [_VP, _VP]),
    "b200p_ipc_open": (_I, [_VP, C.POINTER(_VP)]),
    "b200p_ipc_close": (_I, [_VP]),
    "b200p_memcpy_d2d_async": (_I, [_VP, _VP, _I64, _VP]),
    "b200p_memcpy_h2d": (_I, [_VP, _VP, _I64]),
    "b200p_memcpy_d2h": (_I, [_VP, _VP, _I64]),
    "b200p_memset": (_I, [_VP, _I, _I64]),
    "b200p_device_synchronize": (_I, []),
    "b200p_abi_version": (_I, []),
    "b200p_has_experiments": (_I, []),
}
ABI_VERSION = 2  # B200P_ABI_VERSION these bindings (struct layouts above) were written for


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        got = L.b200p_abi_version() if hasattr(L, "b200p_abi_version") else 1
        if got != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI version {got}, these bindings need {ABI_VERSION}: rebuild it "
                              "(`make -C paper_2401_06744_b200/csrc`)")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().b200p_last_error().decode("utf-8", "replace")


def check(rc: int) -> int:
    """Map a C-ABI status to the reference's exception types."""
    if rc == 0:
        return 0
    msg = last_error()
    if rc == ERR_EMPTY_MASK:
        from .core import EmptyMaskError
        raise EmptyMaskError(msg)
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == ERR_STATE:
        raise RuntimeError(msg)
    raise B200PaintError(f"CUDA error {rc}: {msg}")
