"""Device-memory handoff: torch CUDA tensors carry the buffers, nothing else.

PyTorch is plumbing here (allocation, streams, pinned host memory); all
arithmetic of the path happens inside libb200paint.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def require_cuda():
    if not torch.cuda.is_available() or _lib.lib().b200p_device_count() < 1:
        raise _lib.B200PaintError(
            "no CUDA device: paper_2401_06744_b200 has no CPU fallback (sm_100a kernels only)")


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr())


def call(name, *args):
    return _lib.check(getattr(_lib.lib(), name)(*args))


def to_device_f64(a) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to(device(), non_blocking=False)


def to_device_u8(a) -> torch.Tensor:
    a = np.asarray(a)
    if a.dtype != np.uint8:
        a = a.astype(bool).astype(np.uint8)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device())


def empty_f64(shape) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=torch.float64, device=device())


def empty_u8(shape) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=torch.uint8, device=device())


def empty_host(shape, dtype=np.float64) -> np.ndarray:
    """A fresh host array for results, backed by page-locked memory from torch's caching host allocator:
    the D2H copy runs at PCIe speed (a pageable target is staged and page-faults on first touch -- 55 ms
    for a 4K RGB float64 frame against 4 ms), and the block goes back to the cache when the caller drops
    the array.  The first result of a given size pays for the allocation."""
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8}[np.dtype(dtype)]
    try:
        return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()
    except RuntimeError:          # no pinned memory left: pageable still works
        return np.empty(tuple(shape), dtype=dtype)


def to_host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.current_stream().synchronize()
    return t.cpu().numpy()


def check_tensor(t, name: str, dtype: str, numel: int):
    """Device buffers cross the C-ABI as raw pointers: insist on the exact layout."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != getattr(torch, dtype):
        raise ValueError(f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous (row-major), got strides {tuple(t.stride())}")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
