"""Overlapping-block geometry and partition-of-unity tables.

Same interface as the reference's ``diffpaint.partition`` (partition.py:38-168).
The tables come from libb200paint's host-side geometry code (the very code the
plan uploads to the GPU), so tests of this module pin what the kernels see.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class BlockRect:
    """One block: origin, extent, and which sides are cut (inner) sides."""

    x0: int
    y0: int
    w: int
    h: int
    inner_left: bool
    inner_right: bool
    inner_top: bool
    inner_bottom: bool


@dataclass(frozen=True)
class BlockPartition:
    width: int
    height: int
    block_size: int
    overlap: int
    xs: np.ndarray
    ys: np.ndarray
    block_w: int
    block_h: int

    @property
    def nx(self) -> int:
        return len(self.xs)

    @property
    def ny(self) -> int:
        return len(self.ys)

    @property
    def nblocks(self) -> int:
        return self.nx * self.ny

    def rect(self, i: int) -> BlockRect:
        if not 0 <= i < self.nblocks:
            raise IndexError(f"block index {i} out of range")
        iy, ix = divmod(i, self.nx)
        x0, y0 = int(self.xs[ix]), int(self.ys[iy])
        return BlockRect(x0, y0, self.block_w, self.block_h,
                         x0 > 0, x0 + self.block_w < self.width,
                         y0 > 0, y0 + self.block_h < self.height)

    def rects(self):
        return [self.rect(i) for i in range(self.nblocks)]


def _starts(dim: int, block: int, overlap: int) -> np.ndarray:
    L = _lib.lib()
    n = L.b200p_axis_starts(dim, block, overlap, None, 0)
    if n < 0:
        _lib.check(n)
    out = np.zeros(n, dtype=np.int64)
    L.b200p_axis_starts(dim, block, overlap, out.ctypes.data, n)
    return out


def build_partition(width: int, height: int, block_size: int = 32, overlap: int = 6) -> BlockPartition:
    """partition.py:93-116 -- clamped last block, single block when dim <= block."""
    if width < 1 or height < 1:
        raise ValueError(f"image dimensions must be >= 1, got {width}x{height}")
    if overlap < 0 or block_size <= overlap:
        raise ValueError(f"need block_size > overlap >= 0, got {block_size}, {overlap}")
    return BlockPartition(width, height, block_size, overlap,
                          _starts(width, block_size, overlap), _starts(height, block_size, overlap),
                          min(block_size, width), min(block_size, height))


@dataclass(frozen=True)
class BlockWeights:
    """Separable weights: wx (nx, block_w), wy (ny, block_h) (partition.py:119-134)."""

    wx: np.ndarray
    wy: np.ndarray

    def block(self, partition: BlockPartition, i: int) -> np.ndarray:
        iy, ix = divmod(i, partition.nx)
        return np.outer(self.wy[iy], self.wx[ix])


def _weights(dim: int, block: int, overlap: int, n: int) -> np.ndarray:
    bd = min(block, dim)
    out = np.empty((n, bd))
    got = _lib.lib().b200p_axis_weights(dim, block, overlap, out.ctypes.data, out.size)
    if got < 0:
        _lib.check(got)
    assert got == out.size
    return out


def build_weights(partition: BlockPartition) -> BlockWeights:
    """partition.py:157-168 -- linear ramps on inner sides, renormalised per pixel."""
    p = partition
    return BlockWeights(_weights(p.width, p.block_size, p.overlap, p.nx),
                        _weights(p.height, p.block_size, p.overlap, p.ny))


def _inside(field: np.ndarray, rect: BlockRect) -> tuple:
    h, w = field.shape
    if min(rect.x0, rect.y0) < 0 or rect.x0 + rect.w > w or rect.y0 + rect.h > h:
        raise ValueError(f"block {rect} exceeds field bounds {h}x{w}")
    return slice(rect.y0, rect.y0 + rect.h), slice(rect.x0, rect.x0 + rect.w)


def restrict_to_block(field: np.ndarray, rect: BlockRect) -> np.ndarray:
    """R_i u: a COPY of the block's sub-rectangle (partition.py:171-176); host-side helper, the kernels
    gather straight from the level field."""
    return np.array(field[_inside(field, rect)])


def extend_add_weighted(field: np.ndarray, rect: BlockRect, weights: np.ndarray, local: np.ndarray) -> None:
    """field += R_i^T (weights * local), in place (partition.py:179-188; same argument order)."""
    window = _inside(field, rect)
    if local.shape != (rect.h, rect.w) or weights.shape != (rect.h, rect.w):
        raise ValueError("local field / weights do not match the block extent")
    field[window] += weights * local
