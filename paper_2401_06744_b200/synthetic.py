"""Synthetic benchmark inputs (host side, NumPy): the seeded random mask and
the smooth test image of the reference's benchmark recipe (masks.py:13-25,
:50-67; tests/conftest.py:7-12), drawn with the same Generator calls so that
the CPU baseline and the CUDA path see identical bits.  Not on the hot path."""

from __future__ import annotations

import numpy as np

NODE_PITCH = 24  # one random node every ~24 pixels


def random_mask(width: int, height: int, density: float, seed: int = 0) -> np.ndarray:
    """Exactly round(density * W * H) known pixels, drawn without replacement."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    total = width * height
    wanted = int(round(density * total))
    if wanted < 1:
        raise ValueError(f"density {density} selects zero pixels on {width}x{height}")
    flat = np.zeros(total, dtype=bool)
    flat[np.random.default_rng(seed).choice(total, size=wanted, replace=False)] = True
    return flat.reshape(height, width)


def _axis_cells(n_nodes: int, n_px: int):
    """Node cell index and fractional offset of every pixel along one axis."""
    pos = np.linspace(0.0, n_nodes - 1.0, n_px)
    cell = np.clip(pos.astype(int), 0, n_nodes - 2)
    return cell, pos - cell


def synthetic_image(width: int, height: int, seed: int = 0) -> np.ndarray:
    """U(0,255) nodes on a coarse lattice, bilinearly upsampled, rounded to integers."""
    gx = max(2, width // NODE_PITCH + 2)
    gy = max(2, height // NODE_PITCH + 2)
    nodes = np.random.default_rng(seed).uniform(0.0, 255.0, size=(gy, gx))
    cy, fy = _axis_cells(gy, height)
    cx, fx = _axis_cells(gx, width)
    upper, lower = nodes[cy], nodes[cy + 1]
    row_hi = upper[:, cx] * (1 - fx) + upper[:, cx + 1] * fx
    row_lo = lower[:, cx] * (1 - fx) + lower[:, cx + 1] * fx
    img = np.rint(row_hi * (1 - fy)[:, None] + row_lo * fy[:, None])
    return np.ascontiguousarray(img, dtype=np.float64)  # fancy indexing above yields F-ordered data


def step_edge_image(width: int, height: int, edge_x: int) -> np.ndarray:
    """0 left of column edge_x, 255 from edge_x on (masks.py:70-74)."""
    img = np.full((height, width), 255.0)
    img[:, :edge_x] = 0.0
    return img


def edge_concentrated_mask(width: int, height: int, edge_x: int, background_density: float = 0.01,
                           seed: int = 0) -> np.ndarray:
    """Sparse background samples plus the three full columns edge_x-2 .. edge_x (masks.py:77-89):
    the geometry in which plain 2x2 value averaging leaks across the edge."""
    mask = np.random.default_rng(seed).random((height, width)) < background_density
    mask[:, max(0, edge_x - 2):edge_x + 1] = True
    return mask


def seeded_problem(width: int, height: int, density: float, seed: int, channels: int = 1):
    """(mask (H,W) bool, known (C,H,W) float64): mask seed `seed`, channel c image seed+1000+c."""
    mask = random_mask(width, height, density, seed)
    known = np.stack([synthetic_image(width, height, seed + 1000 + c) for c in range(channels)])
    return mask, known


def seeded_frames(width: int, height: int, density: float, frames: int, channels: int = 3,
                  first_seed: int = 0):
    """Batch of independent frames: frame f uses seed first_seed + f."""
    ms, ks = zip(*(seeded_problem(width, height, density, first_seed + f, channels)
                   for f in range(frames)))
    return np.stack(ms), np.stack(ks)
