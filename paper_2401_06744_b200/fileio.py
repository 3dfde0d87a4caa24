"""8-bit image side of the path: the conversions the reference runs around `solve_image`
in its `inpaint` command (cli.py:80-95) -- `ImageFile.channel_fields`, `image_from_fields`
(fileio.py:27-65) and the P4 mask raster of `read_mask` / `write_mask` (fileio.py:181-230).

The PNM codecs themselves (header parsing, file IO) are front-end code and stay with the reference;
what is mirrored here is the pixel arithmetic and the layouts, which the CUDA library consumes and
produces directly (`Plan.solve_host_image_u8`, `pipelines.inpaint_image_u8`)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev


@dataclass(frozen=True)
class ImageFile:
    """fileio.py:27-55: decoded 8-bit image, (h, w) grayscale or (h, w, 3) colour, uint8."""

    pixels: np.ndarray

    def __post_init__(self):
        p = self.pixels
        if p.dtype != np.uint8 or p.ndim not in (2, 3) or (p.ndim == 3 and p.shape[2] != 3):
            raise ValueError("pixels must be uint8 with shape (h, w) or (h, w, 3)")

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def channels(self) -> int:
        return 1 if self.pixels.ndim == 2 else 3

    def channel_fields(self) -> np.ndarray:
        """Float64 channel stack (channels, h, w) for the solvers (fileio.py:51-55)."""
        if self.pixels.ndim == 2:
            return self.pixels[None, :, :].astype(np.float64)
        return np.moveaxis(self.pixels, 2, 0).astype(np.float64)


def image_from_fields(fields) -> ImageFile:
    """Round (half to even) and clip solver output (channels, h, w) back to 8-bit, channels last
    (fileio.py:58-65) -- on the device, with the quantiser the solve's fused egress uses."""
    f = np.asarray(fields, dtype=np.float64)
    if f.ndim != 3:
        raise ValueError(f"expected (channels, h, w), got shape {f.shape}")
    c, h, w = f.shape
    if c not in (1, 3):
        raise ValueError(f"expected 1 or 3 channels, got {c}")
    d_f = _dev.to_device_f64(f)
    d_p = _dev.empty_u8((h, w, c))
    _dev.call("b200p_image_from_fields", _dev.ptr(d_f), 1, c, h, w, _dev.ptr(d_p), _dev.stream())
    px = _dev.to_host(d_p)
    return ImageFile(px[:, :, 0].copy() if c == 1 else px)


def pack_mask_raster(mask) -> np.ndarray:
    """The P4 raster write_mask emits (fileio.py:226): rows padded to whole bytes, MSB first, 1 = known."""
    m = np.asarray(mask, dtype=bool)
    if m.ndim != 2:
        raise ValueError(f"mask must be 2-D, got shape {m.shape}")
    return np.packbits(m.astype(np.uint8), axis=1)


def unpack_mask_raster(bits, width: int) -> np.ndarray:
    """read_mask's P4 branch (fileio.py:206-216) on the device: (h, ceil(w/8)) raster bytes -> bool (h, w)."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    if b.ndim != 2 or b.shape[1] != (int(width) + 7) // 8:
        raise ValueError(f"raster must be (h, {(int(width) + 7) // 8}), got {b.shape}")
    h = b.shape[0]
    d_b = _dev.to_device_u8(b)
    d_m = _dev.empty_u8((h, int(width)))
    _dev.call("b200p_unpack_mask_bits", _dev.ptr(d_b), 1, h, int(width), _dev.ptr(d_m), _dev.stream())
    return _dev.to_host(d_m).astype(bool)
