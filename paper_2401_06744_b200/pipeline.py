"""Host-side frame pipeline: overlaps PCIe with compute for batches of frames.

Frames are independent problems, so a batch that arrives in HOST memory is cut
into chunks of `frames_per_lane` frames and fed to `lanes` worker threads.  Each
lane owns a plan (its own CUDA stream, staging buffers and graphs) and runs
``b200p_solve_host`` on its chunk: H2D, solve, D2H.  With two or more lanes the
copies of one chunk overlap the kernels of another (PCIe is full duplex), which
is what the end-to-end frames/s of a decoder fed from host memory depends on.
Results do not depend on the chunking (bit-identical to a single batched plan).

ctypes releases the GIL during the C call, so plain threads suffice."""

from __future__ import annotations

import ctypes as C
import queue
import threading

import numpy as np

from . import _dev, _lib
from .multigrid import MultigridConfig, Plan


class FramePipeline:
    def __init__(self, width, height, channels, cfg: MultigridConfig | None = None, spacing=1.0,
                 lanes: int = 3, frames_per_lane: int = 1):
        if lanes < 1 or frames_per_lane < 1:
            raise ValueError("need lanes >= 1 and frames_per_lane >= 1")
        _dev.require_cuda()
        self.cfg = cfg or MultigridConfig()
        self.shape = (int(channels), int(height), int(width))
        self.frames_per_lane = int(frames_per_lane)
        dev = C.c_int(0)
        _lib.check(_lib.lib().b200p_get_device(C.byref(dev)))
        self.device = dev.value
        self.plans = [Plan(width, height, channels, frames_per_lane, self.cfg, spacing) for _ in range(lanes)]

    def close(self):
        for p in self.plans:
            p.close()
        self.plans = []

    def _check(self, masks, known, out):
        c, h, w = self.shape
        if masks.dtype != np.uint8 and masks.dtype != np.bool_:
            raise ValueError("masks must be bool or uint8")
        if masks.ndim != 3 or masks.shape[1:] != (h, w):
            raise ValueError(f"masks must be (F,{h},{w}), got {masks.shape}")
        if known.shape != (masks.shape[0], c, h, w):
            raise ValueError(f"known must be (F,{c},{h},{w}), got {known.shape}")
        for a, n in ((masks, "masks"), (known, "known"), (out, "out")):
            if a is not None and not a.flags.c_contiguous:
                raise ValueError(f"{n} must be C-contiguous")
        if masks.shape[0] % self.frames_per_lane:
            raise ValueError(f"frame count {masks.shape[0]} is not a multiple of frames_per_lane "
                             f"{self.frames_per_lane}")

    def run(self, masks, known, out=None, u8: bool = False):
        """masks (F,H,W) bool/uint8, known (F,C,H,W) float64 (or uint8 with u8=True) -> (out, reports).

        `out` may be a preallocated (pinned) array of known's shape and dtype.  reports[f] is the
        list of per-channel SolveReports of frame f."""
        masks = np.asarray(masks)
        known = np.asarray(known)
        want = np.uint8 if u8 else np.float64
        if known.dtype != want:
            raise ValueError(f"known must have dtype {np.dtype(want)}")
        if out is None:
            out = np.empty(known.shape, dtype=want)
        elif out.dtype != want or out.shape != known.shape:
            raise ValueError("out must match known's shape and dtype")
        self._check(masks, known, out)
        m8 = masks.view(np.uint8)
        k = self.frames_per_lane
        nchunks = masks.shape[0] // k
        work: queue.SimpleQueue = queue.SimpleQueue()
        for i in range(nchunks):
            work.put(i)
        reports = [None] * masks.shape[0]
        errors = []

        def lane(plan):
            try:
                _lib.check(_lib.lib().b200p_set_device(self.device))
                while True:
                    try:
                        i = work.get_nowait()
                    except queue.Empty:
                        return
                    sl = slice(i * k, (i + 1) * k)
                    fn = plan.solve_host_u8 if u8 else plan.solve_host
                    _, reps = fn(m8[sl], known[sl], out[sl])
                    c = self.shape[0]
                    for j in range(k):
                        reports[i * k + j] = reps[j * c:(j + 1) * c]
            except BaseException as e:  # surfaced in the caller's thread
                errors.append(e)

        threads = [threading.Thread(target=lane, args=(p,), daemon=True) for p in self.plans[:nchunks]]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out, reports
