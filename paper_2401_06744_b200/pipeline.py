"""Host-side frame pipeline: overlaps PCIe with compute for batches of frames.

Frames are independent problems, so a batch that arrives in HOST memory is cut
into chunks of `frames_per_lane` frames that rotate over `lanes` plans.  Each
lane owns a plan (its own CUDA stream, staging buffers and solve graph).  A
chunk is ENQUEUED with ``b200p_solve_host_async`` -- H2D of mask + known, the
whole FMG solve as one CUDA graph (the V-cycle loop is a WHILE node, so no host
round trip), D2H of the result -- and the call returns at once; the lane is
waited for (``b200p_solve_wait``) only when it is needed for the next chunk.
One host thread therefore keeps `lanes` chunks in flight and the copy engines
run under the kernels of the other lanes (PCIe is full duplex), which is what
the end-to-end frames/s of a decoder fed from host memory depends on.  Pass
pinned arrays: pageable memory makes the copies synchronous.
fp64 ingest of a multi-lane pipeline: the path reads `known` only at mask pixels, so
the library's host threads gather those values into a pinned (index, values) list
(``ingest="host-gather"``: 12 MB instead of 207 MB per 4K RGB frame on the link, which
leaves PCIe to the results; 227 -> 256 frames/s measured on 5 lanes).
Results do not depend on the chunking (bit-identical to a single batched plan)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _dev, _lib
from .multigrid import MultigridConfig, Plan


class FramePipeline:
    def __init__(self, width, height, channels, cfg: MultigridConfig | None = None, spacing=1.0,
                 lanes: int = 5, frames_per_lane: int = 1, sparse_ingest: bool | None = None,
                 ingest: str | None = None):
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
        # fp64 ingest.  "zero-copy": the device fetches the mask pixels' values from the pinned source itself --
        # lowest latency for one lane, but with several lanes those reads queue behind the other lanes' D2H
        # traffic (172 frames/s on 5 lanes); "dense": the copy engine moves the planes (227); "host-gather": host
        # threads compact the values, the copy engine moves 6 % of the bytes (256).  sparse_ingest = True / False
        # is the older spelling of "zero-copy" / "dense".
        if ingest is None:
            if sparse_ingest is None:
                ingest = "zero-copy" if lanes == 1 else "host-gather"
            else:
                ingest = "zero-copy" if sparse_ingest else "dense"
        if ingest not in ("zero-copy", "dense", "host-gather"):
            raise ValueError(f"ingest must be 'zero-copy', 'dense' or 'host-gather', got {ingest!r}")
        self.ingest = ingest
        for p in self.plans:
            p.set_ingest(dense=ingest == "dense", host_gather=ingest == "host-gather")
        self._inflight = [None] * lanes  # (job, chunk index) pending on each lane
        self._next = 0

    def close(self):
        self._drain_quietly()
        for p in self.plans:
            p.close()
        self.plans = []

    def _check(self, masks, known, out, image=False):
        c, h, w = self.shape
        if masks.dtype != np.uint8 and masks.dtype != np.bool_:
            raise ValueError("masks must be bool or uint8")
        mshape = (h, (w + 7) // 8) if image else (h, w)
        if masks.ndim != 3 or masks.shape[1:] != mshape:
            raise ValueError(f"masks must be (F,{mshape[0]},{mshape[1]}), got {masks.shape}")
        kshapes = [(masks.shape[0], h, w, c)] + ([(masks.shape[0], h, w)] if c == 1 else []) if image \
            else [(masks.shape[0], c, h, w)]
        if known.shape not in kshapes:
            raise ValueError(f"known must be {kshapes[0]}, got {known.shape}")
        for a, n in ((masks, "masks"), (known, "known"), (out, "out")):
            if a is not None and not a.flags.c_contiguous:
                raise ValueError(f"{n} must be C-contiguous")
        if masks.shape[0] % self.frames_per_lane:
            raise ValueError(f"frame count {masks.shape[0]} is not a multiple of frames_per_lane "
                             f"{self.frames_per_lane}")

    def submit(self, masks, known, out=None, u8: bool = False, image: bool = False):
        """Enqueue a batch: masks (F,H,W) bool/uint8, known (F,C,H,W) float64 (uint8 with u8=True).
        image=True takes the 8-bit file layouts: masks = P4 raster bits (F,H,ceil(W/8)) uint8, known = interleaved
        pixels (F,H,W,C) uint8; `out` then holds image_from_fields(...).pixels of every frame (Plan.solve_host_image_u8).

        Returns a job dict {"out", "reports", "h2d_bytes", "d2h_bytes"}; its arrays are complete after `flush()` (or once
        later submits have recycled all of its lanes).  Batches submitted back to back keep the
        lanes busy across batch boundaries: only `flush()` drains the pipeline.  `out` may be a
        preallocated (pinned) array of known's shape and dtype.  reports[f] is the list of
        per-channel SolveReports of frame f."""
        masks = np.asarray(masks)
        known = np.asarray(known)
        u8 = u8 or image
        want = np.uint8 if u8 else np.float64
        if known.dtype != want:
            raise ValueError(f"known must have dtype {np.dtype(want)}")
        if out is None:
            out = _dev.empty_host(known.shape, want)
        elif out.dtype != want or out.shape != known.shape:
            raise ValueError("out must match known's shape and dtype")
        self._check(masks, known, out, image=image)
        m8 = masks.view(np.uint8)
        k = self.frames_per_lane
        job = {"out": out, "reports": [None] * masks.shape[0], "h2d_bytes": 0, "d2h_bytes": 0}
        try:
            for i in range(masks.shape[0] // k):
                li = self._next % len(self.plans)
                self._next += 1
                self._retire(li)
                sl = slice(i * k, (i + 1) * k)
                self.plans[li].solve_host_async(m8[sl], known[sl], out[sl], u8=u8, image=image)
                self._inflight[li] = (job, i)
        except BaseException:
            self._drain_quietly()
            raise
        return job

    def _retire(self, li):
        ent = self._inflight[li]
        if ent is None:
            return
        self._inflight[li] = None
        job, i = ent
        reps = self.plans[li].wait()
        up, down = self.plans[li].last_transfer_bytes()
        job["h2d_bytes"] += up
        job["d2h_bytes"] += down
        k, c = self.frames_per_lane, self.shape[0]
        for j in range(k):
            job["reports"][i * k + j] = reps[j * c:(j + 1) * c]

    def _drain_quietly(self):
        for li in range(len(self.plans)):  # leave no solve pending on a plan
            try:
                self._retire(li)
            except Exception:
                pass

    def flush(self):
        """Wait for everything submitted so far."""
        try:
            for li in range(len(self.plans)):
                self._retire(li)
        except BaseException:
            self._drain_quietly()
            raise

    def run(self, masks, known, out=None, u8: bool = False, image: bool = False):
        """submit + flush: returns (out, reports)."""
        job = self.submit(masks, known, out, u8=u8, image=image)
        self.flush()
        return job["out"], job["reports"]
