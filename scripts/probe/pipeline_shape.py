"""End-to-end frames/s of FramePipeline for several (lanes, frames_per_lane) shapes, fp64 and 8-bit image I/O
(4K RGB 2 %, 16 frames per batch, pinned buffers).  Run on a B200: python scripts/probe/pipeline_shape.py"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic

W, H, C, F = 3840, 2160, 3, 16
cfg = bp.MultigridConfig()
masks, known = synthetic.seeded_frames(W, H, 0.02, F, C, first_seed=0)
hm = torch.from_numpy(masks.view(np.uint8)).pin_memory()
hk = torch.from_numpy(known).pin_memory()
ho = torch.empty_like(hk).pin_memory()
hb = torch.from_numpy(np.packbits(masks, axis=2)).pin_memory()
hp = torch.from_numpy(np.ascontiguousarray(np.moveaxis(known.astype(np.uint8), 1, 3))).pin_memory()
hq = torch.empty_like(hp).pin_memory()
import os
shapes = ((5, 1, False), (5, 1, True), (4, 2, True), (8, 1, True), (4, 4, True), (3, 1, True))
for lanes, fpl, hg in shapes:
    pipe = bp.FramePipeline(W, H, C, cfg, lanes=lanes, frames_per_lane=fpl, host_gather=hg)
    res = []
    for image in (False, True):
        a = (hb, hp, hq) if image else (hm, hk, ho)
        pipe.run(a[0].numpy(), a[1].numpy(), a[2].numpy(), image=image)
        t0 = time.perf_counter()
        for _ in range(4):
            pipe.submit(a[0].numpy(), a[1].numpy(), a[2].numpy(), image=image)
        pipe.flush()
        res.append(4 * F / (time.perf_counter() - t0))
    pipe.close()
    print(f"lanes {lanes} x {fpl} frames host_gather={hg} threads={os.environ.get('B200P_HOST_THREADS', 'default')}: fp64 {res[0]:6.1f} frames/s, 8-bit image {res[1]:6.1f} frames/s", flush=True)
