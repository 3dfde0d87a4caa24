"""Probe: end-to-end frames/s of FramePipeline over (lanes, frames_per_lane), f64 and u8 host buffers."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
W, H, C, F = 3840, 2160, 3, 8
cfg = bp.MultigridConfig(block_size=32, overlap=6)
m, k = synthetic.seeded_frames(W, H, 0.02, F, C)
hm = torch.from_numpy(m.view(np.uint8)).pin_memory(); hk = torch.from_numpy(k).pin_memory()
ho = torch.empty_like(hk).pin_memory()
hk8 = torch.from_numpy(k.astype(np.uint8)).pin_memory(); ho8 = torch.empty_like(hk8).pin_memory()
for lanes, fpl in [(5, 1), (3, 2), (4, 2), (6, 1), (8, 1), (2, 4), (3, 4)]:
    pipe = bp.FramePipeline(W, H, C, cfg, lanes=lanes, frames_per_lane=fpl)
    res = []
    for u8, a, o in ((False, hk, ho), (True, hk8, ho8)):
        pipe.run(hm.numpy(), a.numpy(), o.numpy(), u8=u8)
        t0 = time.perf_counter(); R = 6
        for _ in range(R): pipe.submit(hm.numpy(), a.numpy(), o.numpy(), u8=u8)
        pipe.flush(); res.append(R * F / (time.perf_counter() - t0))
    print(f"lanes {lanes} x {fpl}: f64 {res[0]:.1f} fps, u8 {res[1]:.1f} fps", flush=True)
    pipe.close()
