"""Device-resident throughput: one batched plan vs N concurrent single-frame plans on their own streams."""
import sys, time, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic, _dev, _lib

W, H, Cc, dens = 3840, 2160, 3, 0.02
F = 4
cfg = bp.MultigridConfig()
masks, known = synthetic.seeded_frames(W, H, dens, F, Cc, first_seed=0)
d_mask = torch.from_numpy(masks.view(np.uint8)).cuda(); d_known = torch.from_numpy(known).cuda(); d_out = torch.empty_like(d_known)
for fpl in (4, 2, 1):
    n = F // fpl
    plans = [bp.Plan(W, H, Cc, fpl, cfg) for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    def step():
        for i, (p, s) in enumerate(zip(plans, streams)):
            sl = slice(i * fpl, (i + 1) * fpl)
            _dev.call("b200p_solve_async", p.handle, _dev.ptr(d_mask[sl]), _dev.ptr(d_known[sl]), _dev.ptr(d_out[sl]), s.cuda_stream)
        for p in plans:
            _dev.call("b200p_solve_wait", p.handle, None)
    for _ in range(3): step()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    K = 10
    for _ in range(K): step()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{n} plan(s) x {fpl} frame(s): {F*K/dt:.1f} fps")
    for p in plans: p.close()
