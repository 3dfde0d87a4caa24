"""Probe: per-frame cost of the host f64 entry point, dense vs sparse ingest, one plan of one frame."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
W, H, C = 3840, 2160, 3
cfg = bp.MultigridConfig(block_size=32, overlap=6)
m, k = synthetic.seeded_frames(W, H, 0.02, 1, C)
hm = torch.from_numpy(m.view(np.uint8)).pin_memory(); hk = torch.from_numpy(k).pin_memory()
ho = torch.empty_like(hk).pin_memory()
plan = bp.Plan(W, H, C, 1, cfg)
dm, dk = hm.cuda(), hk.cuda(); do = torch.empty_like(dk)
def t(fn, n=8):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("device solve ms", t(lambda: plan.solve_device(dm, dk, do, want_reports=False)))
print("host sparse (pinned->mapped) ms", t(lambda: plan.solve_host(hm.numpy(), hk.numpy(), ho.numpy())))
def enq():
    t0 = time.perf_counter(); plan.solve_host_async(hm.numpy(), hk.numpy(), ho.numpy()); t1 = time.perf_counter(); plan.wait()
    return (t1 - t0) * 1e3
print("  enqueue call ms", [round(enq(), 2) for _ in range(4)])
pk = k.copy()
print("host sparse (pageable->gather) ms", t(lambda: plan.solve_host(hm.numpy(), pk, ho.numpy())))
os.environ["B200P_DENSE_INGEST"] = "1"
print("host dense ms", t(lambda: plan.solve_host(hm.numpy(), hk.numpy(), ho.numpy())))
print("  enqueue call ms", [round(enq(), 2) for _ in range(4)])
# raw copies
s = torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s): dk.copy_(hk, non_blocking=True)
    s.synchronize()
def d2h():
    with torch.cuda.stream(s): ho.copy_(dk, non_blocking=True)
    s.synchronize()
print("H2D 199MB ms", t(h2d), " D2H 199MB ms", t(d2h))
def both():
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s): dk.copy_(hk, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    s.synchronize(); s2.synchronize()
print("H2D+D2H concurrently ms", t(both))
