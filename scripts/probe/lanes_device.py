"""Probe: device-resident frames/s with L concurrent plans of K frames each (own streams)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import _lib, _dev, synthetic
from paper_2401_06744_b200.multigrid import Plan, MultigridConfig

W, H, Cc = 3840, 2160, 3
cfg = MultigridConfig(block_size=32, overlap=6)
NF = 8
ms, ks = [], []
for f in range(NF):
    m, k = synthetic.seeded_problem(W, H, 0.02, f, channels=Cc)
    ms.append(m); ks.append(k)
d_mask = _dev.to_device_u8(np.stack(ms)); d_known = _dev.to_device_f64(np.stack(ks))
d_out = torch.empty_like(d_known)
L = _lib.lib()
for lanes, k in [(1, 8), (2, 4), (4, 2), (8, 1), (2, 8), (3, 8), (4, 4)]:
    plans = [Plan(W, H, Cc, k, cfg) for _ in range(lanes)]
    streams = [torch.cuda.Stream() for _ in range(lanes)]
    def go():
        for i, (p, s) in enumerate(zip(plans, streams)):
            o = (i * k) % NF
            _dev.call("b200p_solve_async", p.handle, _dev.ptr(d_mask[o:o + k]), _dev.ptr(d_known[o:o + k]),
                      _dev.ptr(d_out[o:o + k]), C.c_void_p(s.cuda_stream))
        for p in plans:
            _dev.call("b200p_solve_wait", p.handle, None)
    for _ in range(3): go()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R = 6
    for _ in range(R): go()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"lanes {lanes} x {k} frames: {R * lanes * k / dt:.1f} fps", flush=True)
    for p in plans: p.close()
