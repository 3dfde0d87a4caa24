"""Host-side cost of b200p_solve_host_async per frame (the call returns after enqueueing): plane copy vs host gather,
4K and 8K RGB 2 %.  B200P_HOST_THREADS from the environment."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
for (W, H) in ((3840, 2160), (7680, 4320)):
    masks, known = synthetic.seeded_frames(W, H, 0.02, 1, 3, first_seed=0)
    hm = torch.from_numpy(masks.view(np.uint8)).pin_memory(); hk = torch.from_numpy(known).pin_memory(); ho = torch.empty_like(hk).pin_memory()
    plan = bp.Plan(W, H, 3, 1, bp.MultigridConfig())
    for mode in ("dense", "host_gather"):
        plan.set_ingest(dense=mode == "dense", host_gather=mode == "host_gather")
        ts = []
        for i in range(5):
            t0 = time.perf_counter(); plan.solve_host_async(hm.numpy(), hk.numpy(), ho.numpy()); t1 = time.perf_counter(); plan.wait(); t2 = time.perf_counter()
            ts.append((t1 - t0, t2 - t0))
        print(f"{W}x{H} {mode:12s} threads={os.environ.get('B200P_HOST_THREADS','default')}: enqueue call {1e3*min(t[0] for t in ts[1:]):7.2f} ms, whole solve {1e3*min(t[1] for t in ts[1:]):7.2f} ms", flush=True)
    plan.close()
