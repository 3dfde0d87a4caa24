import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
W,H,C,d=3840,2160,3,0.02
cfg=bp.MultigridConfig()
for F in (1,2,4):
    masks,known=synthetic.seeded_frames(W,H,d,F,C)
    hm=torch.from_numpy(masks.view(np.uint8)).pin_memory(); hk=torch.from_numpy(known).pin_memory(); ho=torch.empty_like(hk).pin_memory()
    dk=torch.empty_like(hk,device='cuda')
    torch.cuda.synchronize()
    t=time.perf_counter(); 
    for _ in range(3): dk.copy_(hk,non_blocking=True)
    torch.cuda.synchronize(); h2d=(time.perf_counter()-t)/3
    t=time.perf_counter()
    for _ in range(3): ho.copy_(dk,non_blocking=True)
    torch.cuda.synchronize(); d2h=(time.perf_counter()-t)/3
    plan=bp.Plan(W,H,C,F,cfg)
    for _ in range(2): plan.solve_host(hm.numpy(),hk.numpy(),ho.numpy())
    t=time.perf_counter()
    for _ in range(3): plan.solve_host(hm.numpy(),hk.numpy(),ho.numpy())
    e2e=(time.perf_counter()-t)/3
    dm=hm.cuda(); do=torch.empty_like(dk)
    for _ in range(2): plan.solve_device(dm,dk,do)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(3): plan.solve_device(dm,dk,do,want_reports=False)
    torch.cuda.synchronize(); dev=(time.perf_counter()-t)/3
    t=time.perf_counter(); 
    for _ in range(3): masks.any(axis=(1,2))
    chk=(time.perf_counter()-t)/3
    print(f"F={F}: h2d {h2d*1e3:.1f} ms ({hk.numel()*8/h2d/1e9:.1f} GB/s)  d2h {d2h*1e3:.1f} ms ({hk.numel()*8/d2h/1e9:.1f} GB/s)  solve_device {dev*1e3:.1f} ms  solve_host {e2e*1e3:.1f} ms  numpy mask check {chk*1e3:.1f} ms", flush=True)
    plan.close()
