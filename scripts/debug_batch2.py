import sys, numpy as np, torch, time
sys.path.insert(0, '.')
import oracle, paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
which = sys.argv[1] if len(sys.argv)>1 else 'all'
cases = {'256':(256,256,1,0.05,16,2),'512':(512,512,3,0.02,32,6),'1080':(1920,1080,3,0.04,16,2),'1080b':(1920,1080,3,0.02,32,6),'4k1':(3840,2160,1,0.02,32,6)}
for name,(W,H,C,d,bs,ov) in cases.items():
    if which!='all' and which!=name: continue
    cfg=bp.MultigridConfig(block_size=bs,overlap=ov)
    masks,known=synthetic.seeded_frames(W,H,d,1,C)
    ref,rr=oracle.solve_image(masks[0],known[0],1.0,oracle.MultigridConfig(block_size=bs,overlap=ov))
    for mode in ('host','device_zero','device_empty','device_knownmasked'):
        plan=bp.Plan(W,H,C,1,cfg)
        if mode=='host':
            out,reps=plan.solve_host(masks.view(np.uint8),known)
        else:
            dm=torch.from_numpy(masks.view(np.uint8)).cuda()
            kk = known if mode!='device_knownmasked' else np.where(masks[:,None],known,0.0)
            dk=torch.from_numpy(kk).cuda()
            do=torch.zeros_like(dk) if mode=='device_zero' else torch.full_like(dk, 1e6)
            torch.cuda.synchronize()
            do,reps=plan.solve_device(dm,dk,do)
            out=do.cpu().numpy()
        print(name,mode,'maxabs',np.abs(out[0]-ref).max(),[r.iterations for r in reps],['%.6e'%r.final_rel_residual for r in reps],['%.6e'%r.final_rel_residual for r in rr],flush=True)
        plan.close()
