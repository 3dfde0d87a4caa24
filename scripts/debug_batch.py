import sys, numpy as np, torch, time
sys.path.insert(0, '.')
import oracle, paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic
W,H,C,d,bs,ov = 3840,2160,3,0.02,32,6
if len(sys.argv)>1 and sys.argv[1]=='small': W,H=1920,1080
cfg=bp.MultigridConfig(block_size=bs,overlap=ov)
refs={}
for F in (1,2,4):
    masks,known=synthetic.seeded_frames(W,H,d,F,C)
    for mode in ('host','device','device_stream'):
        plan=bp.Plan(W,H,C,F,cfg)
        if mode=='host':
            out,reps=plan.solve_host(masks.view(np.uint8),known)
        else:
            dm=torch.from_numpy(masks.view(np.uint8)).cuda(); dk=torch.from_numpy(known).cuda()
            if mode=='device':
                do,reps=plan.solve_device(dm,dk)
            else:
                s=torch.cuda.Stream()
                with torch.cuda.stream(s):
                    do,reps=plan.solve_device(dm,dk)
                    do,reps=plan.solve_device(dm,dk,do)
                    torch.cuda.synchronize()
            out=do.cpu().numpy()
        for f in range(F):
            if f not in refs:
                refs[f]=oracle.solve_image(masks[f],known[f],1.0,oracle.MultigridConfig(block_size=bs,overlap=ov))
            ref,rr=refs[f]
            print(F,mode,f,'maxabs',np.abs(out[f]-ref).max(),[r.iterations for r in reps[f*C:(f+1)*C]],[ '%.6e'%r.final_rel_residual for r in reps[f*C:(f+1)*C]], ['%.6e'%r.final_rel_residual for r in rr], flush=True)
        plan.close()
