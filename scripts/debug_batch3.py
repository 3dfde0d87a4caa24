import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic, _lib
W,H,Cn,d,bs,ov=256,256,1,0.05,16,2
cfg=bp.MultigridConfig(block_size=bs,overlap=ov)
masks,known=synthetic.seeded_frames(W,H,d,1,Cn)
ref,rr=oracle.solve_image(masks[0],known[0],1.0,oracle.MultigridConfig(block_size=bs,overlap=ov))
def rep(tag,out,reps): print(tag,'maxabs',np.abs(out-ref).max(),[r.iterations for r in reps],flush=True)
for graphs in (True,False):
    plan=bp.Plan(W,H,Cn,1,cfg,use_graphs=graphs)
    dm=torch.from_numpy(masks.view(np.uint8)).cuda(); dk=torch.from_numpy(known).cuda()
    do,reps=plan.solve_device(dm,dk); rep(f'device graphs={graphs}',do.cpu().numpy()[0],reps)
    plan.close()
# device mode with library-malloc'd buffers
L=_lib.lib()
plan=bp.Plan(W,H,Cn,1,cfg)
pm,pk,po=C.c_void_p(),C.c_void_p(),C.c_void_p()
n=W*H
L.b200p_malloc(C.byref(pm),n); L.b200p_malloc(C.byref(pk),8*n*Cn); L.b200p_malloc(C.byref(po),8*n*Cn)
mk=np.ascontiguousarray(masks.view(np.uint8)); kk=np.ascontiguousarray(known)
L.b200p_memcpy_h2d(pm,mk.ctypes.data,n); L.b200p_memcpy_h2d(pk,kk.ctypes.data,8*n*Cn)
raw=(_lib.Report*Cn)()
rc=L.b200p_solve(plan.handle,pm,pk,po,C.cast(raw,C.c_void_p),None); print('rc',rc)
out=np.empty((Cn,H,W)); L.b200p_memcpy_d2h(out.ctypes.data,po,8*n*Cn)
print('libmalloc device maxabs',np.abs(out-ref).max(), raw[0].iterations)
# host mode, second call on same plan
o2,r2=plan.solve_host(mk,kk); rep('host after device on same plan',o2[0],r2)
plan.close()
plan=bp.Plan(W,H,Cn,1,cfg)
o2,r2=plan.solve_host(mk,kk); rep('host fresh',o2[0],r2)
dm=torch.from_numpy(masks.view(np.uint8)).cuda(); dk=torch.from_numpy(known).cuda()
do,reps=plan.solve_device(dm,dk); rep('device after host same plan',do.cpu().numpy()[0],reps)
