import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic, _lib, _dev
W,H,Cn,d,bs,ov=256,256,1,0.05,16,2
cfg=bp.MultigridConfig(block_size=bs,overlap=ov)
masks,known=synthetic.seeded_frames(W,H,d,1,Cn)
print(masks.dtype, masks.shape, masks.flags['C_CONTIGUOUS'], known.dtype, known.shape, known.flags['C_CONTIGUOUS'], known.strides)
ocfg=oracle.MultigridConfig(block_size=bs,overlap=ov)
ho=oracle.build_hierarchy(masks[0],known[0],1.0,ocfg)
plan=bp.Plan(W,H,Cn,1,cfg,use_graphs=False)
dm=torch.from_numpy(masks.view(np.uint8)).cuda(); dk=torch.from_numpy(known).cuda()
print('ptrs',hex(dm.data_ptr()),hex(dk.data_ptr()), 'roundtrip', np.array_equal(dm.cpu().numpy(),masks.view(np.uint8)), np.array_equal(dk.cpu().numpy(),known))
L=_lib.lib()
_dev.call("b200p_plan_build_hierarchy", plan.handle, _dev.ptr(dm), _dev.ptr(dk), _dev.stream())
torch.cuda.synchronize()
for l in range(1,plan.num_levels):
    info=plan.level_info(l); pm,pr=C.c_void_p(),C.c_void_p()
    L.b200p_plan_level_ptrs(plan.handle,l,C.byref(pm),C.byref(pr))
    m=np.empty((info.height,info.width),np.uint8); r=np.empty((Cn,info.height,info.width))
    L.b200p_memcpy_d2h(m.ctypes.data,pm,m.nbytes); L.b200p_memcpy_d2h(r.ctypes.data,pr,r.nbytes)
    print('level',l,'mask eq',np.array_equal(m.astype(bool),ho.levels[l].mask),'rhs maxabs',np.abs(r-ho.levels[l].rhs).max())
du=torch.zeros_like(dk)
_dev.call("b200p_plan_cascade", plan.handle, _dev.ptr(du), _dev.stream())
torch.cuda.synchronize()
print('cascade maxabs', np.abs(du.cpu().numpy()[0,0]-oracle.cascadic_init(ho,ocfg,0)).max())
# baseline norm
b=np.where(masks[0],known[0,0],0.0)
r=oracle.residual(masks[0],1.0,b,b); print('oracle baseline',np.sqrt(np.vdot(r,r)))
do,reps=plan.solve_device(dm,dk); print('solve baseline',reps[0].baseline_residual, reps[0].history, 'ref hist', oracle.solve_image(masks[0],known[0],1.0,ocfg)[1][0].history)
