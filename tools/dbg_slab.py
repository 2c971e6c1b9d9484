import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2403_10706_b200 import hysco as H
from synth import phantom
p=phantom.make_config("C1_16x16x8")
n1,n2,n3=p.Ip.shape
for nr in (1,2):
    ctxs=H.hysco_create_loopback((n1,n2,n3),p.h,nr)
    keep=[]; bs=[]
    for r,c in enumerate(ctxs):
        i0,i1=H.slab_bounds(n1,nr,r)
        a=torch.from_numpy(np.ascontiguousarray(p.Ip[None,i0:i1])).cuda(); b=torch.from_numpy(np.ascontiguousarray(p.Im[None,i0:i1])).cuda(); keep+=[a,b]
        H.hysco_bind_images(c,a,b); bs.append(torch.zeros((1,i1-i0,n2,n3+1),device='cuda'))
    for mg in (0,1):
        reps,_=H.hysco_group_correct(ctxs,bs,solve_opts=H.default_solve_opts(max_gn=mg,armijo=0))
        print(nr, mg, reps[0], float(bs[0].abs().max()), H.hysco_last_launch_count(ctxs[0]))
