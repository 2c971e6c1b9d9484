import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2403_10706_b200 import hysco as H
from synth import phantom
p = phantom.make_config("C2_hcp3t")
n1, n2, n3 = p.Ip.shape
Ip, Im = torch.from_numpy(p.Ip[None]).cuda(), torch.from_numpy(p.Im[None]).cuda()
ctx = H.hysco_create((n1, n2, n3), p.h, 1, stream=torch.cuda.current_stream().cuda_stream)
H.hysco_bind_images(ctx, Ip, Im)
b = torch.zeros((1, n1, n2, n3 + 1), device="cuda"); Tp = torch.zeros((1, n1, n2, n3), device="cuda"); Tm = torch.zeros_like(Tp)
torch.cuda.synchronize()
for _ in range(8):
    H.hysco_correct(ctx, b, Tp, Tm)
for rep in range(3):
    try:
        print(H.hysco_profile_kernels(ctx, 20, flush_l2=True), flush=True)
    except Exception as e:
        print("FAIL", e, flush=True)
        break
