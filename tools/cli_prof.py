import time, os, sys, json, tempfile
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2403_10706_b200 import hysco as H
from synth import phantom
shape, h, seed = phantom.CONFIGS["C2_hcp3t"]
p = phantom.make_pair(shape, h, seed)
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
st = torch.cuda.current_stream(dev)
Ip = torch.from_numpy(p.Ip[None]).to(dev); Im = torch.from_numpy(p.Im[None]).to(dev)
for rep in range(4):
    T = {}
    t = time.perf_counter(); ctx = H.hysco_create(shape, h, 1, stream=st.cuda_stream); torch.cuda.synchronize(); T['create'] = time.perf_counter() - t
    H.hysco_bind_images(ctx, Ip, Im)
    b = torch.zeros((1, shape[0], shape[1], shape[2] + 1), device=dev); o1 = torch.zeros_like(Ip); o2 = torch.zeros_like(Ip)
    torch.cuda.synchronize()
    t = time.perf_counter(); r, _ = H.hysco_correct(ctx, b, o1, o2, H.default_ot_opts(), H.default_solve_opts(fixed_iters=0)); T['correct1'] = time.perf_counter() - t
    t = time.perf_counter(); r, _ = H.hysco_correct(ctx, b, o1, o2, H.default_ot_opts(), H.default_solve_opts(fixed_iters=0)); T['correct2'] = time.perf_counter() - t
    t = time.perf_counter(); H.hysco_destroy(ctx); torch.cuda.synchronize(); T['destroy'] = time.perf_counter() - t
    print(rep, {k: round(v * 1e3, 2) for k, v in T.items()}, r[0]['gn_iters'], r[0]['stop_reason'], flush=True)
