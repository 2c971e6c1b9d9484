"""Time ADMM (fixed 33 iterations, fp32, HCP 3T pair) single-context vs a
loopback slab group of N contexts on one GPU (transposed z-update); the OT
start comes from the single context.  CUDA events on the group's stream."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_10706_b200 import hysco as H  # noqa: E402
from synth import phantom                      # noqa: E402

p = phantom.make_config("C2_hcp3t")
n1, n2, n3 = p.Ip.shape
Ip, Im = torch.from_numpy(p.Ip[None]).cuda(), torch.from_numpy(p.Im[None]).cuda()
ao = H.default_admm_opts(max_iter=33, fixed_iters=1)
ctx = H.hysco_create((n1, n2, n3), p.h, 1)
H.hysco_bind_images(ctx, Ip, Im)
b0 = torch.zeros((1, n1, n2, n3 + 1), device="cuda")
torch.cuda.synchronize()
H.hysco_ot_init(ctx, b0)
torch.cuda.synchronize()
out = {}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        z.record()
        z.synchronize()
        ts.append(a.elapsed_time(z))
    return float(np.median(ts))


b = b0.clone()
out["single_ms"] = timed(lambda: (b.copy_(b0), H.hysco_admm(ctx, b, ao)))
J1 = H.hysco_admm(ctx, b.copy_(b0), ao)[0]["J"]
H.hysco_destroy(ctx)
for N in (1, 2, 4):
    ctxs = H.hysco_create_loopback((n1, n2, n3), p.h, N, stream=torch.cuda.current_stream().cuda_stream)
    keep, bs, b0s = [], [], []
    for r, c in enumerate(ctxs):
        i0, i1 = H.slab_bounds(n1, N, r)
        tI = Ip[:, i0:i1].contiguous()
        tM = Im[:, i0:i1].contiguous()
        keep += [tI, tM]
        H.hysco_bind_images(c, tI, tM)
        b0s.append(b0[:, i0:i1].contiguous())
        bs.append(b0s[-1].clone())
    torch.cuda.synchronize()

    def run():
        for x, y in zip(bs, b0s):
            x.copy_(y)
        return H.hysco_group_admm(ctxs, bs, ao)
    out[f"group{N}_ms"] = timed(run)
    out[f"group{N}_J_rel"] = abs(run()[0]["J"] - J1) / J1
    for c in ctxs:
        H.hysco_destroy(c)
print(json.dumps(out), flush=True)
