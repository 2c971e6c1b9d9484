"""CUPTI kernel totals of one ADMM correction (OT + hysco_admm + apply) on the
3T shape (diagnostic).  usage: python tools/timeline_admm.py [config]"""
import os
import sys
import json
import collections

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
from torch.profiler import profile, ProfilerActivity
from paper_2403_10706_b200 import hysco as H
from synth import phantom

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2_hcp3t"
p = phantom.make_config(cfg)
n1, n2, n3 = p.Ip.shape
ctx = H.hysco_create(p.Ip.shape, p.h, 1, stream=torch.cuda.current_stream().cuda_stream)
Ip = torch.from_numpy(p.Ip[None]).cuda()
Im = torch.from_numpy(p.Im[None]).cuda()
H.hysco_bind_images(ctx, Ip, Im)
b = torch.zeros((1, n1, n2, n3 + 1), device="cuda")
Tp = torch.zeros((1, n1, n2, n3), device="cuda")
Tm = torch.zeros_like(Tp)
opts = H.default_admm_opts(max_iter=50)
for _ in range(2):
    H.hysco_ot_init(ctx, b)
    H.hysco_admm(ctx, b, opts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    H.hysco_ot_init(ctx, b)
    r = H.hysco_admm(ctx, b, opts)
    H.hysco_apply(ctx, b, Tp, Tm)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "timeline_admm.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
t0, t1 = ks[0]["ts"], ks[-1]["ts"] + ks[-1]["dur"]
tot = collections.defaultdict(lambda: [0, 0.0])
for e in ks:
    k = e["name"].split("(")[0].replace("void ", "")[:60]
    tot[k][0] += 1
    tot[k][1] += e["dur"]
print(f"span {t1 - t0:.1f} us, kernels {sum(v[1] for v in tot.values()):.1f} us, iterations {r[0]['iters']}")
for k, (n, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {k:60s} n={n:4d} total {d:9.1f} us avg {d / n:7.1f}")
H.hysco_destroy(ctx)
