"""Kernel timeline of one hysco_correct step (CUPTI via torch.profiler): every
kernel's device start/end, the gaps between consecutive kernels, and totals
per kernel name.  Diagnostic only.  usage: python tools/timeline.py [config]"""
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


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2_hcp3t"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1      # pairs per context (batch)
    p = phantom.make_config(cfg)
    n1, n2, n3 = p.Ip.shape
    dev = "cuda:0"
    Ip = torch.from_numpy(p.Ip[None]).to(dev).repeat(B, 1, 1, 1).contiguous()
    Im = torch.from_numpy(p.Im[None]).to(dev).repeat(B, 1, 1, 1).contiguous()
    stream = torch.cuda.current_stream()
    ctx = H.hysco_create((n1, n2, n3), p.h, B, device=0, stream=stream.cuda_stream)
    H.hysco_bind_images(ctx, Ip, Im)
    b = torch.zeros((B, n1, n2, n3 + 1), device=dev)
    Tp = torch.zeros((B, n1, n2, n3), device=dev)
    Tm = torch.zeros_like(Tp)
    for _ in range(3):
        H.hysco_correct(ctx, b, Tp, Tm, batch=B)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            H.hysco_correct(ctx, b, Tp, Tm, batch=B)
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", "timeline_trace.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
    # the second step: kernels after the largest gap in the middle
    gaps = [(ks[i + 1]["ts"] - (ks[i]["ts"] + ks[i]["dur"]), i) for i in range(len(ks) - 1)]
    half = len(ks) // 2
    split = max(gaps[half - 5: half + 5])[1] + 1 if len(ks) > 20 else 0
    step = ks[split:]
    t0 = step[0]["ts"]
    t1 = step[-1]["ts"] + step[-1]["dur"]
    tot = collections.defaultdict(lambda: [0, 0.0])
    gap_sum = 0.0
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  kernel")
    prev_end = None
    for e in step:
        g = 0.0 if prev_end is None else e["ts"] - prev_end
        gap_sum += max(g, 0.0)
        prev_end = e["ts"] + e["dur"]
        name = e["name"].split("(")[0].replace("void ", "")[:60]
        tot[name][0] += 1
        tot[name][1] += e["dur"]
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} {g:7.1f}  {name}")
    print(f"\nstep span {t1 - t0:.1f} us, kernel time {sum(v[1] for v in tot.values()):.1f} us, gaps {gap_sum:.1f} us")
    for k, (n, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"  {k:60s} n={n:3d} total {d:8.1f} us avg {d / n:7.1f}")
    H.hysco_destroy(ctx)


if __name__ == "__main__":
    main()
