"""Device timeline (CUPTI via torch.profiler) of hysco_correct_host_stream over
a few 3T items: kernels and copies per stream, the gaps on the compute stream
between one item's last kernel and the next item's first.  Diagnostic only.
usage: python tools/timeline_stream.py [items]"""
import os
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2403_10706_b200 import hysco as H
from synth import phantom


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    p = phantom.make_config("C2_hcp3t")
    n1, n2, n3 = p.Ip.shape
    ctx = H.hysco_create((n1, n2, n3), p.h, 1, device=0)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hIp, hIm = pin(p.Ip[None]), pin(p.Im[None])
    hb = torch.zeros((1, n1, n2, n3 + 1)).pin_memory()
    hTp, hTm = torch.zeros((1, n1, n2, n3)).pin_memory(), torch.zeros((1, n1, n2, n3)).pin_memory()
    run = lambda k: H.hysco_correct_host_stream(ctx, [hIp] * k, [hIm] * k, [hb] * k, [hTp] * k, [hTm] * k)
    run(2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run(n)
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", "timeline_stream.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    last_end = {}
    for e in ks:
        name = e["name"].split("(")[0].replace("void ", "")[:50]
        s = e.get("args", {}).get("stream", "?")
        g = e["ts"] - last_end.get(s, e["ts"])
        last_end[s] = e["ts"] + e["dur"]
        if e.get("cat") != "kernel" or g > 5 or "eval" in name and False:
            print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} gap {g:7.1f} s{s}  {e.get('cat')[:10]:10s} {name}")
    span = ks[-1]["ts"] + ks[-1]["dur"] - t0
    kt = sum(e["dur"] for e in ks if e.get("cat") == "kernel")
    print(f"span {span:.1f} us for {n} items = {span / n:.1f} us per item; kernel time {kt / n:.1f} us per item")
    H.hysco_destroy(ctx)


if __name__ == "__main__":
    main()
