"""fp32 ADMM (hysco_admm) vs the fp64 oracle (O.admm) over the iteration count:
relative L2 of b after k fixed iterations from the same OT start, and the same
run with the GPU in fp64 (DESIGN.md ADMM tolerances).  Writes one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import hysco_oracle as O          # noqa: E402
from paper_2403_10706_b200 import hysco as H  # noqa: E402
from synth import phantom                      # noqa: E402

out = []
for shape, seed in [((12, 10, 24), 3), ((5, 7, 37), 5), ((4, 5, 144), 7), ((24, 20, 48), 9)]:
    p = phantom.make_pair(shape, (1.25, 1.25, 1.1), seed)
    for dtype, nd, td in [(H.HYSCO_F32, np.float32, torch.float32), (H.HYSCO_F64, np.float64, torch.float64)]:
        Ip, Im = p.Ip.astype(nd).astype(np.float64), p.Im.astype(nd).astype(np.float64)
        b0 = O.ot_init(Ip, Im, p.h[2])[0].astype(nd).astype(np.float64)
        for its in (1, 2, 4, 8, 16, 33):
            tIp = torch.from_numpy(Ip[None].astype(nd)).cuda()
            tIm = torch.from_numpy(Im[None].astype(nd)).cuda()
            ctx = H.hysco_create(shape, p.h, 1, dtype=dtype)
            H.hysco_bind_images(ctx, tIp, tIm)
            b = torch.from_numpy(b0.reshape((1,) + b0.shape).astype(nd)).cuda()
            torch.cuda.synchronize()
            reps = H.hysco_admm(ctx, b, H.default_admm_opts(max_iter=its, fixed_iters=1))
            torch.cuda.synchronize()
            bg = b.cpu().numpy()[0].astype(np.float64)
            H.hysco_destroy(ctx)
            bref, _, rep = O.admm(Ip, Im, b0, p.h, max_iter=its, fixed=True)
            e = float(np.linalg.norm(bg - bref) / np.linalg.norm(bref))
            out.append({"shape": shape, "dtype": "f32" if dtype == H.HYSCO_F32 else "f64", "iters": its, "rel_b": e,
                        "rho_gpu": reps[0]["rho"], "rho_oracle": rep["rho_final"]})
            print(shape, out[-1]["dtype"], its, "%.2e" % e, reps[0]["rho"] == rep["rho_final"], flush=True)
json.dump(out, open("gpurun_out/admm_f32_error.json", "w"), indent=1)
