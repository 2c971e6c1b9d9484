"""Command-line front-end (the paper's CLI):

    python -m paper_2403_10706_b200.cli PLUS.nii.gz MINUS.nii.gz --pe-axis 2 --out OUT

reads the reversed-polarity pair (NIfTI-1, read natively by libhysco), moves the
PE axis last on the GPU, estimates the field map (OT init + blur +
guard -> Gauss-Newton-PCG or ADMM), corrects (Jacobian modulation and / or
least squares), moves the results back to the file's axis order and writes

    OUT_fieldmap.nii.gz   field map at the cell centres, voxel displacement along
                          +PE of the file's PE axis (--fieldmap-units mm: mm; R31)
    OUT_plus.nii.gz       Jacobian-modulation corrected I+   
    OUT_minus.nii.gz      Jacobian-modulation corrected I-
    OUT_lsq.nii.gz        least-squares corrected image      (--correction lsq|both)

with the geometry of the PLUS file.  Every numeric step is a libhysco call;
this module only parses arguments and moves buffers.  Prints one JSON line
with the stage timings and the solver report.

Exit status: 0 success; 2 bad arguments or mismatched image sizes; 3 the field
map is infeasible (|d_v b| >= 1 somewhere: the OT start, the GN or ADMM
result, or a least-squares column), nothing is written; 4 an I/O error
(unreadable / malformed input, unwritable output).
"""
import argparse
import ctypes
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def parse(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2403_10706_b200.cli",
                                 description="Reversed-gradient-polarity EPI distortion correction on a B200.")
    ap.add_argument("plus", help="image acquired with +PE (NIfTI-1 .nii / .nii.gz)")
    ap.add_argument("minus", help="image acquired with -PE")
    ap.add_argument("--pe-axis", type=int, choices=[1, 2, 3], required=True,
                    help="phase-encoding axis of the files (1 = x, 2 = y, 3 = z)")
    ap.add_argument("--out", required=True, help="output prefix")
    ap.add_argument("--alpha", type=float, default=300.0, help="smoothness weight (P:100)")
    ap.add_argument("--beta", type=float, default=1e-4, help="barrier weight (P:100)")
    ap.add_argument("--solver", default="gn", choices=["gn", "admm"])
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "block"])
    ap.add_argument("--stop", default="paper", choices=["paper", "fixed"],
                    help="paper stop rules (P:284) or fixed 10 GN x 10 PCG")
    ap.add_argument("--max-gn", type=int, default=10)
    ap.add_argument("--correction", default="jacobian", choices=["jacobian", "lsq", "both"])
    ap.add_argument("--lsq-lambda", type=float, default=0.05)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--no-blur", action="store_true")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--log-iters", action="store_true",
                    help="per-GN-step history (objective parts, gamma, PCG iterations; P:284) to stderr and the report")
    ap.add_argument("--no-gzip", action="store_true", help="write .nii instead of .nii.gz")
    ap.add_argument("--fieldmap-units", default="voxel", choices=["voxel", "mm"],
                    help="unit of OUT_fieldmap: voxel displacement (default) or mm, along +PE (R31)")
    return ap.parse_args(argv)


EXIT_OK, EXIT_ARGS, EXIT_INFEASIBLE, EXIT_IO = 0, 2, 3, 4


def _fail(code, msg):
    print(f"hysco: {msg}", file=sys.stderr, flush=True)
    return code


def main(argv=None):
    args = parse(argv)
    import torch
    from paper_2403_10706_b200 import hysco as H

    t0 = time.perf_counter()
    dtype = H.HYSCO_F64 if args.dtype == "f64" else H.HYSCO_F32
    tdt = torch.float64 if dtype == H.HYSCO_F64 else torch.float32
    try:
        info_p = H.hysco_nifti_info_read(args.plus)
        info_m = H.hysco_nifti_info_read(args.minus)
    except H.HyscoError as e:
        return _fail(EXIT_IO, str(e))
    dims = tuple(info_p.dim)
    if tuple(info_m.dim) != dims:
        return _fail(EXIT_ARGS, f"image sizes differ: {dims} vs {tuple(info_m.dim)}")
    n, h = H.hysco_pe_shape(dims, tuple(info_p.pixdim), args.pe_axis)
    nvox = dims[0] * dims[1] * dims[2]
    host = torch.empty((4, nvox), dtype=tdt, pin_memory=True)    # rows 0-1: the pair in; rows 0-3: results out
    L = H.lib()

    def read(k):
        # the I/O error message is thread-local in libhysco: fetch it in this worker
        s = L.hysco_nifti_read(os.fsencode((args.plus, args.minus)[k]), dtype, ctypes.c_void_p(host[k].data_ptr()),
                               nvox, None)
        return None if s == H.HYSCO_OK else f"{(args.plus, args.minus)[k]}: {L.hysco_io_last_error().decode()}"

    with ThreadPoolExecutor(2) as ex:            # the two files decompress concurrently (ctypes drops the GIL)
        errs = [e for e in ex.map(read, (0, 1)) if e]
    if errs:
        return _fail(EXIT_IO, "; ".join(errs))
    t_read = time.perf_counter()

    torch.cuda.set_device(args.device)
    dev = torch.device("cuda", args.device)
    stream = torch.cuda.current_stream(dev)
    raw = host[:2].to(dev, non_blocking=True)
    img = torch.empty((2,) + tuple(n), dtype=tdt, device=dev)
    H.hysco_permute_pe(raw, img, dims, args.pe_axis, False, dtype, batch=2, stream=stream.cuda_stream)
    ctx = H.hysco_create(n, h, 1, args.alpha, args.beta, dtype=dtype, device=args.device, stream=stream.cuda_stream)
    try:
        H.hysco_bind_images(ctx, img[0:1], img[1:2])
        b = torch.zeros((1, n[0], n[1], n[2] + 1), dtype=tdt, device=dev)
        outs = torch.zeros((4,) + tuple(n), dtype=tdt, device=dev)        # fieldmap, plus, minus, lsq
        ot = H.default_ot_opts(blur=0 if args.no_blur else 1)
        if args.solver == "gn":
            so = H.default_solve_opts(max_gn=args.max_gn, fixed_iters=1 if args.stop == "fixed" else 0,
                                      precond=H.HYSCO_PRECOND_PE_BLOCK if args.precond == "block"
                                      else H.HYSCO_PRECOND_JACOBI)
            reps, infeas = H.hysco_correct(ctx, b, outs[1:2], outs[2:3], ot, so)
            report = dict(reps[0], stop=H.STOP_NAMES.get(reps[0]["stop_reason"], "?"))
            if args.log_iters:                   # PyHySCO's OptimizationLogger
                report["history"] = H.hysco_history(ctx, 0)
                for r in report["history"]:
                    print(f"hysco: GN {r['k']:3d}  J {r['J']:.6e}  D {r['D']:.4e}  S {r['S']:.4e}  P {r['P']:.4e}  "
                          f"|grad| {r['grad_norm']:.3e}  gamma {r['gamma']:.4g}  pcg {r['pcg_iters']}  "
                          f"relres {r['relres']:.3e}", file=sys.stderr, flush=True)
            infeas = bool(infeas) or not np.isfinite(report["J"])
        else:
            H.hysco_ot_init(ctx, b, ot)
            report = H.hysco_admm(ctx, b, H.default_admm_opts(fixed_iters=1 if args.stop == "fixed" else 0))[0]
            H.hysco_apply(ctx, b, outs[1:2], outs[2:3])
            infeas = not np.isfinite(report["J"])        # ADMM reports J = +inf at an infeasible b
        if args.correction in ("lsq", "both") and not infeas:
            lrep, linf = H.hysco_lsq_correct(ctx, b, outs[3:4], H.default_lsq_opts(lam=args.lsq_lambda))
            report["lsq"] = lrep[0]
            infeas = bool(linf) or lrep[0]["infeasible"] > 0
        H.hysco_fieldmap_cells(ctx, b, outs[0:1],
                               H.HYSCO_FIELDMAP_VOXEL if args.fieldmap_units == "voxel" else H.HYSCO_FIELDMAP_MM)
        back = torch.empty((4, nvox), dtype=tdt, device=dev)
        H.hysco_permute_pe(outs, back, dims, args.pe_axis, True, dtype, batch=4, stream=stream.cuda_stream)
        res = host                                   # one pinned buffer per run (pinning costs ~ms per 10 MB)
        res.copy_(back, non_blocking=True)
        torch.cuda.synchronize(dev)
    finally:
        H.hysco_destroy(ctx)
    t_gpu = time.perf_counter()
    if infeas:
        print(json.dumps({"files": [], "infeasible": True, "report": {k: v for k, v in report.items()
                                                                       if not isinstance(v, float) or np.isfinite(v)}}),
              flush=True)
        return _fail(EXIT_INFEASIBLE, "infeasible field map (|d_v b| >= 1): nothing written")

    ext = ".nii" if args.no_gzip else ".nii.gz"
    names = ["fieldmap", "plus", "minus", "lsq"]
    keep = [0] + ([1, 2] if args.correction in ("jacobian", "both") else []) + \
        ([3] if args.correction in ("lsq", "both") else [])
    shape_file = (dims[2], dims[1], dims[0])
    files = [f"{args.out}_{names[k]}{ext}" for k in keep]

    def write(kp):
        try:
            H.hysco_nifti_write(kp[1], res[kp[0]].numpy().reshape(shape_file), info_p)
        except H.HyscoError as e:            # message fetched on this worker thread (thread-local)
            return f"{kp[1]}: {e}"
        return None

    with ThreadPoolExecutor(len(keep)) as ex:
        errs = [e for e in ex.map(write, zip(keep, files)) if e]
    if errs:
        return _fail(EXIT_IO, "; ".join(errs))
    t_write = time.perf_counter()
    print(json.dumps({"files": files, "kernel_shape": list(n), "pe_axis": args.pe_axis, "infeasible": False,
                      "fieldmap_units": args.fieldmap_units,
                      "seconds": {"read": t_read - t0, "gpu": t_gpu - t_read, "write": t_write - t_gpu,
                                  "total": t_write - t0},
                      "report": {k: v for k, v in report.items() if not isinstance(v, float) or np.isfinite(v)}}),
          flush=True)
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
