#!/usr/bin/env python
"""bench.py — volume pairs corrected per second (HCP 3T shape) on N B200s.

A step = the whole hot path for the pairs each
rank owns: OT init + blur + guard -> 10 GN x 10 Jacobi-PCG (+Armijo) -> apply,
one hysco_correct() call through the C ABI (one CUDA-graph launch).  Inputs
are already resident in HBM (device timing, CUDA events on the context
stream, L2 flushed by a 256 MiB write between timed steps); `e2e` is the same
metric through hysco_correct_host() with pinned host buffers (H2D of the pair
and D2H of b and the two corrected images inside the timed region).

Multi-GPU (torchrun, one process per GPU): pairs are independent (BASELINE.json
configs[3], "batch ... split across GPUs"), so each rank corrects its own
pairs with no data-path collective ("scaling": "weak"); timing is the max over
ranks of the device-timed region.

--impl reference: the CPU fp64 oracle (oracle/), as it stands, on the host
cores — the reference arm of this tier.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import phantom  # noqa: E402

METRIC = "volume pairs corrected/sec (HCP 3T shape)"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hysco", choices=["hysco", "reference"])
    ap.add_argument("--config", default="C2_hcp3t", choices=sorted(phantom.CONFIGS))
    ap.add_argument("--batch", type=int, default=1, help="pairs per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="items timed through the host entry (default: --steps, one item per step)")
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "block"],
                    help="PCG preconditioner: Jacobi (P:198, the headline) or per-PE-column blocks (P:200)")
    ap.add_argument("--stop", default="fixed", choices=["fixed", "paper"],
                    help="fixed 10 GN x 10 PCG (the headline) or the paper's stop rules (P:196, P:284, R16)")
    ap.add_argument("--solver", default="gn", choices=["gn", "admm"],
                    help="Gauss-Newton-PCG (the headline, P:183-199) or ADMM (P:203-239) with the paper-style stop")
    ap.add_argument("--stage", default="path", choices=["path", "lsq", "cli"],
                    help="the GN path (default) or the NEXT-3 stage: push-forward simulation of the pair from the "
                         "true image + least-squares correction (P:289, P:331); or the whole command-line run "
                         "(NIfTI .nii.gz in/out, P:291-295; the paper's 'Run' column)")
    ap.add_argument("--slab", action="store_true",
                    help="partition ONE pair of --config into slabs along dim 1 across the ranks (configs[4])")
    return ap.parse_args()


def solver_desc(args=None):
    pc = "Jacobi" if args is None or args.precond == "jacobi" else "PE-block"
    if args is None or args.stop == "fixed":
        return f"fixed 10 GN x 10 {pc}-PCG + Armijo"
    return f"GN-{pc}-PCG with the paper's stop rules (PCG rtol 0.1, R16 GN tests, <= 50 GN) + Armijo"


def solve_opts(H, args):
    kw = {}
    if args.precond == "block":
        kw["precond"] = H.HYSCO_PRECOND_PE_BLOCK
    if args.stop == "paper":
        kw.update(fixed_iters=0, max_gn=50)
    return H.default_solve_opts(**kw)


def workload_desc(cfg, batch, args=None):
    shape, h, seed = phantom.CONFIGS[cfg]
    return {"workload": f"{cfg}: {shape[0]}x{shape[1]}x{shape[2]} cells (PE last), h={tuple(round(v, 4) for v in h)} mm, "
                        f"OT+blur+guard -> {solver_desc(args)} -> Jacobian-modulation apply",
            "pairs_per_gpu": batch, "seed": seed, "alpha": 300.0, "beta": 1e-4,
            "l2": "flushed (256 MiB write) between timed steps"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(2)
        except Exception:
            self.p.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].lower() in ("active", "1")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- CPU oracle timing (reference)

def host_info():
    """Host CPU model and the cores this process may run on."""
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cpus": aff}


def oracle_sample(pair, planes):
    """Time the oracle, as it stands, on a bounded sample of the workload: the
    WHOLE path (OT + blur + guard -> fixed 10 GN x 10 Jacobi-PCG + Armijo ->
    apply, O.correct_pair) on the slab of planes [0, planes) of dim 1 of the
    pair, a volume of its own.  Seconds per pair = the slab's time x n1 /
    planes (the path's work is linear in the number of PE columns).  BLAS /
    OpenMP pools are limited to one thread.  Returns (s_per_pair, desc, wall)."""
    from oracle import hysco_oracle as O
    from threadpoolctl import threadpool_limits
    n1 = pair.Ip.shape[0]
    planes = max(2, min(n1, int(planes)))
    Ip = pair.Ip[:planes].astype(np.float64)
    Im = pair.Im[:planes].astype(np.float64)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        O.correct_pair(Ip, Im, pair.h)
        wall = time.perf_counter() - t0
    desc = (f"oracle (NumPy fp64, 1 thread) whole path OT+blur+guard -> 10 GN x 10 PCG + Armijo -> apply on "
            f"planes [0, {planes}) of the {tuple(pair.Ip.shape)} pair; per pair = time x {n1}/{planes}")
    return wall * n1 / planes, desc, wall


def oracle_planes_for(pair, seconds):
    """Planes whose oracle sample takes about `seconds` (probe on 4 planes)."""
    _, _, w4 = oracle_sample(pair, 4)
    return int(max(2, min(pair.Ip.shape[0], round(4 * seconds / max(w4, 1e-3)))))


def run_reference(args):
    """The reference arm of this tier: the CPU oracle as it stands, each step a
    bounded sample of the workload (oracle_sample), on rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    shape, h, seed = phantom.CONFIGS[args.config]
    pair = phantom.make_pair(shape, h, seed)
    # bounded: the whole --steps K --warmup W run takes ~2-3 minutes
    planes = oracle_planes_for(pair, 150.0 / max(args.steps + args.warmup, 1))
    for _ in range(args.warmup):
        oracle_sample(pair, planes)
    vals, ms = [], []
    desc = ""
    for _ in range(args.steps):
        spp, desc, wall = oracle_sample(pair, planes)
        vals.append(spp)
        ms.append(wall * 1e3)
    spp = float(np.mean(vals))
    v = 1.0 / spp
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(ms)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload_desc(args.config, 1), parallelism="dp1 (independent pairs per rank)"),
            "cpu_baseline": dict({"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc}, **host_info()),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- roofline

# FP32 pipe peak for the ALU-bound path: 148 SMs x 128 FP32 lanes x 2 flop/FMA x
# 1.965 GHz (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz; 4 SMSPs x 32
# FP32 lanes per SM) = 74.4 TFLOP/s.  DESIGN.md §10.
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
# algorithmic fp32 flops per node per PCG iteration of the resident kernel:
# matvec 14 (M p, 2 PE FMAs, 3 in-plane adds, 2 FMAs, p.Hp), update 10, direction 4
RESIDENT_FLOPS_PER_NODE_ITER = 28


_L2PK = {}


def l2_peak_gbs():
    """Measured L2 bandwidth: torch copy of a 24 MiB buffer into another (48 MiB
    working set, L2-resident), read + write bytes, best of 50 (CUDA events)."""
    if _L2PK:
        return _L2PK
    import torch
    n = 24 << 18
    a = torch.ones(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    best = None
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    _L2PK.update(gbs=2 * 4 * n / (best * 1e-3) / 1e9,
                 how="measured live: torch copy of 24 MiB (48 MiB read + write working set, L2-resident), best of 50")
    return _L2PK


def ncu_kernel_summary(config, name):
    """profiles/ncu_summary.json entry of kernel `name` on workload `config`
    (ncu --set full of this round's build, per launch; make_ncu_summary.py)."""
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return summ.get("configs", {}).get(config, {}).get(name)
    except Exception:
        return None


def roofline_entry(H, ctx, args, r0, B, shape, ms_per_step):
    """The kernel with the largest share of a step, timed by hysco_profile_kernels
    (each hot kernel re-launched on the context stream, same grid and buffers,
    CUDA events per launch; cold = L2 flushed before each launch).  DESIGN.md §10."""
    n1, n2, n3 = shape
    prof_cold = H.hysco_profile_kernels(ctx, args.profile_reps, flush_l2=True)
    prof_warm = H.hysco_profile_kernels(ctx, args.profile_reps, flush_l2=False)
    Nn, Nc = B * n1 * n2 * (n3 + 1), B * n1 * n2 * n3
    resident = prof_warm["pcg_resident"] > 0
    l2pcg = prof_warm.get("pcg_l2", -1) > 0
    flat = prof_warm.get("pcg_dirmv", -1) > 0
    gn = r0["gn_iters"]
    if resident:   # one cooperative launch per GN step runs all PCG iterations and the Armijo start
        per_step = {"pcg_resident": gn, "eval": r0["f_evals"]}
    elif l2pcg:    # the same with the PCG state in L2 (hysco_l2pcg.cuh)
        per_step = {"pcg_l2": gn, "eval": r0["f_evals"]}
    elif flat:     # two vectorised launches per PCG iteration (hysco_flat.cuh)
        per_step = {"pcg_dirmv": r0["h_evals"], "pcg_upd": r0["pcg_iters"], "eval": r0["f_evals"],
                    "trial_init": gn}
    else:
        per_step = {"matvec": r0["h_evals"], "pcg_update": r0["pcg_iters"], "pcg_dir": r0["pcg_iters"],
                    "eval": r0["f_evals"], "trial_init": gn}
    # algorithmic bytes per launch of the streaming kernels (DESIGN.md §7 table);
    # flat form: dirmv reads z, p_old, dt, et, x and writes p, Hp, x; upd reads
    # r, Hp, dt and writes r, z; its Armijo start also reads the last p
    algo_bytes = {"matvec": 16 * Nn, "pcg_update": 28 * Nn, "pcg_dir": 16 * Nn, "eval": 16 * Nn + 8 * Nc,
                  "trial_init": (28 if flat else 20) * Nn, "pcg_dirmv": 32 * Nn, "pcg_upd": 20 * Nn}
    share = {k: prof_warm[k] * per_step[k] / ms_per_step for k in per_step}
    dom = max(share, key=share.get)
    hbm_peak, peak_src = peaks()
    out = {"kernel": dom, "kernel_share_of_step": share,
           "avg_launch_ms_cold_l2": prof_cold[dom], "avg_launch_ms_warm_l2": prof_warm[dom],
           "launches_per_step": per_step}
    ncu = ncu_kernel_summary(args.config, dom)
    out["traffic"] = ncu.get("dram_bytes_per_launch") if ncu else None
    if dom == "pcg_resident":
        # The resident PCG keeps p, M, et on chip (shared memory) and r, z in
        # registers: its DRAM traffic is the per-launch in/out only, so it is not
        # HBM-bound.  Its limit is the per-iteration dependency chain (p-halo
        # exchange with the neighbour CTAs, two grid-wide all-reduces): the
        # roofline is that chain's MEASURED floor -- the same launch running
        # only the synchronisation, no arithmetic or data movement
        # (hysco_profile_kernels slot 6) -- against the measured iteration time.
        its = max(r0["pcg_iters"] / max(gn, 1), 1.0)
        it_us = prof_warm[dom] * 1e3 / its
        floor_us = prof_warm["resident_sync_floor"] * 1e3 / 10.0
        flops = RESIDENT_FLOPS_PER_NODE_ITER * Nn * its
        ach_f = flops / (prof_warm[dom] * 1e-3) / 1e12
        out.update({"bound": "latency", "achieved": it_us, "peak": floor_us, "unit": "us per PCG iteration",
                    "frac": floor_us / it_us,
                    "peak_source": "measured live: pcg_sync_floor_kernel, the resident launch's synchronisation "
                                   "chain alone (DESIGN.md §10)",
                    "note": "frac = floor / achieved (time-like: lower is better)",
                    "physical": {
                        "fp32_pipe": {"achieved_tflops": ach_f, "peak_tflops": FP32_PEAK_TFLOPS,
                                      "frac": ach_f / FP32_PEAK_TFLOPS,
                                      "flops_per_launch": flops, "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1.965 GHz"},
                        "dram": ({"bytes_per_launch": ncu["dram_bytes_per_launch"],
                                  "achieved_gbs": ncu["dram_bytes_per_launch"] / (prof_warm[dom] * 1e-3) / 1e9,
                                  "peak_gbs": hbm_peak,
                                  "frac": ncu["dram_bytes_per_launch"] / (prof_warm[dom] * 1e-3) / 1e9 / hbm_peak}
                                 if ncu and ncu.get("dram_bytes_per_launch") else None),
                        "sm_throughput_frac": (ncu.get("sm_throughput_pct") / 100.0
                                               if ncu and ncu.get("sm_throughput_pct") is not None else None),
                        "source": "ncu --set full of this build (profiles/ncu_summary.json) for dram / sm; "
                                  "fp32 from the live launch time"}})
    elif dom == "pcg_l2":
        # PCG state (p, dt, et, r, x, Hp) L2-resident across the launch: the
        # bytes it moves per launch are the streaming kernels' (SURVEY §8(d4):
        # per iteration matvec 16 + update 28 + direction 16 B/node, start and
        # Armijo start 20 + 20 B/node), served by L2; the roofline is the
        # MEASURED L2 bandwidth (l2_peak_gbs), DRAM traffic in `traffic`
        its = max(r0["pcg_iters"] / max(gn, 1), 1.0)
        byts = (60 * its + 40) * Nn
        ach = byts / (prof_warm[dom] * 1e-3) / 1e9
        l2pk = l2_peak_gbs()
        out.update({"bound": "l2", "achieved": ach, "peak": l2pk["gbs"], "unit": "GB/s", "frac": ach / l2pk["gbs"],
                    "algorithmic_bytes_per_launch": byts, "peak_source": l2pk["how"],
                    "hbm_view": {"achieved_gbs": ach, "peak_gbs": hbm_peak, "frac": ach / hbm_peak,
                                 "note": "algorithmic bytes over the HBM peak: > 1 means the kernel beats any "
                                         "HBM-streaming PCG; not a physical fraction"},
                    "us_per_iteration": prof_warm[dom] * 1e3 / its})
    else:
        ach = algo_bytes[dom] / (prof_cold[dom] * 1e-3) / 1e9
        out.update({"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                    "algorithmic_bytes_per_launch": algo_bytes[dom], "peak_source": peak_src,
                    "achieved_warm_l2": algo_bytes[dom] / (prof_warm[dom] * 1e-3) / 1e9})
    # whole step against HBM: SURVEY §8(d4) bytes of a streaming fixed 10 x 10 solve
    step_bytes = (r0["pcg_iters"] * 52 + r0["f_evals"] * 32 + gn * 16 + 40) * Nn
    out["step_view"] = {"algorithmic_bytes": step_bytes, "achieved_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
                        "frac_of_hbm_peak": step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm_peak,
                        "note": "SURVEY §8(d4) bytes a streaming implementation of the step must move, / step time"}
    # the HBM-bound kernels of the step, for context (cold L2)
    out["hbm_kernels"] = {k: {"GBps_cold": algo_bytes[k] / (prof_cold[k] * 1e-3) / 1e9,
                              "frac_cold": algo_bytes[k] / (prof_cold[k] * 1e-3) / 1e9 / hbm_peak}
                          for k in (("eval", "trial_init", "pcg_dirmv", "pcg_upd") if flat else
                                    ("eval", "trial_init", "matvec", "pcg_update", "pcg_dir"))
                          if prof_cold.get(k, -1) > 0}
    return out


# ---------------------------------------------------------------- GPU path

def run_hysco(args):
    import torch
    from paper_2403_10706_b200 import hysco as H

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    shape, h, seed = phantom.CONFIGS[args.config]
    n1, n2, n3 = shape
    B = args.batch
    pairs = [phantom.make_pair(shape, h, seed + 1000 * rank + k) for k in range(B)]
    Ip_h = np.stack([p.Ip for p in pairs])
    Im_h = np.stack([p.Im for p in pairs])
    Ip = torch.from_numpy(Ip_h).to(dev)
    Im = torch.from_numpy(Im_h).to(dev)
    stream = torch.cuda.current_stream(dev)
    ctx = H.hysco_create(shape, h, B, device=local, stream=stream.cuda_stream)
    H.hysco_bind_images(ctx, Ip, Im)
    so = solve_opts(H, args)
    b = torch.zeros((B, n1, n2, n3 + 1), dtype=torch.float32, device=dev)
    Tp = torch.zeros((B, n1, n2, n3), dtype=torch.float32, device=dev)
    Tm = torch.zeros_like(Tp)
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2

    for _ in range(max(args.warmup, 0)):
        H.hysco_correct(ctx, b, Tp, Tm, solve_opts=so, batch=B)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    reps = None
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        reps, inf = H.hysco_correct(ctx, b, Tp, Tm, solve_opts=so, batch=B)
        ev[k][1].record(stream)
        launches += H.hysco_last_launch_count(ctx)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    step_ms = [a.elapsed_time(z) for a, z in ev]
    total_ms = float(np.sum(step_ms))
    step_stats = {"median": float(np.median(step_ms)), "p10": float(np.percentile(step_ms, 10)),
                  "p90": float(np.percentile(step_ms, 90)), "min": float(np.min(step_ms)),
                  "max": float(np.max(step_ms))}
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_max = float(t.item())
    value = world * B * args.steps / (total_max / 1e3)
    ms_per_step = total_max / args.steps

    # correction quality of the timed result (pair 0): relative improvement of
    # the SSD and the field-map error against the analytic b_true,
    # everywhere and inside the object (I_true > 10 % of its max)
    torch.cuda.synchronize(dev)
    bh = b[0].double().cpu().numpy()
    Tph, Tmh = Tp[0].double().cpu().numpy(), Tm[0].double().cpu().numpy()
    p0 = pairs[0]
    d0 = float(np.sum((p0.Ip.astype(np.float64) - p0.Im.astype(np.float64)) ** 2))
    mask_c = p0.I_true > 0.1 * p0.I_true.max()
    mask_n = np.zeros(bh.shape, bool)
    mask_n[..., :-1] |= mask_c
    mask_n[..., 1:] |= mask_c
    quality = {"relative_improvement_pct": 100.0 * (1.0 - float(np.sum((Tph - Tmh) ** 2)) / d0),
               "fieldmap_rel_l2_vs_true": float(np.linalg.norm(bh - p0.b_true) / np.linalg.norm(p0.b_true)),
               "fieldmap_rel_l2_vs_true_in_object": float(np.linalg.norm((bh - p0.b_true)[mask_n]) /
                                                          np.linalg.norm(p0.b_true[mask_n])),
               "fieldmap_max_abs_err_mm_in_object": float(np.abs(bh - p0.b_true)[mask_n].max()),
               "object_mask": "I_true > 0.1 max (cells; nodes touching them)", "pair": "rank 0, pair 0"}
    roofline = roofline_entry(H, ctx, args, reps[0], B, (n1, n2, n3), ms_per_step)
    r0 = reps[0]
    Nn, Nc = B * n1 * n2 * (n3 + 1), B * n1 * n2 * n3

    # ---- e2e through the host entry point (pinned buffers)
    hIp = torch.from_numpy(Ip_h).pin_memory()
    hIm = torch.from_numpy(Im_h).pin_memory()
    hb = torch.empty((B, n1, n2, n3 + 1), dtype=torch.float32).pin_memory()
    hTp = torch.empty((B, n1, n2, n3), dtype=torch.float32).pin_memory()
    hTm = torch.empty_like(hTp).pin_memory()
    # e2e: the pipelined host entry (hysco_correct_host_stream) over e2e_steps
    # items; every item's pair is copied in from pinned host memory and its b
    # and corrected pair copied back inside the timed region (the copies of
    # items k+1 / k-1 overlap the correction of item k on a second stream).
    ne = max(2, args.e2e_steps if args.e2e_steps is not None else args.steps)
    H.hysco_correct_host_stream(ctx, [hIp] * 2, [hIm] * 2, [hb] * 2, [hTp] * 2, [hTm] * 2, solve_opts=so, batch=B)
    flush.zero_()
    torch.cuda.synchronize(dev)
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record(stream)
    H.hysco_correct_host_stream(ctx, [hIp] * ne, [hIm] * ne, [hb] * ne, [hTp] * ne, [hTm] * ne,
                                solve_opts=so, batch=B)
    z.record(stream)
    z.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3
    te = torch.tensor([a.elapsed_time(z)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_val = world * B * ne / (float(te.item()) / 1e3)
    e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 2 * Nc * 4,
           "d2h_bytes_per_step": (Nn + 2 * Nc) * 4, "ms_per_step": float(te.item()) / ne,
           "api": "hysco_correct_host_stream (copies of neighbouring items overlap the correction)",
           "items": ne, "wall_ms_per_step": wall_ms / ne}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        spp, desc, wall = oracle_sample(pairs[0], oracle_planes_for(pairs[0], 15.0))
        cpu = dict({"value": 1.0 / spp, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                    "sample_seconds": wall}, **host_info())

    H.hysco_destroy(ctx)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(workload_desc(args.config, B, args), parallelism=f"dp{world} (independent pairs per rank)"),
                "step_ms": step_stats, "quality": quality,
                "clocks": clocks, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
                "cpu_baseline": cpu,
                "solver": {k: r0[k] for k in ("gn_iters", "f_evals", "h_evals", "pcg_iters", "stop", "J")},
                # a batch holds B different synthetic pairs (seeds), whose Armijo
                # searches differ: objective evaluations per pair of the last step
                **({"f_evals_per_pair": [int(r["f_evals"]) for r in reps]} if B > 1 else {}),
                "paper_context": {"seconds_per_pair": 4.38, "pairs_per_s": 1 / 4.38,
                                  "hardware": "GPU inferred RTX A6000, fp32, real HCP 3T data",
                                  "source": "PAPER.md Table 3 (P:476)"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_admm(args):
    """ADMM mode (not the headline): per step OT init + blur + guard, ADMM
    (hysco_admm: per-column b-update, cuFFT z-update, residual balancing;
    stops on the change tolerance, <= 50 iterations) and the correction."""
    import torch
    from paper_2403_10706_b200 import hysco as H

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shape, h, seed = phantom.CONFIGS[args.config]
    n1, n2, n3 = shape
    p = phantom.make_pair(shape, h, seed + 1000 * rank)
    Ip = torch.from_numpy(p.Ip[None]).to(dev)
    Im = torch.from_numpy(p.Im[None]).to(dev)
    stream = torch.cuda.current_stream(dev)
    ctx = H.hysco_create(shape, h, 1, device=local, stream=stream.cuda_stream)
    H.hysco_bind_images(ctx, Ip, Im)
    ao = H.default_admm_opts(max_iter=50)
    b = torch.zeros((1, n1, n2, n3 + 1), dtype=torch.float32, device=dev)
    Tp = torch.zeros((1, n1, n2, n3), dtype=torch.float32, device=dev)
    Tm = torch.zeros_like(Tp)
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)

    def step():
        H.hysco_ot_init(ctx, b)
        r = H.hysco_admm(ctx, b, ao)
        H.hysco_apply(ctx, b, Tp, Tm)
        return r

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ms, launches, rep = [], 0, None
    for _ in range(args.steps):
        flush.zero_()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rep = step()
        z.record(stream)
        z.synchronize()
        ms.append(a.elapsed_time(z))
        launches += H.hysco_last_launch_count(ctx)
    clocks = clk.stop()
    H.hysco_destroy(ctx)
    if rank == 0:
        tot = float(np.sum(ms))
        line = {"metric": METRIC, "value": world * args.steps / (tot / 1e3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": f"{args.config}: OT+blur+guard -> ADMM (P:203-239, stop on change tol 1e-3, "
                                       "<= 50 iterations) -> Jacobian-modulation apply", "pairs_per_gpu": 1,
                           "seed": seed, "l2": "flushed (256 MiB write) between timed steps",
                           "parallelism": f"dp{world} (independent pairs per rank)"},
                "clocks": clocks, "gpu_launches": launches, "solver": rep[0],
                "note": "mode line (not the headline); host-synchronised ADMM loop, cuFFT launches not counted"}
        print(json.dumps(line), flush=True)


def run_lsq(args):
    """NEXT-3 mode (not the headline): per step the distorted pair is simulated
    from the synthetic true image and field map by push-forward and
    corrected by least squares (R28, lambda = 0.05), both through the
    C ABI.  Timed with CUDA events on the context stream; each kernel timed
    alone as well."""
    import torch
    from paper_2403_10706_b200 import hysco as H

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shape, h, seed = phantom.CONFIGS[args.config]
    n1, n2, n3 = shape
    p = phantom.make_pair(shape, h, seed + 1000 * rank)
    T = torch.from_numpy(p.I_true[None].astype(np.float32)).to(dev)
    b = torch.from_numpy(p.b_true[None].astype(np.float32)).to(dev)
    Ip, Im, out = torch.zeros_like(T), torch.zeros_like(T), torch.zeros_like(T)
    stream = torch.cuda.current_stream(dev)
    ctx = H.hysco_create(shape, h, 1, device=local, stream=stream.cuda_stream)
    H.hysco_bind_images(ctx, Ip, Im)
    lo = H.default_lsq_opts()
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)          # noqa: E731
    rep = None
    for _ in range(max(args.warmup, 0)):
        H.hysco_push_forward(ctx, b, T, Ip, Im)
        rep, _ = H.hysco_lsq_correct(ctx, b, out, lo)
    torch.cuda.synchronize(dev)
    err = float(torch.linalg.norm(out - T) / torch.linalg.norm(T))
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ms, ms_pf, ms_lsq, launches = [], [], [], 0
    for _ in range(args.steps):
        flush.zero_()
        a, m, z = ev(), ev(), ev()
        a.record(stream)
        H.hysco_push_forward(ctx, b, T, Ip, Im)
        launches += H.hysco_last_launch_count(ctx)
        m.record(stream)
        rep, _ = H.hysco_lsq_correct(ctx, b, out, lo)
        launches += H.hysco_last_launch_count(ctx)
        z.record(stream)
        z.synchronize()
        ms.append(a.elapsed_time(z))
        ms_pf.append(a.elapsed_time(m))
        ms_lsq.append(m.elapsed_time(z))
    clocks = clk.stop()
    H.hysco_destroy(ctx)
    if rank == 0:
        tot = float(np.sum(ms))
        Nc, Nn = n1 * n2 * n3, n1 * n2 * (n3 + 1)
        pf_bytes, lsq_bytes = 4 * (3 * Nc + Nn), 4 * (3 * Nc + Nn)
        peak, peak_src = peaks()
        t_pf, t_lsq = float(np.mean(ms_pf)), float(np.mean(ms_lsq))
        line = {"metric": "volume pairs simulated + least-squares corrected/sec", "value": world * args.steps / (tot / 1e3),
                "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}: push-forward simulation of I+- from the true image and "
                                       "field map (P:331, R27) -> least-squares correction (P:289, R28, "
                                       "lambda 0.05, Jacobi-PCG to rtol 1e-6 per PE column)",
                           "pairs_per_gpu": 1, "seed": seed, "l2": "flushed (256 MiB write) between timed steps",
                           "parallelism": f"dp{world} (independent pairs per rank)"},
                "clocks": clocks, "gpu_launches": launches,
                "kernels_ms": {"push_forward": t_pf, "lsq": t_lsq},
                "roofline": {"bound": "latency (per-column PCG in shared memory)",
                             "hbm_view": {"push_forward_GBs": pf_bytes / (t_pf * 1e6),
                                          "lsq_GBs": lsq_bytes / (t_lsq * 1e6), "peak": peak, "peak_src": peak_src,
                                          "bytes_per_pair": {"push_forward": pf_bytes, "lsq": lsq_bytes}}},
                "lsq_report": rep[0], "rel_error_vs_true_image": err,
                "note": "mode line (not the headline); kernel times include the host read of the per-pair stats"}
        print(json.dumps(line), flush=True)


def run_cli(args):
    """NEXT-4 mode (not the headline): the command-line front-end end to end
    on the --config pair written as gzip NIfTI files with the PE axis along y
    (the file order needs the GPU permutation): read + decompress, H2D,
    permute, OT + GN-PCG (paper stop rules) + Jacobian correction, permute
    back, D2H, compress + write fieldmap / plus / minus.  Wall clock of
    cli.main() per step (the paper's 'Run' time includes its I/O, T3)."""
    import tempfile
    from paper_2403_10706_b200 import cli
    from paper_2403_10706_b200 import hysco as H

    shape, h, seed = phantom.CONFIGS[args.config]
    p = phantom.make_pair(shape, h, seed)
    d = tempfile.mkdtemp(prefix="hysco_cli_")
    info = H.hysco_nifti_info()
    n1, n2, n3 = shape                                   # file (nx, ny, nz) = (n2, n3, n1): PE on y
    for k, (n, hh) in enumerate(((n2, h[1]), (n3, h[2]), (n1, h[0]))):
        info.dim[k] = n
        info.pixdim[k] = hh
    info.qfac = 1.0
    for name, img in (("p", p.Ip), ("m", p.Im)):
        H.hysco_nifti_write(os.path.join(d, name + ".nii.gz"), np.ascontiguousarray(img.transpose(0, 2, 1)), info)
    argv = [os.path.join(d, "p.nii.gz"), os.path.join(d, "m.nii.gz"), "--pe-axis", "2", "--out",
            os.path.join(d, "o")]
    import contextlib
    import io
    for _ in range(max(args.warmup, 0)):
        with contextlib.redirect_stdout(io.StringIO()):
            cli.main(argv)
    secs, stages = [], []
    for _ in range(args.steps):
        buf = io.StringIO()
        t0 = time.perf_counter()
        with contextlib.redirect_stdout(buf):
            cli.main(argv)
        secs.append(time.perf_counter() - t0)
        stages.append(json.loads(buf.getvalue().strip().splitlines()[-1])["seconds"])
    last = json.loads(buf.getvalue().strip().splitlines()[-1])
    import subprocess
    t0 = time.perf_counter()                            # like the paper's Linux `time` of the CLI: cold process
    subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli"] + argv, check=True, cwd=ROOT,
                   stdout=subprocess.DEVNULL)
    cold = time.perf_counter() - t0
    line = {"metric": "command-line run time per pair (NIfTI .nii.gz in and out)", "value": float(np.median(secs)),
            "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(secs)), "higher_is_better": False, "scaling": "none",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} as gzip NIfTI, PE along the file's y axis: python -m "
                                   "paper_2403_10706_b200.cli (OT + GN-PCG with the paper's stop rules + Jacobian "
                                   "correction), wall clock in-process (CUDA context already up)"},
            "stage_seconds_median": {k: float(np.median([s[k] for s in stages])) for k in stages[0]},
            "cold_process_s": cold, "paper_run_s_context": {"3T": 10.37, "7T": 13.62, "source": "T3 (RTX A6000)"},
            "report": last["report"],
            "note": "mode line (not the headline); the paper's T3 'Run' column is the same pipeline incl. I/O"}
    print(json.dumps(line), flush=True)


def run_slab(args):
    """Strong scaling of ONE large pair (BASELINE.json configs[4]): rank r owns
    planes slab_bounds(n1, N, r) of dim 1; libhysco exchanges one halo plane and
    allreduces the per-pair scalars over NCCL."""
    import torch
    from paper_2403_10706_b200 import dist as D
    from paper_2403_10706_b200 import hysco as H

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    shape, h, seed = phantom.CONFIGS[args.config]
    n1, n2, n3 = shape
    i0, i1 = D.slab_bounds(n1, world, rank)
    pair = phantom.make_pair(shape, h, seed, planes=(i0, i1))
    nid = D.share_nccl_id() if world > 1 else None
    stream = torch.cuda.current_stream(dev)
    ctx = H.hysco_create_slab((i1 - i0, n2, n3), h, rank, world, n1, i0, nid, device=local,
                              stream=stream.cuda_stream)
    Ip = torch.from_numpy(pair.Ip[None]).to(dev)
    Im = torch.from_numpy(pair.Im[None]).to(dev)
    H.hysco_bind_images(ctx, Ip, Im)
    b = torch.zeros((1, i1 - i0, n2, n3 + 1), dtype=torch.float32, device=dev)
    Tp = torch.zeros((1, i1 - i0, n2, n3), dtype=torch.float32, device=dev)
    Tm = torch.zeros_like(Tp)
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
    so = solve_opts(H, args)
    for _ in range(max(args.warmup, 0)):
        H.hysco_correct(ctx, b, Tp, Tm, solve_opts=so)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    step_ms = []
    launches = 0
    reps = None
    for _ in range(args.steps):
        flush.zero_()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        reps, _ = H.hysco_correct(ctx, b, Tp, Tm, solve_opts=so)
        z.record(stream)
        z.synchronize()
        step_ms.append(a.elapsed_time(z))
        launches += H.hysco_last_launch_count(ctx)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clocks = clk.stop()
    total = D.max_over_ranks(float(np.sum(step_ms)), device=dev)
    value = args.steps / (total / 1e3)
    Nn = n1 * n2 * (n3 + 1)
    # algorithmic bytes of one fixed 10 x 10 solve, streaming kernels
    r0 = reps[0]
    step_bytes = (r0["pcg_iters"] * 60 + r0["f_evals"] * 24 + r0["gn_iters"] * 28 + 40) * Nn
    if rank == 0:
        line = {"metric": "volume pairs corrected/sec (slab-partitioned large pair)", "value": value,
                "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": total / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(workload_desc(args.config, 1, args), parallelism=f"slab{world} along dim 1 (NCCL halo + allreduce)"),
                "clocks": clocks, "gpu_launches": launches,
                "step_effective_gbs_per_gpu": step_bytes / world / (total / args.steps * 1e-3) / 1e9,
                "solver": {k: r0[k] for k in ("gn_iters", "f_evals", "h_evals", "pcg_iters", "stop", "J")}}
        print(json.dumps(line), flush=True)
    H.hysco_destroy(ctx)
    if world > 1:
        torch.distributed.destroy_process_group()


def self_launch(args):
    """`bench.py --gpus N` run without torchrun (no WORLD_SIZE): re-run this
    script under torch.distributed.run with N ranks, one per GPU (the
    contract's launch), and return its exit status."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.stage == "lsq":
        run_lsq(args)
    elif args.stage == "cli":
        run_cli(args)
    elif args.solver == "admm":
        run_admm(args)
    elif args.slab:
        run_slab(args)
    else:
        run_hysco(args)


if __name__ == "__main__":
    main()
