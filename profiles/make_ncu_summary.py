#!/usr/bin/env python
"""Build profiles/ncu_summary.json (read by bench.py's roofline) from
`ncu --set full` summaries made by summarize_ncu.py, one per workload config.

usage: python profiles/make_ncu_summary.py C2_hcp3t=profiles/ncu_r2b_3t.json [C3_hcp7t=...] ...

Per config and kernel (bench.py's names), the mean over the captured launches
of: time, DRAM bytes read + written, DRAM / SM throughput (% of peak), FP32
pipe utilisation where captured, registers, top stalls.
"""
import json
import os
import sys

NAMES = {"pcg_resident_kernel": "pcg_resident", "eval_kernel": "eval", "matvec_kernel": "matvec",
         "pcg_update_kernel": "pcg_update", "pcg_dir_kernel": "pcg_dir", "trial_init_kernel": "trial_init",
         "pcg_mvdir_kernel": "pcg_mvdir", "pcg_sync_floor_kernel": "resident_sync_floor",
         "pcg_march_kernel": "pcg_dirmv", "pcg_upd_kernel": "pcg_upd", "trial_flat_kernel": "trial_init",
         "pcg_init_flat_kernel": "pcg_init"}


def mean(v):
    v = [x for x in v if isinstance(x, (int, float))]
    return sum(v) / len(v) if v else None


def main(args):
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_summary.json")
    out = {"configs": {}, "note": __doc__.strip().splitlines()[0]}
    for a in args:
        cfg, paths = a.split("=", 1)
        ent = out["configs"].setdefault(cfg, {})
        for path in paths.split("+"):     # later files win for kernels in several
          src = json.load(open(path))
          for short, launches in src["kernels"].items():
            name = NAMES.get(short)
            if not name:
                continue
            # skip no-op launches (finished pairs exit at once): keep the longer half
            ls = sorted(launches, key=lambda e: -e.get("time_us", 0))[: max(1, (len(launches) + 1) // 2)]
            ent[name] = {
                "launches_averaged": len(ls),
                "time_us": mean([e.get("time_us") for e in ls]),
                "dram_bytes_per_launch": mean([e.get("dram_bytes_per_launch") for e in ls]),
                "dram_pct_peak": mean([e.get("dram_pct_peak") for e in ls]),
                "sm_throughput_pct": mean([e.get("sm_throughput_pct") for e in ls]),
                "regs_per_thread": ls[0].get("regs_per_thread"),
                "warps_active_pct": mean([e.get("warps_active_pct") for e in ls]),
                "inst_executed": mean([e.get("inst_executed") for e in ls]),
                "top_stalls": dict(list(ls[0].get("stall_share", {}).items())[:4]),
                "source": path,
            }
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1:])
