#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

usage:
  python profiles/summarize_ncu.py full  gpurun_out/prof.ncu-rep  profiles/ncu_<tag>.json
  python profiles/summarize_ncu.py launches gpurun_out/launches.csv profiles/launches_<tag>.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_bytes": "lts__t_bytes.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs_per_thread": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
}
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "lg_throttle", "mio_throttle", "barrier", "membar",
          "math_pipe_throttle", "not_selected", "selected", "no_instruction", "dispatch_stall", "drain",
          "imc_miss", "branch_resolving", "sleeping", "tex_throttle"]


def units_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
            "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(u, 1)


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {"report": rep, "kernels": {}}
    for d in data:
        name = d[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        e = {"name": name}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    v = d[i]
                if isinstance(v, float) and k.endswith("bytes"):
                    v *= units_scale(units[i])
                if isinstance(v, float) and k == "time_us":
                    v *= units_scale(units[i])
                e[k] = v
        st = {}
        for s in STALLS:
            m = "smsp__pcsamp_warps_issue_stalled_" + s
            if m in hdr:
                try:
                    st[s] = float(d[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        e["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v > 0}
        if "dram_read_bytes" in e and "time_us" in e and isinstance(e["time_us"], float):
            e["dram_bytes_per_launch"] = e["dram_read_bytes"] + e.get("dram_write_bytes", 0.0)
            e["dram_GBps"] = e["dram_bytes_per_launch"] / (e["time_us"] * 1e-6) / 1e9
        res["kernels"].setdefault(short, []).append(e)
    # one representative (the longest) per kernel for bench.py's "traffic"
    res["summary"] = {k: max(v, key=lambda e: e.get("time_us", 0)) for k, v in res["kernels"].items()}
    json.dump(res, open(out, "w"), indent=1)
    for k, e in res["summary"].items():
        print(f"{k:22s} {e.get('time_us', 0):8.2f} us  DRAM {e.get('dram_bytes_per_launch', 0) / 1e6:7.2f} MB "
              f"({e.get('dram_GBps', 0):7.1f} GB/s, {e.get('dram_pct_peak', 0)}%)  regs {e.get('regs_per_thread')} "
              f"warps {e.get('warps_active_pct')}%  top stalls {list(e['stall_share'].items())[:3]}")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[h0 + 1:]:
        if len(r) != len(hdr):
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        t = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0 if r[ui] in ("us", "usecond") else 1e3)
        a = agg.setdefault(name, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += t
    tot = sum(a["total_us"] for a in agg.values())
    for a in agg.values():
        a["share"] = a["total_us"] / tot
        a["avg_us"] = a["total_us"] / a["launches"]
    json.dump({"source": path, "kernels": agg, "total_us": tot}, open(out, "w"), indent=1)
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]):
        print(f"{k:30s} n={a['launches']:5d} avg {a['avg_us']:8.2f} us share {a['share'] * 100:5.1f}%")


def merge(out, *summaries):
    """profiles/ncu_summary.json: per kernel, the latest capture's DRAM bytes per
    launch (bench.py's roofline `traffic`), time and source report."""
    res = {"kernels": {}}
    for path in summaries:
        d = json.load(open(path))
        for k, e in d["summary"].items():
            res["kernels"][k[:-7] if k.endswith("_kernel") else k] = {"dram_bytes_per_launch": e.get("dram_bytes_per_launch"),
                                 "time_us": e.get("time_us"), "dram_GBps": e.get("dram_GBps"),
                                 "source": path}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "merge":
        merge(sys.argv[2], *sys.argv[3:])
    else:
        {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
