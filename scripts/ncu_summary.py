#!/usr/bin/env python
"""Summarise an ncu launch list (CSV, gpu__time_duration.sum) and an `ncu --set full`
report into profiles/: per-kernel share of the step and the key metrics of the captured
kernels.  Usage:
  python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
      --rep gpurun_out/prof_mlp.ncu-rep --tag r1_c2 [--traffic-config c2 --traffic-kernel k_mlp_fp32<64, 3, 1>]
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        a = agg.setdefault(r[ki], [0.0, 0])
        a[0] += v
        a[1] += 1
    tot = sum(a[0] for a in agg.values())
    return [{"kernel": k, "total_us": v, "launches": c, "avg_us": v / c, "share": v / tot}
            for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0])]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--traffic-config")
    ap.add_argument("--traffic-kernel")
    a = ap.parse_args()
    os.makedirs("profiles", exist_ok=True)
    out = {"tag": a.tag}
    if a.launches:
        out["launch_list"] = launches(a.launches)
    if a.rep:
        out["ncu_full"] = report(a.rep)
    with open(f"profiles/{a.tag}.json", "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# ncu summary {a.tag}", ""]
    if a.launches:
        lines += ["## launch list (cold-cache, serialised; compare shares)", "",
                  "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for x in out["launch_list"]:
            lines.append(f"| `{x['kernel'][:90]}` | {x['launches']} | {x['avg_us']:.1f} | {100 * x['share']:.1f}% |")
    if a.rep:
        lines += ["", "## ncu --set full", ""]
        for d in out["ncu_full"]:
            lines.append(f"### `{d['kernel']}`")
            for k in KEYS:
                if k in d:
                    lines.append(f"- {k}: {d[k]}")
    open(f"profiles/{a.tag}.md", "w").write("\n".join(lines) + "\n")
    if a.traffic_config and a.rep:
        for d in out["ncu_full"]:
            if a.traffic_kernel in d["kernel"]:
                def b(s):
                    v, u = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "byte")
                    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                tr = b(d["dram__bytes_read.sum"]) + b(d["dram__bytes_write.sum"])
                json.dump({"kernel": d["kernel"], "bytes_per_launch": tr, "source": f"profiles/{a.tag}.json"},
                          open(f"profiles/traffic_{a.traffic_config}.json", "w"), indent=1)
    print(open(f"profiles/{a.tag}.md").read())


if __name__ == "__main__":
    main()
