#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) for profiles/: key throughput, traffic,
occupancy and stall metrics per kernel, plus the hottest SASS lines.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--out profiles/x.txt] [--json key]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__inst_executed_pipe_tma.sum", "smsp__inst_executed_op_ldsm.sum",
]


def ncu_csv(rep: str, page: str, extra=()):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                                  text=True, stderr=subprocess.DEVNULL)
    return list(csv.reader(io.StringIO(out)))


def summarise(rep: str):
    rows = ncu_csv(rep, "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for v in data:
        k = {"kernel": v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                k[m] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, name in enumerate(hdr):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                try:
                    val = float(v[i])
                except ValueError:
                    continue
                if val > 0:
                    stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = val
        k["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        try:
            rd = float(v[hdr.index("dram__bytes_read.sum")])
            wr = float(v[hdr.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            k["dram_bytes"] = rd * scale[units[hdr.index("dram__bytes_read.sum")]] + \
                wr * scale[units[hdr.index("dram__bytes_write.sum")]]
        except (ValueError, KeyError):
            pass
        kernels.append(k)
    hot = []
    try:
        src = ncu_csv(rep, "source", ["--print-source", "sass"])
        h2, d2 = src[1], src[2:]
        si, ie, sa = h2.index("Source"), h2.index("Instructions Executed"), \
            h2.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(r[sa]) for r in d2 if r[sa].isdigit()) or 1
        for r in sorted(d2, key=lambda r: -int(r[sa]) if r[sa].isdigit() else 0)[:12]:
            hot.append(f"{100 * int(r[sa]) / tot:5.1f}%  exec={r[ie]:>9}  {r[si].strip()}")
    except Exception:
        pass
    return kernels, hot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out")
    ap.add_argument("--title", default="")
    ap.add_argument("--json", help="update profiles/ncu_traffic.json[key] with dram bytes/launch")
    args = ap.parse_args()
    kernels, hot = summarise(args.rep)
    lines = [f"# ncu --set full summary: {args.title or os.path.basename(args.rep)}", ""]
    for k in kernels:
        lines.append(f"kernel: {k['kernel']}")
        for m in METRICS:
            if m in k:
                lines.append(f"  {m:60s} {k[m]}")
        if "dram_bytes" in k:
            lines.append(f"  {'dram bytes read+write per launch':60s} {k['dram_bytes']:.0f}")
        lines.append("  top stall reasons (pc samples): " +
                     ", ".join(f"{a}={b:.0f}" for a, b in k["stall_samples"].items()))
        lines.append("")
    if hot:
        lines.append("hottest SASS (share of stall samples):")
        lines += ["  " + h for h in hot]
    text = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    print(text)
    if args.json and kernels and "dram_bytes" in kernels[0]:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "profiles", "ncu_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[args.json] = kernels[0]["dram_bytes"]
        json.dump(d, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
