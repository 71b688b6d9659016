#!/usr/bin/env python
"""SASS of one kernel in an ncu report with executed warp-instructions per instruction (per
`--unit` work items) and stall samples: where a kernel's instruction budget goes.

  python tools/ncu_sass.py gpurun_out/x.ncu-rep --unit 1e7 [--min 0.5]
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--unit", type=float, default=1.0, help="divide executions by this")
    ap.add_argument("--min", type=float, default=0.0, help="hide instructions below this")
    ap.add_argument("--kernel", default=None, help="substring of the kernel name to select")
    ap.add_argument("--skip", type=int, default=0, help="matching kernel blocks to skip")
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"]
    out = subprocess.check_output(cmd, text=True)
    rows = list(csv.reader(io.StringIO(out)))
    # one block per kernel: a "Kernel Name" row, then the header and the SASS rows
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    blocks = [(rows[i][1], rows[i:(starts[k + 1] if k + 1 < len(starts) else len(rows))])
              for k, i in enumerate(starts)] or [("", rows)]
    sel = [b for name, b in blocks if not args.kernel or args.kernel in name]
    rows = sel[min(args.skip, len(sel) - 1)]
    hdr = next(r for r in rows if "Instructions Executed" in r)
    ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    total = 0
    lines = []
    for r in rows[rows.index(hdr) + 1:]:
        try:
            n = int(r[ie])
        except (ValueError, IndexError):
            continue
        total += n
        lines.append((r[0][-5:], n / args.unit, int(r[st] or 0), r[1].strip()))
    print(f"total {total} = {total / args.unit:.2f} per unit")
    for a, n, s, ins in lines:
        if n >= args.min:
            print(f"{a} {n:7.2f} {s:6d}  {ins[:80]}")


if __name__ == "__main__":
    main()
