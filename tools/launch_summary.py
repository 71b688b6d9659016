#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of bench.py."""
from __future__ import annotations

import csv
import sys
from collections import defaultdict


def main(path: str, out: str, alg_bytes: float = 4396297936.0, steps: int = 5, warmup: int = 3,
         raw: str = "r02_launches_bench.csv"):
    """alg_bytes: algorithmic bytes of one headline decode (config 4 = blob + 5e8 x 8 B)."""
    rows = list(csv.reader(open(path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
                recs.append((int(d["ID"]), d["Kernel Name"], float(d["Metric Value"]) * scale))
    dec = [t for _, k, t in recs if "lc_decode_kernel" in k]
    full, spans = dec[: warmup + steps], dec[warmup + steps:]
    timed = full[warmup:]
    mean = sum(timed) / len(timed)
    lines = [
        f"# ncu launch list of `python bench.py --steps {steps} --warmup {warmup} --no-cpu`",
        "# (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)",
        f"total kernels launched: {len(recs)} (raw list: {raw})",
        f"lc_decode_kernel full-list launches ({warmup} warm-up + {steps} timed): "
        + ", ".join(f"{t:.1f} us" for t in full),
        f"  mean of the timed launches: {mean:.1f} us -> {alg_bytes / (mean * 1e-6) / 1e9:.0f} GB/s "
        f"algorithmic ({alg_bytes:.0f} B per launch)",
        f"other lc_decode_kernel launches (e2e spans, intersect/union decodes): {len(spans)}, "
        f"mean {sum(spans) / max(len(spans), 1):.1f} us",
        "a bench step is exactly one lc_decode_kernel launch (100% of the timed region); torch",
        "kernels (compare/index) are the post-timing bit-exact checks, outside the timed region;",
        "the other lc_* kernels are the decode_configs / F7 / corpus / access blocks of the line.",
        "",
        "per-kernel totals (count, total us):",
    ]
    agg = defaultdict(lambda: [0, 0.0])
    for _, k, t in recs:
        agg[k[:100]][0] += 1
        agg[k[:100]][1] += t
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"  {n:4d} {t:10.1f}  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(float(x) for x in sys.argv[3:4]))
