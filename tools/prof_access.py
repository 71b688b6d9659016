#!/usr/bin/env python
"""Config-5 random access with and without the access layout (lc_access_layout_build):
1e8 uniform lookups, exact and approximate quantiles; prints ms per launch (CUDA events, median
of R) and checks results on device.  `--only layout|plain` runs one variant (for ncu)."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_queries
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", choices=["layout", "plain"], default=None)
    args = ap.parse_args()
    dev = "cuda:0"
    keys, idx, rs = make_queries()
    d_rs = torch.from_numpy(rs.view(np.int64)).to("cuda:0")
    r_out = torch.empty(rs.size * 64, dtype=torch.int64, device="cuda:0")
    blob = lc.encode(keys, 127)
    v = lc.View(blob, device=dev)
    d_idx = torch.from_numpy(idx.view(np.int64)).to(dev)
    out = torch.empty(idx.size, dtype=torch.int64, device=dev)
    d_keys = torch.from_numpy(keys.view(np.int64)).to(dev)
    res = {}

    def timeit(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record()
        for k in range(reps):
            fn()
            ev[k + 1].record()
        torch.cuda.synchronize()
        return statistics.median(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))

    if args.only != "layout":
        ms = timeit(lambda: lc.access(v, d_idx, out), args.reps)
        assert torch.equal(out, d_keys[d_idx])
        res["plain_ms"] = ms
        res["plain_lookups_per_s"] = idx.size / ms * 1e3
        res["plain_range64_ms"] = timeit(lambda: lc.range_decode(v, d_rs, 64, r_out), args.reps)
    if args.only != "plain":
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        lay = v.build_access_layout()
        t0.record()
        v.build_access_layout(out=lay)
        t1.record()
        torch.cuda.synchronize()
        res["layout_bytes"] = v.access_layout_bytes()
        res["blob_bytes"] = len(blob)
        res["layout_build_ms"] = t0.elapsed_time(t1)
        out.zero_()
        ms = timeit(lambda: lc.access(v, d_idx, out), args.reps)
        assert torch.equal(out, d_keys[d_idx])
        res["layout_ms"] = ms
        res["layout_lookups_per_s"] = idx.size / ms * 1e3
        res["layout_range64_ms"] = timeit(lambda: lc.range_decode(v, d_rs, 64, r_out), args.reps)
        sel = (d_rs[:, None] + torch.arange(64, device=dev)[None, :]).reshape(-1)
        assert torch.equal(r_out, d_keys[sel])
        del sel
        res["layout_ranges_per_s"] = rs.size / res["layout_range64_ms"] * 1e3
        ranks = d_idx[:10_000_000]
        qo = torch.empty(ranks.numel(), dtype=torch.int64, device=dev)
        res["quantile_exact_layout_ms_1e7"] = timeit(
            lambda: lc.quantile(v, ranks, keys.size, True, qo), args.reps)
        assert torch.equal(qo, d_keys[ranks])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
