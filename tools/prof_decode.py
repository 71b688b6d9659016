#!/usr/bin/env python
"""Run the decode (and optionally access / range) kernels a few times on one config for ncu.

  python tools/prof_decode.py --config 2 --reps 5 [--access]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--access", action="store_true")
    args = ap.parse_args()
    import torch

    from paper_2412_10770_b200 import lc
    from synth import CONFIGS, make_keys, make_queries

    spec = CONFIGS[args.config]
    t0 = time.time()
    if args.access:
        keys, idx, rs = make_queries(n=args.n)
    else:
        keys = make_keys(args.config, args.n)
    blob = lc.encode(keys, spec.eps)
    print(f"gen+encode {time.time() - t0:.1f}s n={keys.size} blob={len(blob)}", flush=True)
    view = lc.View(blob)
    out = view.out_tensor(keys.size)
    if args.access:
        d_idx = torch.from_numpy(idx.view(np.int64)).cuda()
        d_rs = torch.from_numpy(rs.view(np.int64)).cuda()
        a_out = torch.empty(idx.size, dtype=torch.int64, device="cuda")
        r_out = torch.empty(rs.size * 64, dtype=torch.int64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(args.reps):
        ev[0].record()
        lc.decode(view, out)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1])
        gbs = (len(blob) + keys.size * keys.itemsize) / ms / 1e6
        print(f"decode rep {r}: {ms:.4f} ms  {gbs:.1f} GB/s", flush=True)
        if args.access:
            lc.access(view, d_idx, a_out)
            lc.range_decode(view, d_rs, 64, r_out)
    ref = torch.from_numpy(keys.view(np.int64) if keys.itemsize == 8 else keys.view(np.int32)).cuda()
    assert torch.equal(out, ref), "decode mismatch"
    print("ok", flush=True)


if __name__ == "__main__":
    main()
