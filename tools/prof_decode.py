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
    ap.add_argument("--no-check", action="store_true", help="experiment builds (LC_LIB)")
    ap.add_argument("--cache", default=None, help="directory to keep keys + blob between runs (A/B)")
    args = ap.parse_args()
    import torch

    from paper_2412_10770_b200 import lc
    from synth import CONFIGS, make_keys, make_queries

    spec = CONFIGS[args.config]
    t0 = time.time()
    if args.access:
        keys, idx, rs = make_queries(n=args.n)
        blob = lc.encode(keys, spec.eps)
    else:
        ck = args.cache and os.path.join(args.cache, f"lc_c{args.config}_{args.n}.npy")
        if ck and os.path.exists(ck) and os.path.exists(ck + ".blob"):
            keys = np.load(ck)
            blob = open(ck + ".blob", "rb").read()
        else:
            keys = make_keys(args.config, args.n)
            blob = lc.encode(keys, spec.eps)
            if ck:
                np.save(ck, keys)
                open(ck + ".blob", "wb").write(blob)
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
            ev[0].record()
            lc.access(view, d_idx, a_out)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            print(f"access rep {r}: {ms:.4f} ms  {idx.size / ms / 1e6:.3e} lookups/s", flush=True)
            ev[0].record()
            lc.range_decode(view, d_rs, 64, r_out)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            print(f"range rep {r}: {ms:.4f} ms  {rs.size / ms / 1e6:.3e} ranges/s", flush=True)
    ref = torch.from_numpy(keys.view(np.int64) if keys.itemsize == 8 else keys.view(np.int32)).cuda()
    assert args.no_check or torch.equal(out, ref), "decode mismatch"
    if args.access and not args.no_check:
        assert torch.equal(a_out, ref[d_idx]), "access mismatch"
        sel = (d_rs[:, None] + torch.arange(64, device="cuda")[None, :]).reshape(-1)
        assert torch.equal(r_out, ref[sel]), "range mismatch"
    print("ok", flush=True)


if __name__ == "__main__":
    main()
