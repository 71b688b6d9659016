#!/usr/bin/env python
"""The posting-list corpus (synth/corpus.py: 1e5 lists, Zipf-like lengths 10..1e6, per-list
eps): one lc_decode_batch launch vs one lc_decode launch per list.  GB/s counts the lists'
payload bytes (header + sections, no alignment padding) read once plus the keys written once."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_corpus
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--per-list", type=int, default=2000, help="lists timed one launch each")
    ap.add_argument("--only-class", default=None, help="time only this length class (for ncu)")
    args = ap.parse_args()
    dev = "cuda:0"
    t0 = time.perf_counter()
    lists, eps, pairs = make_corpus()
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    t_enc = time.perf_counter() - t0
    if args.only_class:
        sizes = np.array([x.size for x in lists])
        lo, hi = {"small": (0, 64), "mid": (65, 1023), "big": (1024, 1 << 40)}[args.only_class]
        idx = np.flatnonzero((sizes >= lo) & (sizes <= hi))
        sb = lc.Batch([blobs[i] for i in idx], device=dev)
        so = lc.decode_batch(sb)
        torch.cuda.synchronize()
        want = torch.from_numpy(np.concatenate([lists[i] for i in idx]).view(np.int32)).to(dev)
        assert torch.equal(so[:want.numel()], want)
        print(json.dumps({"class": args.only_class, "lists": int(idx.size)}))
        return
    bt = lc.Batch(blobs, device=dev)
    out = lc.decode_batch(bt)
    want = torch.from_numpy(np.concatenate(lists).view(np.int32)).to(dev)
    torch.cuda.synchronize()
    assert torch.equal(out[:want.numel()], want)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.reps + 1)]
    for _ in range(3):
        lc.decode_batch(bt, out)
    torch.cuda.synchronize()
    ev[0].record()
    for k in range(args.reps):
        lc.decode_batch(bt, out)
        ev[k + 1].record()
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.reps)]
    ms = statistics.median(per)
    alg = bt.b.payload_bytes + bt.n_total * 4
    res = {"lists": bt.b.m, "keys": bt.n_total, "chunks": int(bt.b.n_chunks),
           "payload_bytes": int(bt.b.payload_bytes), "blob_bytes": int(sum(len(b) for b in blobs)),
           "bits_per_int_payload": 8 * bt.b.payload_bytes / bt.n_total,
           "batch_ms": ms, "batch_GBps": alg / ms / 1e6, "batch_keys_per_s": bt.n_total / ms * 1e3,
           "gen_s": t_gen, "encode_s": t_enc, "sparse": int(bt.b.sparse),
           "max_res_bits": int(bt.b.max_res_bits)}
    # where the time goes: the corpus cut by list length, each class one batch
    sizes = np.array([x.size for x in lists])
    res["classes"] = {}
    for name, lo, hi in (("n<=64", 0, 64), ("64<n<1024", 65, 1023), ("n>=1024", 1024, 1 << 40)):
        idx = np.flatnonzero((sizes >= lo) & (sizes <= hi))
        sb = lc.Batch([blobs[i] for i in idx], device=dev)
        so = lc.decode_batch(sb)
        for _ in range(3):
            lc.decode_batch(sb, so)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            lc.decode_batch(sb, so)
        e1.record()
        torch.cuda.synchronize()
        cms = e0.elapsed_time(e1) / args.reps
        calg = sb.b.payload_bytes + sb.n_total * 4
        res["classes"][name] = {"lists": int(idx.size), "keys": sb.n_total, "ms": cms,
                                "GBps": calg / cms / 1e6, "chunks": int(sb.b.n_chunks),
                                "small": int(sb.b.n_small)}
        del sb, so
    # one launch per list (the same kernels through lc_decode) for the first per_list lists
    k = min(args.per_list, len(blobs))
    views = [lc.View(b, device=dev) for b in blobs[:k]]
    outs = [v.out_tensor(v.n) for v in views]
    for v, o in zip(views, outs):
        lc.decode(v, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for v, o in zip(views, outs):
        lc.decode(v, o)
    e1.record()
    torch.cuda.synchronize()
    nk = sum(x.size for x in lists[:k])
    res["per_list_launch"] = {"lists": k, "keys": nk, "ms": e0.elapsed_time(e1),
                              "keys_per_s": nk / e0.elapsed_time(e1) * 1e3}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
