#!/usr/bin/env python
"""A small run of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
dense and sparse full decode (TMA + mbarrier page reuse), union's shifted decode, range64's
cp.async ring, access with and without the access layout, quantiles, next_geq, intersect, the
batch decode (work queue, flattened small keys) and a batched AND / OR, shard views.  Results
are checked against the generators' keys so a clean sanitizer run is also a correct run.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import setops
    from paper_2412_10770_b200 import lc, shard
    from synth import make_corpus, make_keys

    dev = "cuda:0"

    def d(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64 if a.dtype.itemsize == 8 else np.int32)).to(dev)

    ok = True
    for cid, eps in ((2, 127), (4, 31), (3, 255)):
        keys = make_keys(cid, 150_001)
        blob = lc.encode(keys, eps)
        v = lc.View(blob, device=dev)
        out = lc.decode(v)
        ok &= bool(torch.equal(out, d(keys)))
        rng = np.random.default_rng(cid)
        idx = rng.integers(0, keys.size, 5000).astype(np.uint64)
        ok &= np.array_equal(lc.access(v, d(idx)).cpu().numpy().view(np.uint64), keys[idx.astype(np.int64)])
        st = rng.integers(0, keys.size - 64, 2000).astype(np.uint64)
        rg = lc.range_decode(v, d(st), 64).cpu().numpy().view(np.uint64)
        ok &= np.array_equal(rg, keys[st.astype(np.int64)[:, None] + np.arange(64)])
        v.build_access_layout()
        ok &= np.array_equal(lc.access(v, d(idx)).cpu().numpy().view(np.uint64), keys[idx.astype(np.int64)])
        sv, (i0, i1) = shard.upload_shard(blob, 1, 3, device=dev)
        so, _ = shard.decode_shard(sv, 1, 3)
        ok &= np.array_equal(so.cpu().numpy().view(np.uint64), keys[i0:i1])
        short = np.unique(np.concatenate([keys[::13], rng.integers(0, int(keys[-1]), 3000, dtype=np.uint64)]))
        vs = lc.View(lc.encode(short, 63), device=dev)
        io, ic = lc.intersect(vs, v)
        uo, uc = lc.union(vs, v)
        wi, wu = setops.intersect(short, keys), setops.union(short, keys)
        ok &= int(ic.item()) == wi.size and np.array_equal(io[:wi.size].cpu().numpy().view(np.uint64), wi)
        ok &= int(uc.item()) == wu.size and np.array_equal(uo[:wu.size].cpu().numpy().view(np.uint64), wu)
    lists, eps, pairs = make_corpus(m=400, seed=21, n_max=20_000, pairs=100)
    bt = lc.Batch([lc.encode(k, e) for k, e in zip(lists, eps)], device=dev)
    out = lc.decode_batch(bt)
    ok &= bool(torch.equal(out[:bt.n_total], torch.from_numpy(np.concatenate(lists).view(np.int32)).to(dev)))
    ia = lc.intersect_batch(bt, pairs)
    ua = lc.union_batch(bt, pairs)
    torch.cuda.synchronize()
    for r, fn in ((ia, setops.intersect), (ua, setops.union)):
        o, c, x = r.out_off.cpu().numpy(), r.counts.cpu().numpy(), r.out.cpu().numpy().view(np.uint32)
        for p, (a, b) in enumerate(pairs):
            w = fn(lists[a], lists[b])
            ok &= c[p] == w.size and np.array_equal(x[o[p]:o[p] + c[p]], w)
    torch.cuda.synchronize()
    print("sanitize run", "ok" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
