#!/usr/bin/env python
"""Run every kernel on small adversarial inputs against the bounds-checked build
(LC_LIB=build/liblc_bounds.so, -DLC_DEBUG_BOUNDS) and require zero index violations and
bit-exact results vs the oracle.  Used by tests/test_gpu_bounds.py."""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import native as orc
    from oracle import setops
    from paper_2412_10770_b200 import lc
    from synth import CONFIGS, fuzz_case, make_keys

    viol = lc._lib.lc_debug_violations
    viol.restype = ctypes.c_uint32
    dev = "cuda:0"

    def d(a):
        a = np.ascontiguousarray(a)
        return torch.from_numpy(a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)).to(dev)

    def h(t, dt):
        return t.cpu().numpy().view(dt)

    checks = 0

    def check(name, ok):
        nonlocal checks
        v = int(viol())
        if v or not ok:
            where = (ctypes.c_uint32 * 3)()
            lc._lib.lc_debug_where(where)
            raise SystemExit(f"FAIL {name}: violations={v} ok={ok} at lc_kernels.cu line "
                             f"{where[0]} (index {where[1]} >= {where[2]})")
        checks += 1

    rng = np.random.default_rng(0)
    cases = [fuzz_case(s, n_max=60_000) for s in range(7000, 7080)]
    n = 20_000
    k5 = make_keys(5, n)
    for brk in ("all", "every2", "tile"):
        fb = np.zeros(n, np.uint8)
        fb[:: {"all": 1, "every2": 2, "tile": 1024}[brk]] = 1
        cases.append((k5, 127, 64, "adv-" + brk, orc.encode(k5, 127, force_break=fb)))
    # sparse fast path edges: segment starts exactly at quad ends and chunk edges, N a
    # multiple of 128 / 1024 (clamped candidates repeat N)
    for ns in (1024 * 9, 1024 * 9 + 128, 1024 * 9 + 1):
        ks = np.arange(ns, dtype=np.uint64) * np.uint64(5) + np.uint64(11)
        for step in (128, 1024, 256):
            fb = np.zeros(ns, np.uint8)
            fb[(step - 1 if step == 256 else 0)::step] = 1
            cases.append((ks, 2, 64, f"sparse-{ns}-{step}", orc.encode(ks, 2, force_break=fb)))
    # shard views: the slices of one span only
    from paper_2412_10770_b200 import shard as _shard
    kb4 = make_keys(4, 70_001)
    b4 = lc.encode(kb4, 31)
    for r in range(3):
        sv, (i0, i1) = _shard.upload_shard(b4, r, 3, device=dev)
        so, _ = _shard.decode_shard(sv, r, 3)
        check(f"shard {r}/3", np.array_equal(h(so, np.uint64), kb4[i0:i1]))
    for cid in (1, 2, 3, 4):
        keys = make_keys(cid, 70_001)
        cases.append((keys, CONFIGS[cid].eps, CONFIGS[cid].key_bits, f"cfg{cid}"))
    # FORMAT F7 (free intercept): bias 0 and the first-key search of next_geq
    for s in range(7100, 7130):
        keys, eps, kb, law = fuzz_case(s, n_max=60_000)
        eps = min(eps, (1 << 30) - 1)
        cases.append((keys, eps, kb, "free-" + law, lc.encode(keys, eps, kb, free=True)))
    for cid in (1, 2, 4, 5):
        keys = make_keys(cid, 70_001)
        cases.append((keys, CONFIGS[cid].eps, CONFIGS[cid].key_bits, f"free-cfg{cid}",
                      lc.encode(keys, CONFIGS[cid].eps, free=True)))
    for case in cases:
        keys, eps, kb, law = case[:4]
        blob = case[4] if len(case) > 4 else lc.encode(keys, eps, kb)
        view = lc.View(blob, device=dev)
        out = lc.decode(view)
        check(f"decode {law}", np.array_equal(h(out, keys.dtype), keys))
        idx = rng.integers(0, keys.size, 3000).astype(np.uint64)
        check(f"access {law}", np.array_equal(h(lc.access(view, d(idx)), keys.dtype), keys[idx.astype(np.int64)]))
        for length in (1, 33, 64, 100):
            if keys.size >= length:
                st = rng.integers(0, keys.size - length, 500, endpoint=True).astype(np.uint64)
                want, _ = orc.range_decode(blob, st, length)
                check(f"range{length} {law}", np.array_equal(h(lc.range_decode(view, d(st), length), keys.dtype), want))
        ranks = rng.integers(0, 1000, 500, endpoint=True).astype(np.uint64)
        qi = np.array([orc.quantile_index(keys.size, int(k), 1000) for k in ranks], np.uint64)
        check(f"quantile {law}", np.array_equal(h(lc.quantile(view, d(ranks), 1000), keys.dtype), keys[qi.astype(np.int64)]))
        wa, _ = orc.predict(blob, qi)
        check(f"quantile-approx {law}", np.array_equal(h(lc.quantile(view, d(ranks), 1000, exact=False), keys.dtype), wa))
        x = np.concatenate([keys[rng.integers(0, keys.size, 500)].astype(np.uint64),
                            rng.integers(0, (1 << 63), 500, dtype=np.uint64)])
        gi, gk = lc.next_geq(view, d(x))
        wi, wk = setops.next_geq(keys, x)
        check(f"next_geq {law}", np.array_equal(h(gi, np.uint64), wi) and np.array_equal(h(gk, keys.dtype), wk))
        # the same lookups and 64-key ranges through the access layout (directory + records)
        view.build_access_layout()
        check(f"access-layout {law}", np.array_equal(h(lc.access(view, d(idx)), keys.dtype), keys[idx.astype(np.int64)]))
        if keys.size >= 64:
            st = np.concatenate([rng.integers(0, keys.size - 64, 500, endpoint=True),
                                 [0, keys.size - 64]]).astype(np.uint64)
            want, _ = orc.range_decode(blob, st, 64)
            check(f"range64-layout {law}", np.array_equal(h(lc.range_decode(view, d(st), 64), keys.dtype), want))
    a = np.unique(np.concatenate([k5[::3], rng.integers(0, int(k5[-1]), 5000, dtype=np.uint64)]))
    va, vb = lc.View(lc.encode(a, 31), device=dev), lc.View(lc.encode(k5, 127), device=dev)
    out, cnt = lc.intersect(va, vb)
    c = int(cnt.item())
    check("intersect", np.array_equal(h(out[:c], np.uint64), setops.intersect(a, k5)))
    out, cnt = lc.union(va, vb)
    c = int(cnt.item())
    check("union", np.array_equal(h(out[:c], np.uint64), setops.union(a, k5)))
    vf = lc.View(lc.encode(k5, 127, free=True), device=dev)
    out, cnt = lc.intersect(va, vf)
    c = int(cnt.item())
    check("intersect-free", np.array_equal(h(out[:c], np.uint64), setops.intersect(a, k5)))
    out, cnt = lc.union(va, vf)
    c = int(cnt.item())
    check("union-free", np.array_equal(h(out[:c], np.uint64), setops.union(a, k5)))
    # fused union with > 32 insertions per window (streamed batches) and equal ranks
    lo = int(k5[7 * 1024])
    cl = np.unique(np.concatenate([rng.integers(lo, lo + 40_000, 3000).astype(np.uint64),
                                   k5[-1] + np.arange(1, 40, dtype=np.uint64)]))
    vc = lc.View(lc.encode(cl, 7), device=dev)
    out, cnt = lc.union(vc, vb)
    c = int(cnt.item())
    check("union-clustered", np.array_equal(h(out[:c], np.uint64), setops.union(cl, k5)))
    # the same through the successor-search index (anchored and F7 long lists)
    for vv, nm in ((vb, "idx"), (vf, "idx-free")):
        vv.build_search_index()
        xs = np.concatenate([k5[rng.integers(0, k5.size, 3000)],
                             rng.integers(0, int(k5[-1]) + 100, 3000, dtype=np.uint64)])
        gi, gk = lc.next_geq(vv, d(xs))
        wi, wk = setops.next_geq(k5, xs)
        check(f"next_geq-{nm}", np.array_equal(h(gi, np.uint64), wi) and np.array_equal(h(gk, np.uint64), wk))
        out, cnt = lc.intersect(va, vv)
        c = int(cnt.item())
        check(f"intersect-{nm}", np.array_equal(h(out[:c], np.uint64), setops.intersect(a, k5)))
        out, cnt = lc.union(vc, vv)
        c = int(cnt.item())
        check(f"union-{nm}", np.array_equal(h(out[:c], np.uint64), setops.union(cl, k5)))
    print(f"bounds check ok: {checks} checks, 0 violations")


if __name__ == "__main__":
    main()
