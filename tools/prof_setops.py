#!/usr/bin/env python
"""Time next_geq / intersect / union on config 5 (as in bench.py) for A/B runs (LC_LIB)."""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_keys

    k5 = make_keys(5)
    v5 = lc.View(lc.encode(k5, 127))
    rng = np.random.default_rng(55)
    probes = rng.integers(0, int(k5[-1]), 10_000_000, dtype=np.uint64)
    d_probe = torch.from_numpy(probes.view(np.int64)).cuda()
    na = 1_000_000
    a = np.unique(np.concatenate([k5[np.sort(rng.choice(k5.size, na // 2, replace=False))],
                                  rng.integers(0, int(k5[-1]), na // 2, dtype=np.uint64)]))
    va = lc.View(lc.encode(a, 127))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def t(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            ev[0].record()
            fn()
            ev[1].record()
            torch.cuda.synchronize()
            best = min(best, ev[0].elapsed_time(ev[1]))
        return best

    ranks = torch.from_numpy(rng.integers(0, (1 << 32) - 1, 10_000_000, endpoint=True)
                             .astype(np.uint64).view(np.int64)).cuda()
    qo = torch.empty(ranks.numel(), dtype=torch.int64, device="cuda")
    for exact in (True, False):
        ms = t(lambda: lc.quantile(v5, ranks, (1 << 32) - 1, exact, qo))
        print(f"quantile exact={exact} {ms:.3f} ms {ranks.numel() / ms * 1e3:.3e} per s")
    gi, gk = lc.next_geq(v5, d_probe)
    want = np.searchsorted(k5, probes, side="left")
    assert np.array_equal(gi.cpu().numpy(), want.astype(np.int64)), "next_geq mismatch"
    ms = t(lambda: lc.next_geq(v5, d_probe, gi, gk))
    print(f"next_geq {ms:.3f} ms {probes.size / ms / 1e6:.3e} probes/s")
    out, cnt = lc.intersect(va, v5)
    ms = t(lambda: lc.intersect(va, v5, out=out, count=cnt))
    print(f"intersect {ms:.4f} ms count {int(cnt.item())}")
    uo, uc = lc.union(va, v5)
    want_u = np.union1d(a, k5)
    assert int(uc.item()) == want_u.size, "union count mismatch"
    assert np.array_equal(uo[:want_u.size].cpu().numpy().view(np.uint64), want_u), "union mismatch"
    scr = torch.empty(lc.union_scratch_bytes(va, v5), dtype=torch.uint8, device="cuda")
    ms = t(lambda: lc.union(va, v5, scr, uo, uc))
    print(f"union {ms:.4f} ms keys_out {int(uc.item())}")
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_b[0].record()
    v5.build_search_index()
    ev_b[1].record()
    torch.cuda.synchronize()
    print(f"search index build {ev_b[0].elapsed_time(ev_b[1]):.4f} ms ({v5.d_first.numel() * 8 / 1e6:.1f} MB)")
    gi2, gk2 = lc.next_geq(v5, d_probe)
    assert torch.equal(gi2, gi) and torch.equal(gk2, gk), "indexed next_geq mismatch"
    ms = t(lambda: lc.next_geq(v5, d_probe, gi, gk))
    print(f"next_geq+index {ms:.3f} ms {probes.size / ms / 1e6:.3e} probes/s")
    ms = t(lambda: lc.intersect(va, v5, out=out, count=cnt))
    print(f"intersect+index {ms:.4f} ms count {int(cnt.item())}")
    ms = t(lambda: lc.union(va, v5, scr, uo, uc))
    print(f"union+index {ms:.4f} ms keys_out {int(uc.item())}")
    assert np.array_equal(uo[:want_u.size].cpu().numpy().view(np.uint64), want_u), "union mismatch"
    v5f = lc.View(lc.encode(k5, 127, free=True))
    gf, kf = lc.next_geq(v5f, d_probe)
    ms = t(lambda: lc.next_geq(v5f, d_probe, gf, kf))
    print(f"F7 next_geq {ms:.3f} ms {probes.size / ms / 1e6:.3e} probes/s")
    v5f.build_search_index()
    ms = t(lambda: lc.next_geq(v5f, d_probe, gf, kf))
    assert torch.equal(gf, gi), "F7 indexed next_geq mismatch"
    print(f"F7 next_geq+index {ms:.3f} ms {probes.size / ms / 1e6:.3e} probes/s")
    dec = torch.empty(k5.size, dtype=torch.int64, device="cuda")
    ms = t(lambda: lc.decode(v5, dec))
    print(f"decode (long list alone) {ms:.4f} ms")


if __name__ == "__main__":
    main()
