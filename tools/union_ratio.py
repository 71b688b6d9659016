#!/usr/bin/env python
"""Time lc_union on config 5 (1e8 keys) against short lists of growing size, for choosing the
fused / merge threshold (run once per library variant: LC_LIB=...)."""
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
    rng = np.random.default_rng(56)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for ns in (100_000, 1_000_000, 4_000_000, 12_500_000, 25_000_000, 50_000_000):
        a = np.unique(np.concatenate([k5[np.sort(rng.choice(k5.size, ns // 2, replace=False))],
                                      rng.integers(0, int(k5[-1]), ns // 2, dtype=np.uint64)]))
        va = lc.View(lc.encode(a, 127))
        scr = torch.empty(lc.union_scratch_bytes(va, v5), dtype=torch.uint8, device="cuda")
        uo, uc = lc.union(va, v5, scr)
        torch.cuda.synchronize()
        assert int(uc.item()) == np.union1d(a, k5).size
        best = 1e9
        for _ in range(5):
            ev[0].record()
            lc.union(va, v5, scr, uo, uc)
            ev[1].record()
            torch.cuda.synchronize()
            best = min(best, ev[0].elapsed_time(ev[1]))
        print(f"{os.environ.get('LC_LIB', 'default')} ns={a.size} union {best:.4f} ms", flush=True)
        del va, scr, uo, uc


if __name__ == "__main__":
    main()
