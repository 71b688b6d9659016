#!/usr/bin/env python
"""One lc_union (1e6-key short list with config 5's 1e8-key list, as in bench.py) followed by a
plain lc_decode of the long list, for an ncu --set full comparison of the shifted (UNI) and
the plain decode kernel."""
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
    na = 1_000_000
    a = np.unique(np.concatenate([k5[np.sort(rng.choice(k5.size, na // 2, replace=False))],
                                  rng.integers(0, int(k5[-1]), na // 2, dtype=np.uint64)]))
    va = lc.View(lc.encode(a, 127))
    uo, uc = lc.union(va, v5)
    dec = lc.decode(v5)
    torch.cuda.synchronize()
    print("union", int(uc.item()), "decode", dec.numel())


if __name__ == "__main__":
    main()
