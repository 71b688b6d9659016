#!/usr/bin/env python
"""One batched AND and one batched OR over the corpus' 1e4 query pairs (for an ncu launch list
of their kernels)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_corpus
    lists, eps, pairs = make_corpus()
    bt = lc.Batch([lc.encode(k, e) for k, e in zip(lists, eps)], device="cuda:0")
    ia = lc.SetopBuffers(bt, pairs, lc.LC_SETOP_AND)
    ua = lc.SetopBuffers(bt, pairs, lc.LC_SETOP_OR)
    for _ in range(2):
        lc.intersect_batch(bt, bufs=ia)
        lc.union_batch(bt, bufs=ua)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 10
    ev[0].record()
    for _ in range(reps):
        lc.intersect_batch(bt, bufs=ia)
    ev[1].record()
    for _ in range(reps):
        lc.union_batch(bt, bufs=ua)
    ev[2].record()
    torch.cuda.synchronize()
    print("and", int(ia.counts.sum()), "or", int(ua.counts.sum()),
          f"and_ms {ev[0].elapsed_time(ev[1]) / reps:.4f} or_ms {ev[1].elapsed_time(ev[2]) / reps:.4f}")


if __name__ == "__main__":
    main()
