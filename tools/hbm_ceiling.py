#!/usr/bin/env python
"""Measure HBM ceilings relevant to the decode roofline: copy (read+write 1:1, the
MEASURED_PEAKS definition), write-only (fill), and read-only (sum), with CUDA events."""
from __future__ import annotations

import json

import torch


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    n = 1 << 29  # 4 GiB of int64
    x = torch.empty(n, dtype=torch.int64, device="cuda")
    y = torch.empty(n, dtype=torch.int64, device="cuda")
    x.fill_(1)
    res = {}
    t = timed(lambda: y.copy_(x))
    res["copy_GBps"] = 2 * n * 8 / t / 1e9
    t = timed(lambda: y.fill_(7))
    res["write_GBps"] = n * 8 / t / 1e9
    t = timed(lambda: x.sum())
    res["read_GBps"] = n * 8 / t / 1e9
    # 1:3 read:write, the decode's mix: read a quarter-size array, write the full one
    q = x[: n // 4]
    t = timed(lambda: y.view(4, -1).copy_(q.expand(4, -1)))
    res["read1_write3_GBps"] = (n // 4 * 8 + n * 8) / t / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
