#!/usr/bin/env python
"""One large u32 list decoded by lc_decode (compile-time residual width) and by lc_decode_batch
(runtime width, chunk records, work queue): isolates the batch kernel's overheads from the
corpus' mix of list lengths."""
from __future__ import annotations

import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import list_eps
    dev = "cuda:0"
    rng = np.random.default_rng(5)
    res = {}
    for n in (2_000_000, 50_000_000):
        x = np.sort(rng.integers(0, (1 << 32) - 1 - n, n, endpoint=True, dtype=np.uint64))
        keys = (x + np.arange(n, dtype=np.uint64)).astype(np.uint32)
        eps = list_eps(n)
        blob = lc.encode(keys, eps)
        h = lc.header(blob)
        v = lc.View(blob, device=dev)
        out = v.out_tensor(n)
        bt = lc.Batch([blob], device=dev)
        bout = torch.empty(n, dtype=torch.int32, device=dev)

        def t(fn, reps=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            ev[0].record()
            for k in range(reps):
                fn()
                ev[k + 1].record()
            torch.cuda.synchronize()
            return statistics.median(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))
        ms_d = t(lambda: lc.decode(v, out))
        ms_b = t(lambda: lc.decode_batch(bt, bout))
        want = torch.from_numpy(keys.view(np.int32)).to(dev)
        assert torch.equal(out, want) and torch.equal(bout, want)
        alg = len(blob) + 4 * n
        res[str(n)] = {"b": int(h.res_bits), "segments": int(h.n_seg),
                       "decode_ms": ms_d, "decode_GBps": alg / ms_d / 1e6,
                       "batch_ms": ms_b, "batch_GBps": (bt.b.payload_bytes + 4 * n) / ms_b / 1e6}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
