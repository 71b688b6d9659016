#!/usr/bin/env python
"""Segment counts of the greedy encoders (F4, F7) and of the fewest-segments option
(LC_FLAG_MIN_SEGMENTS) on full-size configs, with host encode times; every blob decoded on the
GPU and compared with the keys."""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2412_10770_b200 import lc
    from synth import CONFIGS, make_keys
    res = {}
    for cid in [int(x) for x in (sys.argv[1:] or ["1", "2", "5"])]:
        keys = make_keys(cid)
        eps = CONFIGS[cid].eps
        want = torch.from_numpy(keys.view(np.int64) if keys.itemsize == 8 else keys.view(np.int32)).cuda()
        row = {}
        for free in (False, True):
            for mn in (False, True):
                t0 = time.perf_counter()
                blob = lc.encode(keys, eps, free=free, min_segments=mn)
                t = time.perf_counter() - t0
                out = lc.decode(lc.View(blob))
                torch.cuda.synchronize()
                ok = bool(torch.equal(out, want))
                row[("F7" if free else "F4") + ("_min" if mn else "")] = {
                    "segments": int(lc.header(blob).n_seg), "blob_bytes": len(blob),
                    "encode_s": t, "bit_exact": ok}
        res[f"config{cid}"] = row
        print(json.dumps({f"config{cid}": row}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
