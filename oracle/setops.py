"""Set operations on sorted key lists (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

The plain definitions behind NEXT-2: successor search and list intersection, the
AND query of inverted-index processing (§III-A).  The compressed form does not
change the answer (Dec(K^c) = K, Def. 1), so the oracle works on the key arrays themselves.
Pins: tests/test_oracle_pins.py (brute force on tiny lists, lcm closed form).
"""
from __future__ import annotations

import numpy as np


def next_geq(keys: np.ndarray, x: np.ndarray):
    """For each probe x_t: the smallest index i with K[i] >= x_t (N if none) and K[i] (0 if
    none)."""
    k = np.asarray(keys)
    xs = np.asarray(x, dtype=np.uint64)
    if k.dtype == np.uint32:
        # probes above the u32 range are past every key
        idx = np.where(xs > 0xFFFFFFFF, k.size,
                       np.searchsorted(k, np.minimum(xs, 0xFFFFFFFF).astype(np.uint32), side="left"))
    else:
        idx = np.searchsorted(k, xs, side="left")
    idx = idx.astype(np.uint64)
    key = np.zeros(xs.size, dtype=k.dtype)
    hit = idx < k.size
    key[hit] = k[idx[hit].astype(np.int64)]
    return idx, key


def intersect(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Sorted keys present in both lists (both strictly increasing)."""
    return np.intersect1d(a, b, assume_unique=True)


def union(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Sorted keys present in either list (each once)."""
    return np.union1d(a, b)
