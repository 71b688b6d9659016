"""Seeded generators for the five BASELINE.json configs and the parity fuzz corpus.

Recipe: numpy.random.default_rng(seed)
(PCG64), draws taken in the order written below, integer bounds inclusive
(`integers(lo, hi, endpoint=True)`, default dtype int64). Every array is a sorted, strictly
increasing key list K with k_1 = 0 unless stated. Nothing here fits, predicts
or packs: this module is shared by the oracle tests and the CUDA-path tests, so it must hold
none of the method's arithmetic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ConfigSpec:
    cid: int
    n: int
    key_bits: int
    eps: int
    seed: int
    desc: str


# BASELINE.json "configs" (index = cid - 1).
CONFIGS = {
    1: ConfigSpec(1, 1_000_000, 32, 63, 0, "uniform gaps [1,64], u32"),
    2: ConfigSpec(2, 100_000_000, 64, 127, 1, "geometric gaps mean 100, u64"),
    3: ConfigSpec(3, 200_000_000, 64, 255, 2, "lognormal(0,2)*1e9 distinct, u64"),
    4: ConfigSpec(4, 500_000_000, 64, 31, 3, "Zipf(1.2) clusters, gaps [1,8], jumps [1e6,1e9], u64"),
    5: ConfigSpec(5, 100_000_000, 64, 127, 4, "uniform gaps [1,256], u64 + access/range queries"),
}

# config 5 query counts at full size (BASELINE.json configs[4])
C5_QUERIES = 100_000_000
C5_RANGES = 10_000_000
C5_RANGE_LEN = 64


def _from_gaps(gaps: np.ndarray, dtype) -> np.ndarray:
    k = np.empty(gaps.size + 1, dtype=np.uint64)
    k[0] = 0
    np.cumsum(gaps, out=k[1:], dtype=np.uint64)
    return k.astype(dtype, copy=False)


def _cfg1(rng, n):
    return _from_gaps(rng.integers(1, 64, n - 1, endpoint=True), np.uint32)


def _cfg2(rng, n):
    # numpy geometric has support {1, 2, ...}; p = 0.01 gives mean 100
    return _from_gaps(rng.geometric(0.01, n - 1), np.uint64)


def _first_n_distinct(x: np.ndarray, n: int) -> np.ndarray:
    """Set of the first n distinct values of x in draw order, sorted.

    Equivalent to `u, first = np.unique(x, return_index=True); keep u[first among the n
    smallest first-indices]`, computed without a stable argsort of the full array.
    """
    v = np.sort(x)
    dup_mask = v[1:] == v[:-1]
    dup_vals = np.unique(v[1:][dup_mask])  # values drawn more than once
    del v, dup_mask
    repeat = np.zeros(x.size, dtype=bool)  # draw i repeats a value drawn earlier
    if dup_vals.size:
        # cheap pre-filter on the low 30 bits, then an exact sorted-membership check
        table = np.zeros(1 << 30, dtype=bool)
        table[(dup_vals & np.uint64((1 << 30) - 1)).astype(np.int64)] = True
        cand = np.flatnonzero(table[(x & np.uint64((1 << 30) - 1)).astype(np.int64)])
        del table
        cv = x[cand]
        pos = np.searchsorted(dup_vals, cv)
        pos[pos == dup_vals.size] = 0
        hit = dup_vals[pos] == cv
        idx = cand[hit]
        vals = cv[hit]
        order = np.argsort(vals, kind="stable")  # stable: equal values keep draw order
        sv = vals[order]
        si = idx[order]
        later = np.empty(sv.size, dtype=bool)
        later[0] = False
        later[1:] = sv[1:] == sv[:-1]
        repeat[si[later]] = True
    distinct_so_far = np.arange(1, x.size + 1, dtype=np.int64) - np.cumsum(repeat)
    if distinct_so_far[-1] < n:
        raise ValueError(f"only {distinct_so_far[-1]} distinct draws, need {n}")
    p = int(np.searchsorted(distinct_so_far, n)) + 1  # shortest prefix with n distinct
    keep = x[:p][~repeat[:p]]
    assert keep.size == n
    keep.sort()
    return keep


def _cfg3(rng, n):
    draws = 210_000_000 if n == 200_000_000 else int(n * 1.05) + 64
    x = np.floor(rng.lognormal(mean=0.0, sigma=2.0, size=draws) * 1e9).astype(np.uint64)
    return _first_n_distinct(x, n)


def _cfg4(rng, n):
    sizes = np.minimum(rng.zipf(1.2, 200_000), 1_000_000)
    cs = np.cumsum(sizes)
    c = int(np.searchsorted(cs, n)) + 1  # clusters needed so that sum >= n
    if cs[-1] < n:
        raise ValueError("200000 Zipf clusters do not cover n")
    sizes = sizes[:c].copy()
    sizes[-1] -= int(cs[c - 1] - n)  # trim the last cluster so the sizes sum to n
    gaps = rng.integers(1, 8, n - 1, endpoint=True)
    jumps = rng.integers(1_000_000, 1_000_000_000, c - 1, endpoint=True)
    bpos = np.cumsum(sizes)[:-1] - 1  # gap index between the last key of a cluster and the next
    gaps[bpos] = jumps
    return _from_gaps(gaps, np.uint64)


def _cfg5(rng, n):
    return _from_gaps(rng.integers(1, 256, n - 1, endpoint=True), np.uint64)


_GEN = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}


def make_keys(cid: int, n: int | None = None) -> np.ndarray:
    """Sorted strictly increasing keys of config `cid` (u32 for config 1, else u64).

    `n` overrides N with the same recipe and seed (the small parity cases)."""
    spec = CONFIGS[cid]
    n = spec.n if n is None else int(n)
    if n < 2:
        raise ValueError("config generators need n >= 2")
    rng = np.random.default_rng(spec.seed)
    return _GEN[cid](rng, n)


def make_queries(n: int | None = None, q: int | None = None, r: int | None = None,
                 rlen: int = C5_RANGE_LEN):
    """Config 5: (keys, access indices u64[q], range starts u64[r]).

    Draw order in the seed-4 stream: gaps, then idx = integers(0, N-1, q), then
    rstart = integers(0, N-rlen, r) (every range in bounds)."""
    spec = CONFIGS[5]
    n = spec.n if n is None else int(n)
    q = C5_QUERIES if q is None else int(q)
    r = C5_RANGES if r is None else int(r)
    rng = np.random.default_rng(spec.seed)
    keys = _cfg5(rng, n)
    idx = rng.integers(0, n - 1, q, endpoint=True).astype(np.uint64)
    rstart = rng.integers(0, max(n - rlen, 0), r, endpoint=True).astype(np.uint64)
    return keys, idx, rstart


# ----------------------------------------------------------------------------- fuzz corpus

_EPS_CHOICES = [0, 1] + [(1 << k) - 1 for k in range(2, 13)]


def fuzz_case(seed: int, n_max: int = 100_000):
    """One parity fuzz corpus (SURVEY §8(d) "Fuzz corpora"): returns (keys, eps, key_bits, law).

    N log-uniform in [1, n_max]; gap law in {uniform [1,2^k] (k<=40), geometric, lognormal
    sample, clustered, AP}; eps in {0, 1, 2^k-1 (k<=12)}; optional start offset, sometimes
    pushing the last key to the top of the key width."""
    rng = np.random.default_rng(seed)
    n = int(math.exp(rng.uniform(0.0, math.log(n_max)))) if n_max > 1 else 1
    n = max(1, min(n, n_max))
    eps = int(rng.choice(_EPS_CHOICES))
    law = str(rng.choice(["uniform", "geometric", "lognormal", "clustered", "ap"]))
    if law == "uniform":
        k = int(rng.integers(0, 40, endpoint=True))
        gaps = rng.integers(1, 1 << k, max(n - 1, 0), endpoint=True).astype(np.uint64)
    elif law == "geometric":
        p = float(rng.choice([0.5, 0.1, 0.01, 0.001]))
        gaps = rng.geometric(p, max(n - 1, 0)).astype(np.uint64)
    elif law == "lognormal":
        sigma = float(rng.uniform(0.5, 3.0))
        x = np.unique(np.floor(rng.lognormal(0.0, sigma, 2 * n + 8) * 1e6).astype(np.uint64))
        x = x[:n]
        gaps = np.diff(x) if x.size > 1 else np.zeros(0, np.uint64)
        n = x.size
    elif law == "clustered":
        gaps = rng.integers(1, 8, max(n - 1, 0), endpoint=True).astype(np.uint64)
        nb = max(1, n // 50)
        pos = rng.integers(0, max(n - 2, 0), nb, endpoint=True)
        if gaps.size:
            gaps[pos] = rng.integers(1 << 20, 1 << 34, nb, endpoint=True).astype(np.uint64)
    else:  # arithmetic progression
        g = int(rng.integers(1, 1 << 24, endpoint=True))
        gaps = np.full(max(n - 1, 0), g, dtype=np.uint64)
    span = int(gaps.sum(dtype=object)) if gaps.size else 0
    want32 = bool(rng.integers(0, 2)) and span < (1 << 32) - 1
    top = (1 << 32) - 1 if want32 else (1 << 64) - 1
    off_mode = int(rng.integers(0, 3))
    if off_mode == 0:
        start = 0
    elif off_mode == 1:
        start = int(rng.integers(0, max(top - span, 0), endpoint=True, dtype=np.uint64))
    else:
        start = top - span  # last key = maximum of the key width
    keys = np.empty(n, dtype=np.uint64)
    keys[0] = start
    if n > 1:
        keys[1:] = np.uint64(start) + np.cumsum(gaps, dtype=np.uint64)
    key_bits = 32 if want32 else 64
    if key_bits == 32:
        keys = keys.astype(np.uint32)
    return keys, eps, key_bits, law
