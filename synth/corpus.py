"""Seeded synthetic posting-list corpus (SURVEY §8(f) NEXT-2 "a synthetic many-list posting
corpus"; the paper's workload is the CCNews inverted index, §II-C, which is not
in this container and is not reconstructed).

Recipe (corpus row): numpy PCG64 from `seed`, draws in this order:
  1. m list lengths n_k = min(floor(10 * U_k^(-1/alpha)), 10^6), U_k uniform in (0, 1]
     (a Pareto tail: the document-frequency law of a Zipf vocabulary, exponent 1/alpha);
  2. per list, in order, n_k docIDs: a sorted sample of n_k integers uniform in
     [0, 2^32 - 1 - n_k] plus their ranks 0..n_k-1 (strictly increasing, < 2^32);
  3. the query pairs: `pairs` (a, b) with both terms drawn with probability ~ n_k^0.25
     (frequent terms are queried more often; the short side of a pair has median ~20 keys,
     the long side ~150).
Per-list eps (the residual budget of each posting list) is part of the input, chosen from
the list's mean docID gap g_k = 2^32 / n_k as eps_k = 2^(ceil(log2 g_k) + 2) - 1 (capped at
2^31 - 1).  Nothing here fits, predicts or packs.
"""
from __future__ import annotations

import math

import numpy as np

UNIVERSE = 1 << 32


def corpus_lengths(m: int, seed: int, alpha: float = 0.7, n_min: int = 10,
                   n_max: int = 1_000_000) -> np.ndarray:
    rng = np.random.default_rng(seed)
    u = 1.0 - rng.random(m)  # (0, 1]
    return np.minimum(np.floor(n_min * u ** (-1.0 / alpha)), n_max).astype(np.int64)


def list_eps(n: int) -> int:
    g = UNIVERSE / max(n, 1)
    return min((1 << (math.ceil(math.log2(g)) + 2)) - 1, (1 << 31) - 1)


def make_corpus(m: int = 100_000, seed: int = 10, alpha: float = 0.7, n_min: int = 10,
                n_max: int = 1_000_000, pairs: int = 10_000):
    """(lists: list of sorted uint32 arrays, eps: list of ints, pairs: int64 [P, 2])."""
    rng = np.random.default_rng(seed)
    u = 1.0 - rng.random(m)
    lens = np.minimum(np.floor(n_min * u ** (-1.0 / alpha)), n_max).astype(np.int64)
    lists, eps = [], []
    for n in lens.tolist():
        x = np.sort(rng.integers(0, UNIVERSE - 1 - n, n, endpoint=True, dtype=np.uint64))
        x += np.arange(n, dtype=np.uint64)
        lists.append(x.astype(np.uint32))
        eps.append(list_eps(n))
    p = lens.astype(np.float64) ** 0.25
    p /= p.sum()
    pr = rng.choice(m, size=(pairs, 2), p=p).astype(np.int64)
    return lists, eps, pr
