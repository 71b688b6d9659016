"""Pins for the free-intercept encoder of the oracle (FORMAT F7).

F7 is the O'Rourke rule of PAPER.md:188 (extend a segment while SOME line fits its keys within
eps) on the format's integer lattice: intercept beta in [K[s] - eps, K[s] + eps] with
beta - eps >= 0, slope S / 2^32 with S integer in [0, G / (len - 1)], prediction
beta + floor(S d / 2^32).  The oracle computes one exact slope interval per intercept (cone
arithmetic with ceil/floor divisions); the pins below check it against things that do not
share that arithmetic:

- brute force over the whole lattice at reduced precision (every beta, every S enumerated,
  the Def. 2 bound evaluated directly): each segment is feasible, cannot be extended by one
  key, uses the least-|delta| intercept and the middle slope of that intercept's S set;
- closed forms: a zigzag sequence that one free line fits exactly while the anchored F4 rule
  needs a segment per two keys; arithmetic progressions (one segment, known intercept/slope);
- Def. 1 / Def. 2 on the fuzz corpus with exact rationals, and the validator.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import native as orc
from synth import fuzz_case, make_keys
from tests import blobparse


def _fits(keys, s, e, beta, S, eps, F):
    """Def. 2 for keys[s..e) under beta + floor(S d / 2^F), evaluated directly."""
    for d in range(e - s):
        if abs(int(keys[s + d]) - (beta + ((S * d) >> F))) > eps:
            return False
    return True


def _lattice(keys, s, e, eps, F, gmax):
    """{delta: sorted feasible S} over the whole lattice of FORMAT F7 (brute force)."""
    ks = int(keys[s])
    smax = gmax // max(e - 1 - s, 1)
    out = {}
    for delta in range(-eps, eps + 1):
        beta = ks + delta
        if beta - eps < 0:
            continue
        ss = [S for S in range(smax + 1) if _fits(keys, s, e, beta, S, eps, F)]
        if ss:
            out[delta] = ss
    return out


@pytest.mark.parametrize("F", range(0, 5))
def test_free_greedy_bruteforce_lattice(F):
    """F7 by enumeration: G = 2^(F+6) - 1, keys < 2^9, N <= 24, eps <= 4, so every (beta, S)
    is tried. Checks maximality (first infeasible index ends a segment), the least-|delta|
    intercept (negative on a tie), the S set being an interval and the F5 middle slope."""
    gmax = (1 << (F + 6)) - 1
    rng = np.random.default_rng(700 + F)
    ends = 0
    for trial in range(40):
        n = int(rng.integers(1, 24, endpoint=True))
        keys = np.unique(rng.integers(0, 1 << 9, 3 * n))[:n].astype(np.uint64)
        n = keys.size
        eps = int(rng.integers(0, 5))
        st, ba, sl = orc.segment_free(keys, eps, F=F, gmax=gmax)
        bounds = [int(x) for x in st] + [n]
        assert bounds[0] == 0 and all(a < b for a, b in zip(bounds, bounds[1:]))
        for j in range(len(st)):
            s, e = bounds[j], bounds[j + 1]
            lat = _lattice(keys, s, e, eps, F, gmax)
            assert lat, (trial, j)
            want_delta = min(lat, key=lambda dl: (abs(dl), dl))
            got_delta = int(ba[j]) + eps - int(keys[s])
            assert got_delta == want_delta, (trial, j, lat.keys())
            ss = lat[want_delta]
            assert ss == list(range(ss[0], ss[-1] + 1))  # the S set of one intercept is an interval
            want_S = 0 if e - s == 1 else ss[0] + (ss[-1] - ss[0]) // 2
            assert int(sl[j]) == want_S
            if e < n:
                assert not _lattice(keys, s, e + 1, eps, F, gmax), (trial, j)
                ends += 1
    assert ends > 50


def _check_def2_exact(keys, blob):
    """Def. 2 with exact rationals: f(i) = beta_j + S_j / 2^32 (i - s_j); |K[i] - floor f(i)|
    <= eps and the stored field equals K[i] - floor(f(i)) + eps; bases never wrap."""
    bl = blobparse.parse(blob)
    assert bl.flags == 1 and bl.bias == 0
    us = blobparse.fields(bl)
    starts = [int(x) for x in bl.starts]
    beta = bl.beta
    j = 0
    for i, k in enumerate(keys):
        while starts[j + 1] <= i:
            j += 1
        f = Fraction(beta[j]) + Fraction(int(bl.slope[j]), 1 << 32) * (i - starts[j])
        fl = math.floor(f)
        assert abs(int(k) - fl) <= bl.eps
        assert us[i] == int(k) - fl + bl.eps
        assert beta[j] - bl.eps >= 0
        assert int(bl.slope[j]) * (starts[j + 1] - starts[j] - 1) <= (1 << 63) - 1


@pytest.mark.parametrize("seed", range(1000, 1030))
def test_free_roundtrip_and_def2_fuzz(seed):
    """Def. 1 round trip against the generator's keys, Def. 2 exactly, the
    validator accepts, and the header carries flags = 1."""
    keys, eps, kb, law = fuzz_case(seed, n_max=3000)
    eps = min(eps, (1 << 30) - 1)
    blob = orc.encode(keys, eps, kb, free=True)
    assert orc.validate(blob) == 0
    assert orc.header(blob).flags == 1
    assert np.array_equal(orc.decode(blob), keys), (seed, law)
    _check_def2_exact(keys, blob)


@pytest.mark.parametrize("seed", range(2000, 2012))
def test_free_access_range_predict(seed):
    keys, eps, kb, law = fuzz_case(seed, n_max=30_000)
    eps = min(eps, (1 << 30) - 1)
    blob = orc.encode(keys, eps, kb, free=True)
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, keys.size, 500)
    got, err = orc.access(blob, idx)
    assert err == 0 and np.array_equal(got, keys[idx])
    if keys.size >= 64:
        st = rng.integers(0, keys.size - 64, 40, endpoint=True)
        got, err = orc.range_decode(blob, st, 64)
        assert err == 0
        for r, s in enumerate(st):
            assert np.array_equal(got[r], keys[s:s + 64])
    # segments-only prediction within eps (F7: f(s_j) = base_j + eps)
    pred, err = orc.predict(blob, np.arange(keys.size, dtype=np.uint64))
    assert err == 0
    assert np.all(np.abs(pred.astype(object) - keys.astype(object)) <= eps)


@pytest.mark.parametrize("n,eps,c", [(3, 1, 0), (1000, 1, 5), (4097, 3, 123456), (100_000, 7, 0),
                                     (100_000, 100, 1 << 40)])
def test_zigzag_closed_form(n, eps, c):
    """K_i = c + g i + 2 eps (i mod 2), g = 2 eps + 4 (strictly increasing): the line
    c + eps + g i misses every key by exactly eps, so F7 needs ONE segment. For n >= 3 delta
    is forced to +eps (i = 1 needs S/2^32 >= g + eps - delta, i = 2 needs 2S/2^32 <
    2g + eps - delta + 1), S = g 2^32 + r with 0 <= r <= floor((2^32 - 1) / m), m the largest
    even index (even keys need floor(r m / 2^32) = 0), and base = beta - eps = c. The
    anchored F4 line must pass through K[s] and cannot reach both parities: about one
    segment per two keys."""
    g = 2 * eps + 4
    i = np.arange(n, dtype=np.uint64)
    keys = np.uint64(c) + np.uint64(g) * i + np.uint64(2 * eps) * (i % 2)
    st, ba, sl = orc.segment_free(keys, eps)
    assert st.tolist() == [0]
    assert int(ba[0]) == c
    m = n - 1 if (n - 1) % 2 == 0 else n - 2
    r = (2**32 - 1) // m
    assert int(sl[0]) == g * 2**32 + r // 2
    st_a, _, _ = orc.segment(keys, eps)
    assert st_a.size >= n // 2
    blob = orc.encode(keys, eps, free=True)
    assert np.array_equal(orc.decode(blob), keys)


@pytest.mark.parametrize("g,eps,c", [(1, 0, 0), (7, 3, 100), (1000, 10, 3), (1 << 20, 2, 50)])
def test_ap_free_closed_form(g, eps, c):
    """K_i = c + g i with n (g + 1) <= 2^31: one segment; the least |delta| is 0 when c >= eps
    (beta = K[0], base = c - eps) and eps - c otherwise (base = 0); S = g 2^32 is feasible."""
    n = min(5000, (2**31 - 1) // g)
    keys = np.uint64(c) + np.uint64(g) * np.arange(n, dtype=np.uint64)
    st, ba, sl = orc.segment_free(keys, eps)
    assert st.tolist() == [0]
    delta = 0 if c >= eps else eps - c
    assert int(ba[0]) == c + delta - eps
    assert _fits(keys, 0, n, c + delta, g << 32, eps, 32)
    assert _fits(keys, 0, n, c + delta, int(sl[0]), eps, 32)


def test_free_single_keys_and_gaps():
    """Huge gaps force one-key segments: delta = clamp(0) and slope 0 (F5); the last key of a
    run that cannot follow its predecessor starts a new segment."""
    keys = np.array([0, 1, 2, 2**40, 2**41, 2**62, 2**63 + 5], dtype=np.uint64)
    st, ba, sl = orc.segment_free(keys, 2)
    blob = orc.encode(keys, 2, free=True)
    assert np.array_equal(orc.decode(blob), keys)
    bl = blobparse.parse(blob)
    for j in range(bl.L):
        s, e = int(bl.starts[j]), int(bl.starts[j + 1])
        if e - s == 1:
            assert int(bl.slope[j]) == 0
            k = int(keys[s])
            assert bl.beta[j] == k + max(0, 2 - k)  # delta = clamp(0, eps - K[s], eps)


@pytest.mark.parametrize("cid,n", [(1, 200_000), (2, 200_000), (4, 200_000), (5, 200_000)])
def test_free_fewer_segments_configs(cid, n):
    """Measured, not a theorem (greedy over a lattice is not L-minimal, FORMAT F7): on the
    configs' distributions the free intercept cuts L by >= 15% against F4; config 3 (heavy
    lognormal gaps, two keys per segment) gains ~1% and is only round-tripped."""
    keys = make_keys(cid, n)
    eps = {1: 63, 2: 127, 4: 31, 5: 127}[cid]
    blob_f = orc.encode(keys, eps, free=True)
    blob_a = orc.encode(keys, eps)
    assert np.array_equal(orc.decode(blob_f), keys)
    Lf, La = orc.header(blob_f).L, orc.header(blob_a).L
    assert Lf <= 0.85 * La, (Lf, La)
    assert len(blob_f) < len(blob_a)


def test_free_errors_and_validation():
    keys = np.arange(10, dtype=np.uint64) * 3
    with pytest.raises(orc.OracleError):
        orc.encode(keys, 1 << 30, free=True)  # F7 needs eps <= 2^30 - 1
    blob = bytearray(orc.encode(keys, 2, free=True))
    assert orc.validate(bytes(blob)) == 0
    bad = bytearray(blob)
    bad[88] = 3  # unknown flag bit
    assert orc.validate(bytes(bad)) < 0
    bad = bytearray(blob)
    bad[88] = 0  # same bytes read as an anchored blob: bias and anchor no longer hold
    assert orc.validate(bytes(bad)) < 0 or not np.array_equal(orc.decode(bytes(bad)), keys)
