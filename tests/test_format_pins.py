"""FORMAT F2 section definitions recomputed by the tests from the raw blob bytes (tests/blobparse,
independent of both encoders' writers and of the oracle's validator).

The hint section is consumed only by the product kernels (the oracle's decode and access never
read it), so a shared misreading of its definition would pass round-trip parity; here it is
pinned to its definition (FORMAT F2, the north star's "segment id every 1024
keys"; PAPER.md:286 the auxiliary segment-localisation structure):
    hint[h] = max{j : starts[j] <= 1024 h}  for h < H = ceil(N / 1024),   hint[H] = L - 1,
together with the starts section (starts[0] = 0, strictly increasing, starts[L] = N; Eq. 1,
PAPER.md:174-177: segment j covers s_j <= i < s_{j+1}).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import native as orc
from synth import fuzz_case, make_keys
from tests.blobparse import parse


def _hint_by_definition(starts: np.ndarray, n: int) -> np.ndarray:
    L = starts.size - 1
    H = (n + 1023) // 1024
    h = np.arange(H, dtype=np.int64) * 1024
    # max{j : starts[j] <= 1024 h}, with j ranging over segment ids 0..L-1
    want = np.searchsorted(starts[:L].astype(np.int64), h, side="right") - 1
    return np.concatenate([want, [L - 1]]).astype(np.int64)


def _hint_brute(starts: np.ndarray, n: int) -> list[int]:
    """Same definition by a plain loop over the segments (small inputs only)."""
    L = starts.size - 1
    out = []
    for h in range((n + 1023) // 1024):
        out.append(max(j for j in range(L) if int(starts[j]) <= 1024 * h))
    return out + [L - 1]


def _check(blob: bytes, n: int, brute: bool = False) -> None:
    bl = parse(blob)
    assert bl.n == n
    s = bl.starts.astype(np.int64)
    assert s[0] == 0 and s[-1] == n and bl.L == s.size - 1
    assert np.all(np.diff(s) > 0)
    assert bl.n_hint == (n + 1023) // 1024 + 1
    got = bl.hint.astype(np.int64)
    assert np.array_equal(got, _hint_by_definition(s, n))
    if brute:
        assert got.tolist() == _hint_brute(s, n)
    # what the kernels rely on: segment hint[h] holds key 1024 h (s_j <= 1024 h < s_{j+1})
    for h in range(bl.n_hint - 1):
        j = int(got[h])
        assert s[j] <= 1024 * h < s[j + 1]


@pytest.mark.parametrize("seed", range(7000, 7060))
def test_hint_oracle_encoder_fuzz(seed):
    keys, eps, kb, _ = fuzz_case(seed, n_max=20_000)
    n = keys.size
    _check(orc.encode(keys, eps, key_bits=kb), n, brute=n <= 5000)
    if eps <= (1 << 30) - 1:
        _check(orc.encode(keys, eps, key_bits=kb, free=True), n, brute=n <= 5000)


@pytest.mark.parametrize("seed", range(7000, 7060))
def test_hint_product_encoder_fuzz(seed):
    from paper_2412_10770_b200 import lc
    keys, eps, kb, _ = fuzz_case(seed, n_max=20_000)
    n = keys.size
    _check(lc.encode(keys, eps, key_bits=kb), n, brute=n <= 5000)
    if eps <= (1 << 30) - 1:
        _check(lc.encode(keys, eps, key_bits=kb, free=True), n, brute=n <= 5000)


@pytest.mark.parametrize("n", [1, 2, 1023, 1024, 1025, 2048, 4097, 9216, 10_001])
@pytest.mark.parametrize("brk", ["none", "every", "edges", "edges_pm1", "every128", "all_but_edges"])
def test_hint_adversarial_breaks(n, brk):
    """Segment starts exactly at, one before and one after 1024-key boundaries (the cases where
    max{j : s_j <= 1024 h} changes), every key a segment, and one segment over everything."""
    keys = np.arange(n, dtype=np.uint64) * np.uint64(3) + np.uint64(5)
    fb = np.zeros(n, np.uint8)
    if brk == "every":
        fb[:] = 1
    elif brk == "edges":
        fb[::1024] = 1
    elif brk == "edges_pm1":
        for e in range(1024, n + 1, 1024):
            fb[e - 1] = 1
            if e + 1 < n:
                fb[e + 1] = 1
    elif brk == "every128":
        fb[::128] = 1
    elif brk == "all_but_edges":
        fb[:] = 1
        fb[::1024] = 0
    blob = orc.encode(keys, 3, force_break=fb if brk != "none" else None)
    assert orc.validate(blob) == 0
    s = set(parse(blob).starts.tolist())
    assert all(i in s for i in np.flatnonzero(fb).tolist())  # every forced break is a start
    if brk == "every":
        assert parse(blob).L == n
    _check(blob, n, brute=True)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_hint_configs_small(cid):
    from paper_2412_10770_b200 import lc
    from synth import CONFIGS
    keys = make_keys(cid, 300_001)
    eps = CONFIGS[cid].eps
    _check(lc.encode(keys, eps), keys.size)
    _check(lc.encode(keys, eps, free=True), keys.size)
