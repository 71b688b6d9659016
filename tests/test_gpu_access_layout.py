"""Access layout (lc_access_layout_build, include/lc.h): segment-major records so a random
access reads its segment's params and residual field from one record (PAPER.md:297 f(j) +
Delta[j]; §IV-E ② memory hierarchy).

CPU: the layout size formula.  GPU (-m gpu): the device-built bytes equal the records the test
assembles from the raw blob sections (tests/blobparse), and lc_access / exact lc_quantile with
the layout attached equal the generator's keys (and the oracle) on fuzz corpora, adversarial
segmentations, the eps extremes (b = 0 and b = 32), F7 blobs and the full config-5 workload."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import native as orc
from synth import CONFIGS, fuzz_case, make_keys, make_queries
from tests.blobparse import parse

DEV = "cuda:0"


@pytest.fixture(scope="module")
def lc():
    from paper_2412_10770_b200 import lc as _lc
    return _lc


def _records(blob: bytes) -> np.ndarray:
    """The layout by its definition (include/lc.h): per 32 keys (word w of 1024-key block h)
    a pair {bits, rank | dist << 11}: bit t of `bits` set iff key 1024 h + 32 w + t starts a
    segment (block position 0 excluded), rank = bits set in words < w of the block, dist = 32 w
    minus the start of the segment holding key 1024 h + 32 w (capped at 2^21 - 1); then record
    j at 16-byte unit 2 j + floor(s_j b / 128): {base_j, slope_j} and the words' 16-byte units
    floor(s_j b/128) .. floor(s_{j+1} b/128)."""
    bl = parse(blob)
    n, L, b = bl.n, bl.L, bl.b
    H = (n + 1023) // 1024
    starts = bl.starts.astype(np.int64)
    bits = np.zeros(32 * H, np.uint32)
    for s in starts[1:L]:
        if s % 1024:
            bits[s >> 5] |= np.uint32(1 << (s & 31))
    ent = np.zeros(32 * H, np.uint32)
    for h in range(H):
        for w in range(32):
            rank = sum(bin(int(x)).count("1") for x in bits[32 * h:32 * h + w])
            key = 1024 * h + 32 * w
            j = int(np.searchsorted(starts[:L], key, side="right")) - 1  # segment holding key
            dist = min(key - int(starts[j]), (1 << 21) - 1)
            ent[32 * h + w] = rank | (dist << 11)
    units = 2 * L + (n * b) // 128
    rec = np.zeros(units * 4, np.uint32)
    w = bl.words
    for j in range(L):
        s0, s1 = int(starts[j]), int(starts[j + 1])
        u0, u1 = (s0 * b) // 128, (s1 * b) // 128
        r = 2 * j + u0
        rec[4 * r:4 * r + 4] = np.array([int(bl.base[j]), int(bl.slope[j])], np.uint64).view(np.uint32)
        rec[4 * (r + 1):4 * (r + 2 + u1 - u0)] = w[4 * u0:4 * (u1 + 1)]
    return np.concatenate([np.stack([bits, ent], axis=1).reshape(-1), rec])


@pytest.mark.parametrize("seed", range(7300, 7310))
def test_layout_bytes_formula(lc, seed):
    keys, eps, kb, _ = fuzz_case(seed, n_max=20_000)
    blob = lc.encode(keys, eps, key_bits=kb)
    bl = parse(blob)

    v = lc.lc_view()  # lc_access_layout_bytes reads only the header of the view
    import ctypes as C
    C.memmove(C.addressof(v.h), blob, 128)
    assert lc._lib.lc_access_layout_bytes(C.byref(v)) == _records(blob).nbytes
    H = (bl.n + 1023) // 1024
    assert _records(blob).nbytes == 256 * H + 16 * (2 * bl.L + bl.n * bl.b // 128)


def _dev(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)).to(DEV)


def _host(t, dtype):
    return t.cpu().numpy().view(dtype)


def _check_blob(lc, blob, keys, rng, m=20_000, layout_bytes=True):
    v = lc.View(blob, device=DEV)
    lay = v.build_access_layout()
    torch.cuda.synchronize()
    if layout_bytes and keys.size <= 200_000:
        got = lay.cpu().numpy().view(np.uint32)[: v.access_layout_bytes() // 4]
        assert np.array_equal(got, _records(blob))
    n = keys.size
    idx = np.unique(np.concatenate([rng.integers(0, n, m), [0, n - 1]])).astype(np.uint64)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    a = lc.access(v, _dev(idx), err=err)
    ranks = rng.integers(0, 1000, 2000, endpoint=True).astype(np.uint64)
    qi = np.array([orc.quantile_index(n, int(k), 1000) for k in ranks], np.int64)
    q = lc.quantile(v, _dev(ranks), 1000, err=err)
    qa = lc.quantile(v, _dev(ranks), 1000, exact=False)
    bad = np.array([n, n + 5, 1 << 40], np.uint64)  # out of range: 0 and the error bit
    ab = lc.access(v, _dev(bad), err=err)
    rgs = {}
    for ln in (1, 2, 31, 32, 33, 63, 64, 100):  # with the layout attached, len <= 64: lc_range64_dir_kernel
        if n >= ln:
            st = rng.integers(0, n - ln, 700, endpoint=True).astype(np.uint64)
            rgs[ln] = (st, lc.range_decode(v, _dev(st), ln))
    torch.cuda.synchronize()
    for ln, (st, rg) in rgs.items():
        want = keys[st.astype(np.int64)[:, None] + np.arange(ln)]
        assert np.array_equal(_host(rg, keys.dtype).reshape(-1, ln), want), ln
    e2 = torch.zeros(1, dtype=torch.int32, device=DEV)
    rb = lc.range_decode(v, _dev(np.array([0, max(n - 63, 0), n], np.uint64)), 64, err=e2)
    torch.cuda.synchronize()
    rbh = _host(rb, keys.dtype).reshape(-1, 64)
    assert not rbh[1:].any() and int(e2.item()) == 1
    if n >= 64:
        assert np.array_equal(rbh[0], keys[:64])
    assert np.array_equal(_host(a, keys.dtype), keys[idx.astype(np.int64)])
    assert np.array_equal(_host(q, keys.dtype), keys[qi])
    assert np.array_equal(_host(qa, keys.dtype), orc.predict(blob, qi.astype(np.uint64))[0])
    assert not _host(ab, keys.dtype).any() and int(err.item()) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(1000, 1080))
def test_layout_fuzz(lc, seed):
    keys, eps, kb, _ = fuzz_case(seed)
    rng = np.random.default_rng(seed)
    _check_blob(lc, lc.encode(keys, eps, key_bits=kb), keys, rng)
    if eps <= (1 << 30) - 1:
        _check_blob(lc, lc.encode(keys, eps, key_bits=kb, free=True), keys, rng)


@pytest.mark.gpu
@pytest.mark.parametrize("brk", ["all", "every3", "tile_edges", "none"])
@pytest.mark.parametrize("eps", [0, 1, 127, (1 << 31) - 1])
def test_layout_adversarial(lc, brk, eps):
    n = 30_000
    keys = make_keys(5, n)
    fb = np.zeros(n, np.uint8)
    if brk == "all":
        fb[:] = 1
    elif brk == "every3":
        fb[::3] = 1
    elif brk == "tile_edges":
        fb[::1024] = 1
        fb[1023::1024] = 1
    blob = orc.encode(keys, eps, force_break=fb if brk != "none" else None)
    _check_blob(lc, blob, keys, np.random.default_rng(eps))


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_layout_configs_small(lc, cid):
    keys = make_keys(cid, 400_001)
    _check_blob(lc, lc.encode(keys, CONFIGS[cid].eps), keys, np.random.default_rng(cid))


@pytest.mark.gpu
def test_layout_full_config5(lc):
    """The bench workload: all 1e8 lookups with the layout attached, on device; 5000 against
    the oracle one by one; exact quantiles; and the same blob without the layout agrees."""
    keys, idx, _ = make_queries()
    blob = lc.encode(keys, 127)
    v = lc.View(blob, device=DEV)
    d_idx = _dev(idx)
    plain = lc.access(v, d_idx)
    v.build_access_layout()
    got = lc.access(v, d_idx)
    d_keys = _dev(keys)
    torch.cuda.synchronize()
    assert torch.equal(got, d_keys[d_idx])
    assert torch.equal(got, plain)
    del plain
    want, err = orc.access(blob, idx[:5000])
    assert err == 0 and np.array_equal(_host(got[:5000], np.uint64), want)
    keys_r, _, rs = make_queries()
    d_rs = _dev(rs)
    rg = lc.range_decode(v, d_rs, 64)
    assert torch.equal(rg, d_keys[d_rs[:, None] + torch.arange(64, device=DEV)[None, :]])
    del rg
    ranks = torch.from_numpy(np.random.default_rng(9).integers(0, 1 << 20, 1_000_000)).to(DEV)
    q = lc.quantile(v, ranks, 1 << 20)
    qi = torch.clamp(ranks * keys.size // (1 << 20), max=keys.size - 1)
    torch.cuda.synchronize()
    assert torch.equal(q, d_keys[qi])


@pytest.mark.gpu
@pytest.mark.parametrize("eps", [0, 3, 1000])
def test_layout_long_segments(lc, eps):
    """Segments longer than 2^21 keys (the directory's dist field saturates, kDistNone): lookups
    and 64-key ranges deep inside them, around their ends, and across a dense stretch."""
    rng = np.random.default_rng(77 + eps)
    ap1 = np.arange(5_000_000, dtype=np.uint64) * np.uint64(7) + np.uint64(3)
    mid = ap1[-1] + np.cumsum(rng.integers(1, 1 << 20, 3000)).astype(np.uint64)
    ap2 = mid[-1] + np.uint64(1) + np.arange(2_500_000, dtype=np.uint64) * np.uint64(2)
    keys = np.concatenate([ap1, mid, ap2])
    blob = lc.encode(keys, eps)
    assert lc.header(blob).n_seg < keys.size // 1000
    v = lc.View(blob, device=DEV)
    v.build_access_layout()
    n = keys.size
    edges = np.array([0, 1, (1 << 21) - 70, (1 << 21) - 1, 1 << 21, (1 << 22) + 5, ap1.size - 64,
                      ap1.size - 63, ap1.size - 1, ap1.size, ap1.size + mid.size - 10,
                      ap1.size + mid.size, n - 64], np.uint64)
    st = np.concatenate([edges, rng.integers(0, n - 64, 4000, endpoint=True).astype(np.uint64)])
    rg = lc.range_decode(v, _dev(st), 64)
    a = lc.access(v, _dev(st))
    torch.cuda.synchronize()
    assert np.array_equal(_host(rg, np.uint64).reshape(-1, 64), keys[st.astype(np.int64)[:, None] + np.arange(64)])
    assert np.array_equal(_host(a, np.uint64), keys[st.astype(np.int64)])
