"""Batches of many lists (lc_batch_init / lc_decode_batch, include/lc.h; NEXT-2's posting-list
corpus, synth/corpus.py): every list's keys equal the generator's (and the oracle's decode of
the same blob), in one launch, for corpora mixing residual widths (per-list eps, b = 0 .. 32),
FORMAT F7 lists, u32 and u64 keys, gapped output offsets and single-key lists."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import native as orc
from synth import fuzz_case, list_eps, make_corpus, make_keys

DEV = "cuda:0"


@pytest.fixture(scope="module")
def lc():
    from paper_2412_10770_b200 import lc as _lc
    return _lc


def _pack(blobs):
    offs, pos = [], 0
    for bl in blobs:
        offs.append(pos)
        pos += (len(bl) + 255) // 256 * 256
    host = np.zeros(pos, np.uint8)
    for o, bl in zip(offs, blobs):
        host[o:o + len(bl)] = np.frombuffer(bl, np.uint8)
    return host, np.asarray(offs, np.uint64)


def test_batch_dir_bytes_and_errors(lc):
    lists = [make_keys(1, 5000), make_keys(1, 3000)]
    blobs = [lc.encode(k, 63) for k in lists]
    host, offs = _pack(blobs)
    nb = C.c_uint64()
    assert lc._lib.lc_batch_dir_bytes(host.ctypes.data, host.nbytes, offs.ctypes.data, 2, C.byref(nb)) == 0
    # list records + one record per 1024-key chunk + the (empty) small-chunk key prefix
    assert nb.value == 64 * 2 + 48 * (5 + 3) + 4
    tiny = [make_keys(1, 1024 + 40), make_keys(1, 7), make_keys(1, 2048)]  # tails 40, 7, none
    ht, ot = _pack([lc.encode(k, 63) for k in tiny])
    assert lc._lib.lc_batch_dir_bytes(ht.ctypes.data, ht.nbytes, ot.ctypes.data, 3, C.byref(nb)) == 0
    assert nb.value == 64 * 3 + 48 * (2 + 1 + 2) + 4 * (2 + 1) + 4 * ((40 + 7 + 31) // 32)
    bad = offs.copy()
    bad[1] += 16  # not 256-byte aligned
    assert lc._lib.lc_batch_dir_bytes(host.ctypes.data, host.nbytes, bad.ctypes.data, 2, C.byref(nb)) == lc.LC_ERR_ARG
    mixed = [blobs[0], lc.encode(make_keys(2, 3000), 127)]  # u32 and u64 lists
    h2, o2 = _pack(mixed)
    assert lc._lib.lc_batch_dir_bytes(h2.ctypes.data, h2.nbytes, o2.ctypes.data, 2, C.byref(nb)) == lc.LC_ERR_ARG
    h3 = host.copy()
    h3[0] = ord("X")  # bad magic
    assert lc._lib.lc_batch_dir_bytes(h3.ctypes.data, h3.nbytes, offs.ctypes.data, 2, C.byref(nb)) == lc.LC_ERR_FORMAT


def _check_batch(lc, lists, blobs, out_off=None):
    bt = lc.Batch(blobs, device=DEV, out_off=out_off)
    out = lc.decode_batch(bt)
    torch.cuda.synchronize()
    h = out.cpu().numpy().view(np.uint32 if bt.b.key_bits == 32 else np.uint64)
    for k, (keys, o) in enumerate(zip(lists, bt.out_off)):
        assert np.array_equal(h[o:o + keys.size], keys), k
    return bt, h


@pytest.mark.gpu
def test_batch_corpus_small(lc):
    lists, eps, _ = make_corpus(m=3000, seed=11, n_max=200_000)
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    bt, h = _check_batch(lc, lists, blobs)
    assert bt.b.m == 3000 and bt.n_total == sum(k.size for k in lists)
    widths = {lc.header(b).res_bits for b in blobs}
    assert len(widths) > 5  # the batch mixes residual widths
    for k in range(0, 3000, 97):  # the oracle's decode of the same blobs
        assert np.array_equal(orc.decode(blobs[k]), lists[k])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_batch_fuzz_mixed(lc, seed):
    """Fuzz corpora of one key width in one batch: eps from 0 (b = 0) to 2^31 - 1 (b = 32),
    F4 and F7 blobs, N from 1 to 1e5, ragged tails; gapped output offsets."""
    rng = np.random.default_rng(seed)
    lists, blobs = [], []
    want_bits = 64 if seed % 2 else 32
    s = 9000 + 1000 * seed
    while len(lists) < 60:
        keys, e, kb, _ = fuzz_case(s, n_max=50_000)
        s += 1
        if kb != want_bits:
            continue
        free = bool(rng.integers(0, 2)) and e <= (1 << 30) - 1
        lists.append(keys)
        blobs.append(lc.encode(keys, e, key_bits=kb, free=free))
    sizes = np.array([k.size for k in lists], np.int64)
    gaps = rng.integers(0, 100, sizes.size)
    out_off = np.concatenate([[0], np.cumsum(sizes + gaps)[:-1]]).astype(np.uint64)
    _check_batch(lc, lists, blobs, out_off=out_off)


@pytest.mark.gpu
def test_batch_big_lists_and_tiny(lc):
    """Dense and sparse lists of the five configs (cut) beside single-key lists."""
    lists = [make_keys(2, 300_001), np.array([7], np.uint64), make_keys(4, 500_000),
             make_keys(3, 200_000), np.array([1 << 63], np.uint64), make_keys(5, 65_536)]
    eps = [127, 0, 31, 255, 5, 127]
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    _check_batch(lc, lists, blobs)


@pytest.mark.gpu
def test_batch_full_corpus(lc):
    """The bench corpus (1e5 posting lists, Zipf-like lengths 10..1e6): every key on device."""
    lists, eps, _ = make_corpus()
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    bt = lc.Batch(blobs, device=DEV)
    out = lc.decode_batch(bt)
    want = torch.from_numpy(np.concatenate(lists).view(np.int32)).to(DEV)
    torch.cuda.synchronize()
    assert torch.equal(out[:want.numel()], want)
    assert list_eps(10) == (1 << 31) - 1


# ------------------------------------------------------------------ batched AND / OR
def _setop_check(lc, lists, blobs, pairs):
    from oracle import setops
    bt = lc.Batch(blobs, device=DEV)
    ia = lc.intersect_batch(bt, pairs)
    ua = lc.union_batch(bt, pairs)
    torch.cuda.synchronize()
    dt = np.uint32 if bt.b.key_bits == 32 else np.uint64
    for name, r, fn in (("AND", ia, setops.intersect), ("OR", ua, setops.union)):
        out = r.out.cpu().numpy().view(dt)
        off = r.out_off.cpu().numpy()
        cnt = r.counts.cpu().numpy()
        for p, (a, b) in enumerate(pairs):
            want = fn(lists[a].astype(np.uint64), lists[b].astype(np.uint64))
            got = out[off[p]:off[p] + cnt[p]].astype(np.uint64)
            assert cnt[p] == want.size and np.array_equal(got, want), (name, p, a, b)
    return bt


@pytest.mark.gpu
def test_setop_batch_corpus_small(lc):
    lists, eps, pairs = make_corpus(m=2000, seed=12, n_max=100_000, pairs=600)
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    # plus pairs with shared keys (subsets, identical lists, single keys)
    rng = np.random.default_rng(5)
    big = int(np.argmax([k.size for k in lists]))
    sub = np.unique(np.concatenate([lists[big][::7], rng.integers(0, 1 << 32, 500, dtype=np.uint64).astype(np.uint32)]))
    lists.append(sub)
    blobs.append(lc.encode(sub, 1023))
    lists.append(lists[big][:1].copy())
    blobs.append(lc.encode(lists[-1], 0))
    extra = np.array([[len(lists) - 2, big], [big, len(lists) - 2], [big, big], [len(lists) - 1, big],
                      [len(lists) - 1, len(lists) - 1]])
    _setop_check(lc, lists, blobs, np.concatenate([pairs, extra]))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [3, 4])
def test_setop_batch_fuzz_u64_free(lc, seed):
    """u64 lists with F4 and F7 blobs, eps from 0 to 2^30 - 1; overlapping lists (one list's
    subset plus noise) so intersections are not empty."""
    rng = np.random.default_rng(seed)
    base = make_keys(5, 200_000)
    lists, blobs = [], []
    for k in range(40):
        take = np.sort(rng.choice(base.size, int(rng.integers(1, 50_000)), replace=False))
        noise = rng.integers(0, int(base[-1]), int(rng.integers(0, 3000)), dtype=np.uint64)
        keys = np.unique(np.concatenate([base[take], noise]))
        e = int(rng.choice([0, 1, 31, 127, 4095, (1 << 30) - 1]))
        lists.append(keys)
        blobs.append(lc.encode(keys, e, free=bool(k % 2)))
    pairs = rng.integers(0, len(lists), (200, 2))
    _setop_check(lc, lists, blobs, pairs)


@pytest.mark.gpu
def test_batch_edges(lc):
    """One-list batches, lists of exactly 1024 k keys (no partial chunk), exactly 64 and 65 keys
    (the small-unit bound), and an empty query batch."""
    for lists in ([make_keys(1, 4096)], [make_keys(1, 64), make_keys(1, 65), make_keys(1, 1024),
                                         make_keys(1, 2048 + 64), np.array([5], np.uint32)]):
        blobs = [lc.encode(k, 63) for k in lists]
        _check_batch(lc, lists, blobs)
    bt = lc.Batch([lc.encode(make_keys(1, 100), 63)], device=DEV)
    r = lc.intersect_batch(bt, np.zeros((0, 2), np.int64))
    assert r.plan.n_pairs == 0
