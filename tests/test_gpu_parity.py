"""GPU parity: the sm_100a kernels, called through the C ABI, against the CPU oracle and the
generators' own key arrays (bit-exact; integer path, zero tolerance).

Expected values never come from the CUDA path: they are the synthetic key arrays themselves
(Def. 1: Dec(K^c) = K) and the oracle's decode / access / range of the same blob.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import native as orc  # noqa: E402
from synth import CONFIGS, fuzz_case, make_keys, make_queries  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lc():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2412_10770_b200 import lc as m
    return m


DEV = "cuda:0"


def _dev(a: np.ndarray):
    a = np.ascontiguousarray(a)
    v = a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)
    return torch.from_numpy(v).to(DEV)


def _host(t, dtype):
    return t.cpu().numpy().view(dtype)


def _decode_equal(lc, blob, keys):
    view = lc.View(blob, device=DEV)
    out = lc.decode(view)
    torch.cuda.synchronize()
    return torch.equal(out, _dev(keys))


# ------------------------------------------------------------------------- full decode
@pytest.mark.parametrize("seed", range(1000, 1300))
def test_decode_fuzz(lc, seed):
    keys, eps, kb, law = fuzz_case(seed, n_max=100_000)
    blob = lc.encode(keys, eps, kb)
    assert _decode_equal(lc, blob, keys), (seed, law, keys.size, eps)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [2, 1023, 1024, 1025, 33_000, 262_145])
def test_decode_configs_small(lc, cid, n):
    keys = make_keys(cid, n)
    eps = CONFIGS[cid].eps
    blob = lc.encode(keys, eps)
    view = lc.View(blob, device=DEV)
    out = lc.decode(view)
    torch.cuda.synchronize()
    want = orc.decode(blob)
    assert np.array_equal(want, keys)
    assert np.array_equal(_host(out, keys.dtype), want)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("brk", ["every3", "tile_edges", "all", "dense_runs"])
def test_decode_adversarial_blobs(lc, mode, brk):
    """P9: valid non-normative blobs from the oracle's test-only builder (lo/mid/hi slopes,
    forced breaks at 1024-key edges, T-1, T+1, all-1-key segments over whole chunks — the
    worst case for the staged segment pages)."""
    n = 40_000
    keys = make_keys(5, n)
    fb = np.zeros(n, np.uint8)
    if brk == "every3":
        fb[::3] = 1
    elif brk == "tile_edges":
        fb[::1024] = 1
        for t in range(4096, n - 1, 4096):
            fb[t - 1] = fb[t + 1] = 1
    elif brk == "all":
        fb[:] = 1
    else:  # alternating dense and sparse chunks
        for c in range(0, n, 2048):
            fb[c:c + 1024] = 1
    blob = orc.encode(keys, 127, force_break=fb, slope_mode=mode)
    assert orc.validate(blob) == 0
    assert _decode_equal(lc, blob, keys)


@pytest.mark.parametrize("eps", [0, 1, 2, 3, 7, 100, 4095, 65535, (1 << 31) - 1])
def test_decode_eps_extremes(lc, eps):
    """b from 0 (no residual words read) up to 32 bits (eps = 2^31 - 1)."""
    rng = np.random.default_rng(eps)
    keys = np.cumsum(rng.integers(1, 1 << 20, 50_000)).astype(np.uint64)
    blob = lc.encode(keys, eps)
    assert _decode_equal(lc, blob, keys)


def test_decode_top_of_range(lc):
    for kb, top in ((32, (1 << 32) - 1), (64, (1 << 64) - 1)):
        n = 5000
        gaps = np.random.default_rng(kb).integers(1, 1000, n - 1).astype(np.uint64)
        span = int(gaps.sum())
        keys = np.empty(n, np.uint64)
        keys[0] = top - span
        keys[1:] = np.uint64(top - span) + np.cumsum(gaps, dtype=np.uint64)
        keys = keys.astype(np.uint32) if kb == 32 else keys
        for eps in (0, 63, 255):
            assert _decode_equal(lc, lc.encode(keys, eps), keys)


def test_decode_single_key(lc):
    for dt in (np.uint32, np.uint64):
        keys = np.array([123456], dt)
        assert _decode_equal(lc, lc.encode(keys, 5), keys)


def test_decode_span_shards(lc):
    """Multi-GPU shard decode: spans at multiples of 1024 tile the output."""
    keys = make_keys(2, 300_000)
    blob = lc.encode(keys, 127)
    view = lc.View(blob, device=DEV)
    cuts = [0, 1024, 50 * 1024, 100 * 1024, 200 * 1024, 300_000]
    parts = [lc.decode_span(view, a, b) for a, b in zip(cuts, cuts[1:])]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), _dev(keys))
    with pytest.raises(lc.LcError):
        lc.decode_span(view, 1000, 2000)
    with pytest.raises(lc.LcError):
        lc.decode_span(view, 0, 300_001)


@pytest.mark.parametrize("n", [1_000_003, 20_000_007, 40_000_000])
def test_decode_host_e2e(lc, n):
    """lc_decode_host: its 4 Mi-key spans (and the ragged last one) tile the list exactly."""
    keys = make_keys(2, n)
    blob = lc.encode(keys, 127)
    h_blob = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
    d_blob = torch.empty(len(blob), dtype=torch.uint8, device=DEV)
    d_out = torch.empty(keys.size, dtype=torch.int64, device=DEV)
    h_out = torch.empty(keys.size, dtype=torch.int64).pin_memory()
    lc.decode_host(h_blob, d_blob, d_out, h_out)
    torch.cuda.synchronize()
    assert np.array_equal(h_out.numpy().view(np.uint64), keys)


# -------------------------------------------------------------- access and range (config 5)
def test_access_and_range_small(lc):
    keys, idx, rs = make_queries(n=500_000, q=200_000, r=20_000)
    blob = lc.encode(keys, 127)
    view = lc.View(blob, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    got = lc.access(view, _dev(idx), err=err)
    rg = lc.range_decode(view, _dev(rs), 64, err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert np.array_equal(_host(got, np.uint64), keys[idx.astype(np.int64)])
    want_r, e = orc.range_decode(blob, rs, 64)
    assert e == 0 and np.array_equal(_host(rg, np.uint64), want_r)


@pytest.mark.parametrize("length", [1, 31, 32, 33, 64, 1000])
def test_range_lengths(lc, length):
    keys = make_keys(3, 100_000)
    blob = lc.encode(keys, 255)
    view = lc.View(blob, device=DEV)
    rs = np.random.default_rng(length).integers(0, keys.size - length, 3000,
                                                endpoint=True).astype(np.uint64)
    rg = lc.range_decode(view, _dev(rs), length)
    want, _ = orc.range_decode(blob, rs, length)
    torch.cuda.synchronize()
    assert np.array_equal(_host(rg, np.uint64), want)


def test_access_range_errors(lc):
    keys = make_keys(5, 5000)
    blob = lc.encode(keys, 127)
    view = lc.View(blob, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    idx = np.array([0, 4999, 5000, 1 << 40], np.uint64)
    got = lc.access(view, _dev(idx), err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 1
    assert _host(got, np.uint64).tolist() == [int(keys[0]), int(keys[4999]), 0, 0]
    err.zero_()
    rs = np.array([0, 4936, 4937], np.uint64)
    rg = lc.range_decode(view, _dev(rs), 64, err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 1
    h = _host(rg, np.uint64)
    assert np.array_equal(h[0], keys[:64]) and np.array_equal(h[1], keys[4936:])
    assert not h[2].any()
    # q == 0 is a no-op
    lc.access(view, torch.empty(0, dtype=torch.int64, device=DEV))


def test_access_u32_keys(lc):
    keys = make_keys(1, 300_000)
    blob = lc.encode(keys, 63)
    view = lc.View(blob, device=DEV)
    idx = np.random.default_rng(1).integers(0, keys.size, 10_000).astype(np.uint64)
    got = lc.access(view, _dev(idx))
    rg = lc.range_decode(view, _dev(idx[:100] % np.uint64(keys.size - 64)), 64)
    torch.cuda.synchronize()
    assert np.array_equal(_host(got, np.uint32), keys[idx.astype(np.int64)])
    want, _ = orc.range_decode(blob, idx[:100] % np.uint64(keys.size - 64), 64)
    assert np.array_equal(_host(rg, np.uint32), want)


# ------------------------------------------------------------- full-size configs (bench sizes)
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_full_config(lc, cid):
    """Each BASELINE config at its full size, in the launch configuration bench.py times:
    decode == the generator's keys (every element, on device); sampled indices == oracle
    access computed one by one on the same blob."""
    keys = make_keys(cid)
    eps = CONFIGS[cid].eps
    blob = lc.encode(keys, eps)
    view = lc.View(blob, device=DEV)
    out = lc.decode(view)
    ref = _dev(keys)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    rng = np.random.default_rng(cid)
    idx = np.unique(np.concatenate([rng.integers(0, keys.size, 20_000),
                                    [0, keys.size - 1]])).astype(np.uint64)
    want, err = orc.access(blob, idx)
    assert err == 0
    assert np.array_equal(_host(out[torch.from_numpy(idx.view(np.int64)).to(DEV)], keys.dtype),
                          want)


def test_full_config5_access_range(lc):
    keys, idx, rs = make_queries()
    blob = lc.encode(keys, 127)
    view = lc.View(blob, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    d_keys = _dev(keys)
    d_idx = _dev(idx)
    got = lc.access(view, d_idx, err=err)
    assert torch.equal(got, d_keys[d_idx])
    del got
    d_rs = _dev(rs)
    rg = lc.range_decode(view, d_rs, 64, err=err)
    ar = d_rs[:, None] + torch.arange(64, device=DEV)[None, :]
    assert torch.equal(rg, d_keys[ar])
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    # sampled against the oracle one by one
    s_idx = idx[:5000]
    want, _ = orc.access(blob, s_idx)
    assert np.array_equal(_host(lc.access(view, _dev(s_idx)), np.uint64), want)


# ------------------------------------------------------------------ NEXT-1: quantiles
@pytest.mark.parametrize("cid,n", [(1, 300_000), (2, 1_000_003), (3, 500_000), (4, 700_001)])
def test_quantiles(lc, cid, n):
    keys = make_keys(cid, n)
    eps = CONFIGS[cid].eps
    blob = lc.encode(keys, eps)
    view = lc.View(blob, device=DEV)
    rng = np.random.default_rng(cid)
    for q in (1, 2, 100, 1_000_003, (1 << 32) - 1):
        ranks = np.unique(np.concatenate([rng.integers(0, q, 2000, endpoint=True), [0, q]]))
        ranks = ranks.astype(np.uint64)
        idx = np.array([orc.quantile_index(keys.size, int(k), q) for k in ranks], np.uint64)
        ex = lc.quantile(view, _dev(ranks), q, exact=True)
        ap = lc.quantile(view, _dev(ranks), q, exact=False)
        torch.cuda.synchronize()
        assert np.array_equal(_host(ex, keys.dtype), keys[idx.astype(np.int64)])
        want_ap, err = orc.predict(blob, idx)
        assert err == 0
        got_ap = _host(ap, keys.dtype)
        assert np.array_equal(got_ap, want_ap)
        diff = got_ap.astype(np.int64) - keys[idx.astype(np.int64)].astype(np.int64)
        assert np.abs(diff).max() <= eps


def test_quantile_errors(lc):
    keys = make_keys(5, 5000)
    view = lc.View(lc.encode(keys, 127), device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = lc.quantile(view, _dev(np.array([0, 5, 11], np.uint64)), 10, err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 1 and int(_host(out, np.uint64)[2]) == 0
    with pytest.raises(lc.LcError):
        lc.quantile(view, _dev(np.array([0], np.uint64)), 0)
    with pytest.raises(lc.LcError):
        lc.quantile(view, _dev(np.array([0], np.uint64)), 1 << 32)


# ------------------------------------------------ NEXT-2: successor search and intersection
from oracle import setops  # noqa: E402


def _probes(keys, rng, m):
    k = keys.astype(np.uint64)
    hits = k[rng.integers(0, k.size, m // 2)]
    lo, hi = int(k[0]), int(k[-1])
    top = (1 << 32) - 1 if keys.dtype == np.uint32 else (1 << 64) - 1
    a, b = max(lo - 10, 0), min(hi + 10, top)
    between = rng.integers(a, max(b, a + 1), m - m // 2, dtype=np.uint64, endpoint=True)
    return np.concatenate([hits, between, np.array([0, lo, hi, (1 << 64) - 1], np.uint64)])


@pytest.mark.parametrize("cid,n", [(1, 200_000), (2, 500_000), (3, 400_000), (4, 300_000), (5, 300_000)])
def test_next_geq(lc, cid, n):
    keys = make_keys(cid, n)
    view = lc.View(lc.encode(keys, CONFIGS[cid].eps), device=DEV)
    x = _probes(keys, np.random.default_rng(cid), 20_000)
    idx, key = lc.next_geq(view, _dev(x))
    torch.cuda.synchronize()
    want_i, want_k = setops.next_geq(keys, x)
    assert np.array_equal(_host(idx, np.uint64), want_i)
    assert np.array_equal(_host(key, keys.dtype), want_k)


@pytest.mark.parametrize("seed", range(3000, 3040))
def test_next_geq_fuzz(lc, seed):
    keys, eps, kb, law = fuzz_case(seed, n_max=50_000)
    view = lc.View(lc.encode(keys, eps, kb), device=DEV)
    x = _probes(keys, np.random.default_rng(seed), 2000)
    idx, key = lc.next_geq(view, _dev(x))
    torch.cuda.synchronize()
    want_i, want_k = setops.next_geq(keys, x)
    assert np.array_equal(_host(idx, np.uint64), want_i), (seed, law)
    assert np.array_equal(_host(key, keys.dtype), want_k), (seed, law)


def _isect_case(lc, a, b, eps_a, eps_b):
    va = lc.View(lc.encode(a, eps_a), device=DEV)
    vb = lc.View(lc.encode(b, eps_b), device=DEV)
    out, cnt = lc.intersect(va, vb)
    torch.cuda.synchronize()
    c = int(cnt.item())
    want = setops.intersect(a, b)
    assert c == want.size
    assert np.array_equal(_host(out[:c], a.dtype), want)


@pytest.mark.parametrize("na", [1, 1000, 33_333, 300_000])
def test_intersect_subset_plus_noise(lc, na):
    b = make_keys(2, 1_000_000)
    rng = np.random.default_rng(na)
    pick = b[np.sort(rng.choice(b.size, na // 2 + 1, replace=False))]
    noise = rng.integers(0, int(b[-1]) + 1000, na, dtype=np.uint64)
    a = np.unique(np.concatenate([pick, noise]))[:na]
    _isect_case(lc, a, b, 63, 127)
    _isect_case(lc, b, a, 127, 63)  # longer list first: decoded / searched roles swap inside


def test_intersect_closed_form_and_edges(lc):
    M = 3_000_000
    a = np.arange(0, M, 6, dtype=np.uint64)
    b = np.arange(0, M, 10, dtype=np.uint64)
    _isect_case(lc, a, b, 0, 31)                     # multiples of 30
    _isect_case(lc, b, b, 127, 127)                  # identical lists
    _isect_case(lc, a + np.uint64(1), a, 7, 7)       # disjoint
    a32 = np.arange(5, 2_000_000, 3, dtype=np.uint32)
    b32 = make_keys(1, 1_000_000)
    _isect_case(lc, a32, b32, 15, 63)                # u32 lists, a longer than b


def test_intersect_key_width_mismatch(lc):
    va = lc.View(lc.encode(np.arange(10, dtype=np.uint32), 1), device=DEV)
    vb = lc.View(lc.encode(np.arange(10, dtype=np.uint64), 1), device=DEV)
    with pytest.raises(lc.LcError):
        lc.intersect(va, vb)


def test_full_config5_quantile_next_geq(lc):
    """NEXT-1/NEXT-2 at the config-5 size (1e8 keys): 1e6 quantiles and 1e6 successor probes,
    every answer checked (exact quantiles / next_geq vs the key array, approximate quantiles vs
    the oracle's prediction)."""
    keys = make_keys(5)
    blob = lc.encode(keys, 127)
    view = lc.View(blob, device=DEV)
    rng = np.random.default_rng(5)
    q = (1 << 32) - 1
    ranks = rng.integers(0, q, 1_000_000, endpoint=True).astype(np.uint64)
    idx = np.minimum((ranks.astype(object) * keys.size) // q, keys.size - 1).astype(np.int64)
    ex = _host(lc.quantile(view, _dev(ranks), q), np.uint64)
    assert np.array_equal(ex, keys[idx])
    ap = _host(lc.quantile(view, _dev(ranks), q, exact=False), np.uint64)
    want_ap, _ = orc.predict(blob, idx[:20_000].astype(np.uint64))
    assert np.array_equal(ap[:20_000], want_ap)
    assert np.abs(ap.astype(np.int64) - keys[idx].astype(np.int64)).max() <= 127
    x = _probes(keys, rng, 1_000_000)
    gi, gk = lc.next_geq(view, _dev(x))
    wi, wk = setops.next_geq(keys, x)
    assert np.array_equal(_host(gi, np.uint64), wi) and np.array_equal(_host(gk, np.uint64), wk)


@pytest.mark.parametrize("free", [False, True])
@pytest.mark.parametrize("cid,n", [(1, 300_000), (2, 400_003), (3, 500_000), (4, 700_001), (5, 300_000)])
def test_search_index(lc, cid, n, free):
    """lc_search_index_build: the index holds each segment's first key K[s_j] (checked against
    the generator's keys at the blob's segment starts), and next_geq / intersect / union give
    the same answers with the index attached as the oracle's set definitions."""
    from tests import blobparse
    keys = make_keys(cid, n)
    eps = CONFIGS[cid].eps
    blob = lc.encode(keys, eps, free=free)
    view = lc.View(blob, device=DEV)
    idx = _host(view.build_search_index(), np.uint64)
    starts = blobparse.parse(blob).starts[:-1].astype(np.int64)
    L = starts.size
    assert np.array_equal(idx[:L], keys[starts].astype(np.uint64))
    off = (L + 31) // 32 * 32  # then the sample: every 16th first key
    assert np.array_equal(idx[off: off + (L + 15) // 16], keys[starts[::16]].astype(np.uint64))
    rng = np.random.default_rng(cid)
    x = _probes(keys, rng, 200_000)
    gi, gk = lc.next_geq(view, _dev(x))
    wi, wk = setops.next_geq(keys, x)
    assert np.array_equal(_host(gi, np.uint64), wi) and np.array_equal(_host(gk, keys.dtype), wk)
    a = np.unique(np.concatenate([keys[rng.integers(0, keys.size, n // 20)],
                                  rng.integers(0, int(keys[-1]) + 10, n // 20).astype(keys.dtype)]))
    va = lc.View(lc.encode(a, 31), device=DEV)
    out, cnt = lc.intersect(va, view)
    uo, uc = lc.union(va, view)
    torch.cuda.synchronize()
    wi_, wu_ = setops.intersect(a, keys), setops.union(a, keys)
    assert int(cnt.item()) == wi_.size and np.array_equal(_host(out[: wi_.size], keys.dtype), wi_)
    assert int(uc.item()) == wu_.size and np.array_equal(_host(uo[: wu_.size], keys.dtype), wu_)


def test_full_config5_intersect_union(lc):
    """NEXT-2 at the bench's size: a 1e6-key list (half drawn from config 5's keys, half
    uniform in its key range) intersected with and united with the full 1e8-key config-5 list,
    anchored (F4) and free-intercept (F7) long lists, without and with the successor-search
    index (plus 1e6 next_geq probes through the index), every output key checked against the
    oracle's set definitions."""
    k5 = make_keys(5)
    rng = np.random.default_rng(55)
    na = 1_000_000
    a = np.unique(np.concatenate([k5[np.sort(rng.choice(k5.size, na // 2, replace=False))],
                                  rng.integers(0, int(k5[-1]), na // 2, dtype=np.uint64)]))
    va = lc.View(lc.encode(a, 127), device=DEV)
    want_i = setops.intersect(a, k5)
    want_u = setops.union(a, k5)
    for free in (False, True):
        vb = lc.View(lc.encode(k5, 127, free=free), device=DEV)
        out, cnt = lc.intersect(va, vb)
        torch.cuda.synchronize()
        c = int(cnt.item())
        assert c == want_i.size and np.array_equal(_host(out[:c], np.uint64), want_i)
        for x, y in ((va, vb), (vb, va)):
            out, cnt = lc.union(x, y)
            torch.cuda.synchronize()
            c = int(cnt.item())
            assert c == want_u.size and np.array_equal(_host(out[:c], np.uint64), want_u)
        vb.build_search_index()  # same answers through the successor-search index
        out, cnt = lc.intersect(va, vb)
        torch.cuda.synchronize()
        c = int(cnt.item())
        assert c == want_i.size and np.array_equal(_host(out[:c], np.uint64), want_i)
        out, cnt = lc.union(va, vb)
        torch.cuda.synchronize()
        c = int(cnt.item())
        assert c == want_u.size and np.array_equal(_host(out[:c], np.uint64), want_u)
        x = _probes(k5, rng, 1_000_000)
        gi, gk = lc.next_geq(vb, _dev(x))
        wi, wk = setops.next_geq(k5, x)
        assert np.array_equal(_host(gi, np.uint64), wi) and np.array_equal(_host(gk, np.uint64), wk)
        del vb, out


def _union_case(lc, a, b, eps_a, eps_b):
    va = lc.View(lc.encode(a, eps_a), device=DEV)
    vb = lc.View(lc.encode(b, eps_b), device=DEV)
    out, cnt = lc.union(va, vb)
    torch.cuda.synchronize()
    c = int(cnt.item())
    want = setops.union(a, b)
    assert c == want.size
    assert np.array_equal(_host(out[:c], a.dtype), want)


@pytest.mark.parametrize("na", [1, 1000, 33_333, 300_000])
def test_union_subset_plus_noise(lc, na):
    b = make_keys(2, 500_000)
    rng = np.random.default_rng(na + 1)
    pick = b[np.sort(rng.choice(b.size, na // 2 + 1, replace=False))]
    noise = rng.integers(0, int(b[-1]) + 1000, na, dtype=np.uint64)
    a = np.unique(np.concatenate([pick, noise]))[:na]
    _union_case(lc, a, b, 63, 127)
    _union_case(lc, b, a, 127, 63)


def test_union_closed_form_and_edges(lc):
    M = 2_000_000
    a = np.arange(0, M, 6, dtype=np.uint64)
    b = np.arange(0, M, 10, dtype=np.uint64)
    _union_case(lc, a, b, 0, 31)
    _union_case(lc, b, b, 127, 127)                  # identical lists
    _union_case(lc, a + np.uint64(1), a, 7, 7)       # disjoint, interleaved
    _union_case(lc, a, a + np.uint64(M), 7, 7)       # disjoint, b entirely after a
    _union_case(lc, np.array([5], np.uint64), np.array([5], np.uint64), 1, 1)
    a32 = np.arange(5, 2_000_000, 3, dtype=np.uint32)
    _union_case(lc, a32, make_keys(1, 1_000_000), 15, 63)


def _union_fused_case(lc, a, b, eps_a=31, eps_b=127, free=False):
    """a short (fused path: |a| * 8 <= |b|), checked in both argument orders."""
    assert a.size * 8 <= b.size
    _union_case_v(lc, lc.View(lc.encode(a, eps_a), device=DEV),
                  lc.View(lc.encode(b, eps_b, free=free), device=DEV), a, b)


def _union_case_v(lc, va, vb, a, b):
    want = setops.union(a, b)
    for x, y in ((va, vb), (vb, va)):
        out, cnt = lc.union(x, y)
        torch.cuda.synchronize()
        c = int(cnt.item())
        assert c == want.size
        assert np.array_equal(_host(out[:c], a.dtype), want)


@pytest.mark.parametrize("free", [False, True])
def test_union_fused_insertion_patterns(lc, free):
    """lc_union's fused path (short list <= 1/8 of the long one): the long list is decoded once
    with every key shifted by the number of absent short-list keys below it.  Cases: insertions
    spread thin (<= 32 per 1024-key chunk, held in registers), clustered (> 32 per chunk and
    > 32 per 32-key window: streamed), many absent keys between two consecutive long-list keys
    (equal ranks), absent keys below / above every long-list key (rank 0 / n), ranks exactly at
    chunk boundaries, long lists with n a multiple of 1024 and with a ragged tail."""
    rng = np.random.default_rng(11)
    for n in (1 << 16, 100_003):
        b = np.arange(n, dtype=np.uint64) * np.uint64(16) + np.uint64(1000)
        top = int(b[-1])
        # thin: random keys, about half present
        a = np.unique(np.concatenate([rng.choice(b, 300, replace=False),
                                      rng.integers(0, top + 5000, 300).astype(np.uint64)]))
        _union_fused_case(lc, a, b, free=free)
        # clustered: 2000 absent keys inside one 1024-key chunk's key range
        lo = int(b[5 * 1024 + 10])
        a = np.unique(rng.integers(lo, lo + 16 * 300, 2000).astype(np.uint64))
        a = a[a % 16 != 1000 % 16][: n // 10]
        _union_fused_case(lc, a, b, free=free)
        # equal ranks: all 15 absent keys between b[i] and b[i+1] for a few i (incl. chunk edges)
        gaps = [0, 1023, 1024, 2047, n // 2, n - 2]
        a = np.concatenate([b[i] + np.arange(1, 16, dtype=np.uint64) for i in gaps])
        _union_fused_case(lc, np.sort(a), b, free=free)
        # below and above everything, plus the key right before each chunk start (rank = 1024 h)
        edge = b[np.arange(1024, n, 1024)] - np.uint64(1)
        a = np.unique(np.concatenate([np.arange(0, 50, dtype=np.uint64), edge,
                                      np.uint64(top) + np.arange(1, 60, dtype=np.uint64)]))
        _union_fused_case(lc, a, b, free=free)
        # a subset of b (nothing inserted) and a single key
        _union_fused_case(lc, b[::9].copy(), b, free=free)
        _union_fused_case(lc, np.array([3], np.uint64), b, free=free)


def test_union_fused_u32_and_configs(lc):
    """Fused path on u32 keys (config 1) and on a config-5-like long list with several residual
    widths (b = 0, 5, 8, 13)."""
    rng = np.random.default_rng(12)
    b = make_keys(1, 1_000_000)
    a = np.unique(rng.integers(0, int(b[-1]) + 100, 60_000).astype(np.uint32))
    _union_fused_case(lc, a, b, 63, 63)
    b = make_keys(5, 400_000)
    a = np.unique(np.concatenate([b[rng.integers(0, b.size, 20_000)],
                                  rng.integers(0, int(b[-1]), 20_000).astype(np.uint64)]))
    for eps in (0, 17, 127, 4095):
        _union_fused_case(lc, a, b, 7, eps)


def test_max_size_u32(lc):
    """Maximum list size of the format (N = 2^32 - 1, FORMAT F1): u32 keys 0..N-1 at eps = 1,
    so residual bit offsets reach 8.6e9 (> 2^32) and key indices the top of the 32-bit range.
    Decode is checked element by element (in 2^28-key slices against arange on device);
    access, range and quantile probe both ends and 2^31."""
    N = (1 << 32) - 1
    keys = np.arange(N, dtype=np.uint32)
    blob = lc.encode(keys, 1)
    del keys
    view = lc.View(blob, device=DEV)
    out = view.out_tensor(N)
    lc.decode(view, out)
    step = 1 << 28
    for s in range(0, N, step):
        e = min(s + step, N)
        assert torch.equal(out[s:e], torch.arange(s, e, dtype=torch.int64, device=DEV).to(torch.int32)), s
    del out
    probe = [0, 1, (1 << 31) - 1, 1 << 31, N - 1025, N - 65, N - 2, N - 1]
    idx = np.array(probe, np.uint64)
    assert _host(lc.access(view, _dev(idx)), np.uint32).tolist() == probe
    rs = np.array([0, (1 << 31) - 32, N - 64], np.uint64)
    rg = _host(lc.range_decode(view, _dev(rs), 64), np.uint32)
    assert all(rg[r].tolist() == list(range(int(s), int(s) + 64)) for r, s in enumerate(rs))
    q = _host(lc.quantile(view, _dev(np.array([0, 1, 2], np.uint64)), 2), np.uint32)
    assert q.tolist() == [0, N // 2, N - 1]
    torch.cuda.empty_cache()


def test_concurrent_streams(lc):
    """The library is stateless (lc.h): decodes / accesses of different blobs on different
    streams, interleaved without synchronisation, each produce their own exact result."""
    lists = [(make_keys(2, 3_000_001), 127), (make_keys(4, 2_000_003), 31),
             (make_keys(1, 1_000_000), 63), (make_keys(3, 1_500_000), 255)]
    views = [lc.View(lc.encode(k, e), device=DEV) for k, e in lists]
    streams = [torch.cuda.Stream() for _ in lists]
    outs = [v.out_tensor(v.n) for v in views]
    idx = [torch.from_numpy(np.random.default_rng(i).integers(0, k.size, 100_000)).to(DEV)
           for i, (k, _) in enumerate(lists)]
    acc = [None] * len(lists)
    torch.cuda.synchronize()  # inputs were staged on the default stream
    for rep in range(3):
        for i, (v, s) in enumerate(zip(views, streams)):
            lc.decode(v, outs[i], stream=s)
            acc[i] = lc.access(v, idx[i], stream=s)
    torch.cuda.synchronize()
    for i, (k, _) in enumerate(lists):
        assert torch.equal(outs[i], _dev(k))
        assert np.array_equal(_host(acc[i], k.dtype), k[idx[i].cpu().numpy()])


def test_decode_host_two_threads(lc):
    """lc_decode_host from two host threads at once (its internal copy streams are shared)."""
    import threading
    cases = [make_keys(2, 9_000_000), make_keys(5, 7_000_000)]
    res = [None, None]

    def run(t):
        keys = cases[t]
        blob = lc.encode(keys, 127)
        s = torch.cuda.Stream()
        h_blob = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
        d_blob = torch.empty(len(blob), dtype=torch.uint8, device=DEV)
        d_out = torch.empty(keys.size, dtype=torch.int64, device=DEV)
        h_out = torch.empty(keys.size, dtype=torch.int64).pin_memory()
        torch.cuda.synchronize()
        for _ in range(3):
            lc.decode_host(h_blob, d_blob, d_out, h_out, stream=s)
        s.synchronize()
        res[t] = np.array_equal(h_out.numpy().view(np.uint64), keys)

    th = [threading.Thread(target=run, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert res == [True, True]
