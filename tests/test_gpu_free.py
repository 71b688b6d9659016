"""GPU parity for FORMAT F7 blobs (free-intercept segments).

The same kernels run with the decode bias 0 (F3) and, for successor search / intersection, a
search over decoded first keys instead of the anchored bases.  Expected values come from the
generators' key arrays (Def. 1) and from the oracle's decode / predict of the same blob; the
blobs themselves are byte-equal to the oracle's (tests/test_host_library.py).
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import native as orc  # noqa: E402
from oracle import setops  # noqa: E402
from synth import CONFIGS, fuzz_case, make_keys, make_queries  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
EPS_MAX_FREE = (1 << 30) - 1


@pytest.fixture(scope="module")
def lc():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2412_10770_b200 import lc as m
    return m


def _dev(a: np.ndarray):
    a = np.ascontiguousarray(a)
    v = a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)
    return torch.from_numpy(v).to(DEV)


def _host(t, dtype):
    return t.cpu().numpy().view(dtype)


def _enc(lc, keys, eps, kb=None):
    blob = lc.encode(keys, eps, kb, free=True)
    assert lc.header(blob).flags == lc.LC_FLAG_FREE_INTERCEPT
    return blob


def _decode_equal(lc, blob, keys):
    out = lc.decode(lc.View(blob, device=DEV))
    torch.cuda.synchronize()
    return torch.equal(out, _dev(keys))


@pytest.mark.parametrize("seed", range(1000, 1150))
def test_free_decode_fuzz(lc, seed):
    keys, eps, kb, law = fuzz_case(seed, n_max=100_000)
    blob = _enc(lc, keys, min(eps, EPS_MAX_FREE), kb)
    assert _decode_equal(lc, blob, keys), (seed, law, keys.size, eps)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [2, 1025, 33_000, 262_145])
def test_free_decode_configs_small(lc, cid, n):
    keys = make_keys(cid, n)
    blob = _enc(lc, keys, CONFIGS[cid].eps)
    out = lc.decode(lc.View(blob, device=DEV))
    torch.cuda.synchronize()
    want = orc.decode(blob)
    assert np.array_equal(want, keys)
    assert np.array_equal(_host(out, keys.dtype), want)


@pytest.mark.parametrize("eps", [0, 1, 2, 100, 4095, 65535, 1 << 29, EPS_MAX_FREE])
def test_free_decode_eps_extremes(lc, eps):
    """b from 0 up to 31 bits (F7 stops at eps = 2^30 - 1)."""
    rng = np.random.default_rng(eps)
    keys = np.cumsum(rng.integers(1, 1 << 20, 50_000)).astype(np.uint64)
    assert _decode_equal(lc, _enc(lc, keys, eps), keys)


def test_free_decode_top_and_bottom_of_range(lc):
    """Keys ending at 2^w - 1 and keys starting at 0 (where beta - eps >= 0 restricts delta)."""
    for kb, top in ((32, (1 << 32) - 1), (64, (1 << 64) - 1)):
        n = 5000
        gaps = np.random.default_rng(kb).integers(1, 1000, n - 1).astype(np.uint64)
        span = int(gaps.sum())
        keys = np.empty(n, np.uint64)
        keys[0] = top - span
        keys[1:] = np.uint64(top - span) + np.cumsum(gaps, dtype=np.uint64)
        low = np.concatenate([[0], np.cumsum(gaps, dtype=np.uint64)]).astype(np.uint64)
        if kb == 32:
            keys, low = keys.astype(np.uint32), low.astype(np.uint32)
        for eps in (0, 63, 255):
            assert _decode_equal(lc, _enc(lc, keys, eps), keys)
            assert _decode_equal(lc, _enc(lc, low, eps), low)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_free_full_config(lc, cid):
    """Every full-size config encoded with F7: every element on device, 1e7 random accesses
    against the generator's keys on device, sampled indices against the oracle's access of the
    same blob."""
    keys = make_keys(cid)
    blob = _enc(lc, keys, CONFIGS[cid].eps)
    view = lc.View(blob, device=DEV)
    out = lc.decode(view)
    torch.cuda.synchronize()
    assert torch.equal(out, _dev(keys))
    rng = np.random.default_rng(cid)
    idx = np.unique(np.concatenate([rng.integers(0, keys.size, 20_000),
                                    [0, keys.size - 1]])).astype(np.uint64)
    want, err = orc.access(blob, idx)
    assert err == 0
    got = lc.access(view, _dev(idx))
    assert np.array_equal(_host(got, keys.dtype), want)
    d_idx = torch.from_numpy(rng.integers(0, keys.size, 10_000_000)).to(DEV)
    assert torch.equal(lc.access(view, d_idx), out[d_idx])


def test_free_access_range(lc):
    keys, idx, rs = make_queries(n=2_000_000, q=500_000, r=50_000)
    blob = _enc(lc, keys, 127)
    view = lc.View(blob, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    got = lc.access(view, _dev(idx), err=err)
    rg = lc.range_decode(view, _dev(rs), 64, err=err)
    rg33 = lc.range_decode(view, _dev(rs), 33, err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert np.array_equal(_host(got, np.uint64), keys[idx.astype(np.int64)])
    want_r, e = orc.range_decode(blob, rs, 64)
    assert e == 0 and np.array_equal(_host(rg, np.uint64), want_r)
    assert np.array_equal(_host(rg33, np.uint64).reshape(-1, 33), want_r[:, :33])


@pytest.mark.parametrize("cid,n", [(1, 300_000), (2, 1_000_003), (3, 500_000), (4, 700_001)])
def test_free_quantiles(lc, cid, n):
    """Exact = K[index]; approximate = floor(f(i)) = base + eps + floor(slope d / 2^32) for
    F7 (the oracle's predict), within eps of the key."""
    keys = make_keys(cid, n)
    eps = CONFIGS[cid].eps
    blob = _enc(lc, keys, eps)
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


def _probes(keys, rng, m):
    k = keys.astype(np.uint64)
    hits = k[rng.integers(0, k.size, m // 2)]
    lo, hi = int(k[0]), int(k[-1])
    top = (1 << 32) - 1 if keys.dtype == np.uint32 else (1 << 64) - 1
    a, b = max(lo - 10, 0), min(hi + 10, top)
    between = rng.integers(a, max(b, a + 1), m - m // 2, dtype=np.uint64, endpoint=True)
    return np.concatenate([hits, between, np.array([0, lo, hi, (1 << 64) - 1], np.uint64)])


@pytest.mark.parametrize("cid,n", [(1, 200_000), (2, 500_000), (3, 400_000), (4, 300_000), (5, 300_000)])
def test_free_next_geq(lc, cid, n):
    keys = make_keys(cid, n)
    view = lc.View(_enc(lc, keys, CONFIGS[cid].eps), device=DEV)
    x = _probes(keys, np.random.default_rng(cid), 20_000)
    idx, key = lc.next_geq(view, _dev(x))
    torch.cuda.synchronize()
    want_i, want_k = setops.next_geq(keys, x)
    assert np.array_equal(_host(idx, np.uint64), want_i)
    assert np.array_equal(_host(key, keys.dtype), want_k)


@pytest.mark.parametrize("seed", range(3000, 3030))
def test_free_next_geq_fuzz(lc, seed):
    keys, eps, kb, law = fuzz_case(seed, n_max=50_000)
    view = lc.View(_enc(lc, keys, min(eps, EPS_MAX_FREE), kb), device=DEV)
    x = _probes(keys, np.random.default_rng(seed), 2000)
    idx, key = lc.next_geq(view, _dev(x))
    torch.cuda.synchronize()
    want_i, want_k = setops.next_geq(keys, x)
    assert np.array_equal(_host(idx, np.uint64), want_i), (seed, law)
    assert np.array_equal(_host(key, keys.dtype), want_k), (seed, law)


@pytest.mark.parametrize("free_a,free_b", [(True, True), (False, True), (True, False)])
def test_free_intersect_union(lc, free_a, free_b):
    """Mixed formats: A decoded by its own bias, B searched by first keys (F7) or bases (F2)."""
    b = make_keys(2, 1_000_000)
    rng = np.random.default_rng(int(free_a) * 2 + int(free_b))
    pick = b[np.sort(rng.choice(b.size, 20_001, replace=False))]
    noise = rng.integers(0, int(b[-1]) + 1000, 40_000, dtype=np.uint64)
    a = np.unique(np.concatenate([pick, noise]))
    va = lc.View(lc.encode(a, 63, free=free_a), device=DEV)
    vb = lc.View(lc.encode(b, 127, free=free_b), device=DEV)
    out, cnt = lc.intersect(va, vb)
    uo, uc = lc.union(va, vb)
    torch.cuda.synchronize()
    want = setops.intersect(a, b)
    assert int(cnt.item()) == want.size
    assert np.array_equal(_host(out[:want.size], a.dtype), want)
    wu = setops.union(a, b)
    assert int(uc.item()) == wu.size
    assert np.array_equal(_host(uo[:wu.size], a.dtype), wu)


# ------------------------------------------------ fewest segments (LC_FLAG_MIN_SEGMENTS)
@pytest.mark.parametrize("seed", range(1200, 1240))
def test_min_segments_decode_fuzz(lc, seed):
    """Blobs of the fewest-segments option (segments shorter than the greedy ones at places)
    through every kernel family: decode, access, range."""
    keys, eps, kb, _ = fuzz_case(seed)
    for free in (False, True):
        if free and eps > EPS_MAX_FREE:
            continue
        blob = lc.encode(keys, eps, key_bits=kb, free=free, min_segments=True)
        assert _decode_equal(lc, blob, keys)


@pytest.mark.parametrize("cid", [1, 2, 5])
def test_min_segments_configs(lc, cid):
    keys = make_keys(cid, 400_001)
    for free in (False, True):
        blob = lc.encode(keys, CONFIGS[cid].eps, free=free, min_segments=True)
        v = lc.View(blob, device=DEV)
        out = lc.decode(v)
        idx = np.random.default_rng(cid).integers(0, keys.size, 20_000).astype(np.uint64)
        got = lc.access(v, _dev(idx))
        torch.cuda.synchronize()
        assert torch.equal(out, _dev(keys))
        assert np.array_equal(_host(got, keys.dtype), keys[idx.astype(np.int64)])
