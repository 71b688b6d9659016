"""Host-side tests of the product library (no GPU): C-ABI exports, the C++ encoder's byte
equality with the oracle, the validator, error codes, and the oracle/product
boundary."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from oracle import native as orc
from synth import fuzz_case, make_keys
from tests import blobparse

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lc():
    from paper_2412_10770_b200 import _build
    _build.build()
    from paper_2412_10770_b200 import lc as m
    return m


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "lc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lc_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lc):
    names = _declared_functions()
    assert "lc_decode" in names and "lc_access" in names and "lc_range_decode" in names
    out = subprocess.check_output(["nm", "-D", "--defined-only", lc.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (lc_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(lc.EXPORTS)


def test_library_is_sm100a(lc):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lc.LIB_PATH],
                                  text=True)
    assert "sm_100a" in out


@pytest.mark.parametrize("seed", range(5000, 5150))
def test_blob_equals_oracle_fuzz(lc, seed):
    """P8: the product encoder and the oracle emit identical bytes (FORMAT F4/F5 are normative)."""
    keys, eps, kb, law = fuzz_case(seed, n_max=20_000)
    a = lc.encode(keys, eps, kb)
    b = orc.encode(keys, eps, kb)
    assert a == b, (seed, law)
    assert lc.validate(a) == 0


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_blob_equals_oracle_configs_small(lc, cid):
    keys = make_keys(cid, 200_000 if cid != 1 else None)
    eps = {1: 63, 2: 127, 3: 255, 4: 31, 5: 127}[cid]
    a = lc.encode(keys, eps)
    assert a == orc.encode(keys, eps)
    bl = blobparse.parse(a)
    assert len(a) == blobparse.expected_size(keys.size, bl.L, bl.b)


def test_overflow_and_extremes_equal(lc):
    cases = [
        (np.array([0, (1 << 31) - 1, 1 << 32], np.uint64), 0),
        (np.array([0, 1 << 31, (1 << 32) + 5], np.uint64), 0),
        (np.array([0, 1, 2, 1 << 40, (1 << 64) - 6, (1 << 64) - 2, (1 << 64) - 1], np.uint64), 255),
        (np.array([5], np.uint64), 3),
        (np.array([0xFFFFFFFF], np.uint32), 0),
        (np.arange(5000, dtype=np.uint64) * np.uint64(1 << 20), 0),
        (np.arange(5000, dtype=np.uint64) * np.uint64(1 << 20), (1 << 31) - 1),
    ]
    for keys, eps in cases:
        assert lc.encode(keys, eps) == orc.encode(keys, eps), (keys[:3], eps)


def test_encode_errors(lc):
    def code(fn):
        with pytest.raises(lc.LcError) as e:
            fn()
        return e.value.code
    assert code(lambda: lc.encode(np.zeros(0, np.uint64), 3)) == lc.LC_ERR_EMPTY
    assert code(lambda: lc.encode(np.array([1, 5, 5], np.uint64), 3)) == lc.LC_ERR_UNSORTED
    assert code(lambda: lc.encode(np.array([9, 3], np.uint64), 3)) == lc.LC_ERR_UNSORTED
    assert code(lambda: lc.encode(np.array([1, 2], np.uint64), 1 << 31)) == lc.LC_ERR_ARG
    assert code(lambda: lc.encode(np.array([1, 1 << 33], np.uint64), 3, 32)) == lc.LC_ERR_TOO_LARGE
    assert code(lambda: lc.encode(np.array([1, 2], np.uint64), 3, 16)) == lc.LC_ERR_ARG


def test_validator_agrees_with_oracle(lc):
    keys = make_keys(5, 7000)
    blob = lc.encode(keys, 127)
    bl = blobparse.parse(blob)

    def put(off, val):
        b = bytearray(blob)
        b[off:off + len(val)] = val
        return bytes(b)

    variants = [
        blob, blob[:-4], put(0, b"ZZZZ"), put(4, b"\x07"), put(7, b"\x03"), put(12, b"\x0b"),
        put(bl.o_starts + 4, np.uint32(0).tobytes()),
        put(bl.o_starts + 4 * bl.L, np.uint32(keys.size + 1).tobytes()),
        put(bl.o_hint, np.uint32(3).tobytes()),
        put(bl.o_params + 24, np.uint64((1 << 63) - 1).tobytes()),
        put(bl.o_words, np.uint32(0xFFFFFFFF).tobytes()),
        put(bl.o_words + 4 * bl.W - 4, b"\x80"),
        put(200, b"\x01"),
        put(bl.o_words, np.uint32(int(bl.words[0]) ^ 1).tobytes()),  # anchor field u_0 != eps
        put(bl.o_params, np.uint64(int(bl.base[0]) + 1).tobytes()),  # shifted base: still valid
    ]
    for i, v in enumerate(variants):
        want = orc.validate(v)
        got = lc.validate(v)
        assert (got == 0) == (want == 0), (i, got, want)
        if want:
            assert got == lc.LC_ERR_FORMAT, i


def test_header_struct_matches_format(lc):
    keys = make_keys(1, 5000)
    blob = lc.encode(keys, 63)
    h = lc.header(blob)
    bl = blobparse.parse(blob)
    assert h.magic == b"LCG1" and h.version == 1 and h.key_bits == 32 and h.res_bits == 7
    assert (h.n, h.n_seg, h.n_hint, h.n_words) == (bl.n, bl.L, bl.n_hint, bl.W)
    assert (h.off_starts, h.off_params, h.off_hint, h.off_words, h.total_bytes) == (
        bl.o_starts, bl.o_params, bl.o_hint, bl.o_words, len(blob))


@pytest.mark.parametrize("n", [2, 17, 5000, 70_001])
def test_view_and_search_index_sizes(lc, n):
    """lc_view_init leaves the search index detached; lc_search_index_bytes = the L first keys
    padded to 32 entries plus ceil(L/16) samples (8 bytes each); lc_search_index_build rejects a
    null or misaligned buffer before touching the device.  No device memory is dereferenced
    (the view's device pointer is only recorded)."""
    import ctypes as C
    keys = make_keys(2, n)
    blob = lc.encode(keys, 127)
    L = lc.header(blob).n_seg
    v = lc.lc_view()
    host = np.frombuffer(blob, np.uint8)
    assert lc._lib.lc_view_init(C.byref(v), host.ctypes.data, 1 << 20, host.nbytes) == 0
    assert v.d_first is None
    assert lc._lib.lc_search_index_bytes(C.byref(v)) == 8 * ((L + 31) // 32 * 32 + (L + 15) // 16)
    assert lc._lib.lc_search_index_build(C.byref(v), None, None) == -1
    assert lc._lib.lc_search_index_build(C.byref(v), 1 << 20 | 8, None) == -1
    assert v.d_first is None
    assert lc._lib.lc_view_init(C.byref(v), host.ctypes.data, (1 << 20) + 8, host.nbytes) == -1


# ------------------------------------------------------------ FORMAT F7 (NEXT-3, free intercept)
@pytest.mark.parametrize("seed", range(5000, 5120))
def test_free_blob_equals_oracle_fuzz(lc, seed):
    """The product's free-intercept encoder (line envelopes + witness cone) emits the same
    bytes as the oracle's per-intercept brute force (FORMAT F7 is normative)."""
    keys, eps, kb, law = fuzz_case(seed, n_max=8_000)
    eps = min(eps, 4095)  # the oracle is O(N eps)
    a = lc.encode(keys, eps, kb, free=True)
    assert a == orc.encode(keys, eps, kb, free=True), (seed, law, eps)
    assert lc.validate(a) == 0 and lc.header(a).flags == lc.LC_FLAG_FREE_INTERCEPT


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_free_blob_equals_oracle_configs_small(lc, cid):
    keys = make_keys(cid, 300_000 if cid != 1 else None)
    eps = {1: 63, 2: 127, 3: 255, 4: 31, 5: 127}[cid]
    a = lc.encode(keys, eps, free=True)
    assert a == orc.encode(keys, eps, free=True)
    bl = blobparse.parse(a)
    assert bl.flags == 1
    assert len(a) == blobparse.expected_size(keys.size, bl.L, bl.b)


def test_free_extremes(lc):
    """Large eps (up to 2^30 - 1, where the oracle's O(N eps) scan is out of reach) is checked
    by round trip through the oracle's decoder and both validators; small-eps extremes by bytes."""
    rng = np.random.default_rng(77)
    for trial in range(60):
        n = int(rng.integers(1, 2000))
        eps = int(rng.choice([0, 1, 3, (1 << 20) - 1, 1 << 29, (1 << 30) - 1]))
        gmax = int(rng.choice([2, 1000, 1 << 20, 1 << 31, 1 << 40]))
        g = rng.integers(1, gmax, n, endpoint=True).astype(np.uint64)
        k = np.cumsum(g, dtype=np.uint64)
        top = (1 << 64) - 1 - int(g.sum()) - 1
        k = k + np.uint64(top if trial % 3 == 0 else int(rng.integers(0, 1 << 40)))
        k = np.unique(k)
        b = lc.encode(k, eps, free=True)
        assert lc.validate(b) == 0 and orc.validate(b) == 0, trial
        assert np.array_equal(orc.decode(b), k), trial
        if eps <= 3:
            assert b == orc.encode(k, eps, free=True), trial
    for keys, eps in [(np.array([5], np.uint64), 3), (np.array([0xFFFFFFFF], np.uint32), 0),
                      (np.array([0, 1, 2, 3], np.uint32), 2),
                      (np.arange(5000, dtype=np.uint64) * np.uint64(1 << 20), 0)]:
        assert lc.encode(keys, eps, free=True) == orc.encode(keys, eps, free=True)


def test_free_encode_errors_and_validator(lc):
    with pytest.raises(lc.LcError) as e:
        lc.encode(np.array([1, 2], np.uint64), 1 << 30, free=True)
    assert e.value.code == lc.LC_ERR_ARG
    keys = make_keys(5, 7000)
    blob = lc.encode(keys, 127, free=True)
    bl = blobparse.parse(blob)

    def put(off, val):
        b = bytearray(blob)
        b[off:off + len(val)] = val
        return bytes(b)

    variants = [
        blob,
        put(88, b"\x02"),                                   # unknown flag bit
        put(88, b"\x00"),                                   # read as anchored: anchor/bias break
        put(8, np.uint32(1 << 30).tobytes()),               # eps above the F7 limit
        put(bl.o_params, np.uint64(int(bl.base[0]) + 1).tobytes()),
        put(bl.o_params + 16, np.uint64(int(bl.base[1]) + 10**6).tobytes()),
        put(bl.o_words, np.uint32(int(bl.words[0]) ^ 1).tobytes()),
    ]
    for i, v in enumerate(variants):
        want = orc.validate(v)
        got = lc.validate(v)
        assert (got == 0) == (want == 0), (i, got, want)
    assert lc.validate(variants[0]) == 0 and lc.validate(variants[1]) != 0


def test_product_never_touches_oracle():
    """The product path must not import, load or call anything under oracle/ (task ②/③)."""
    pkg = os.path.join(ROOT, "paper_2412_10770_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                bad = re.findall(r"import oracle|from oracle|liblc_oracle|lc_oracle|"
                                 r"oracle_[a-z_]+\(|oracle\.native|oracle\.pyref", src)
                assert not bad, (f, bad)


def test_oracle_never_touches_product():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "oracle")):
        for f in files:
            if f.endswith((".py", ".c", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import paper_2412_10770_b200" not in src
                assert "from paper_2412_10770_b200" not in src
                assert "liblc.so" not in src
                assert "lc_kernels" not in src
