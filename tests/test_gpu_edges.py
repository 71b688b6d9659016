"""Edge cases of the CUDA path beyond the fuzz corpus (-m gpu):

* the sparse instantiation's single-segment fast path per 128-key quad (lc_decode.cuh), aimed
  at its boundaries: a segment start exactly at a quad's end (wb + 128), at 1024-key chunk
  edges, and N a multiple of 128 / 1024 so that clamped candidates repeat N;
* the largest residual stream of the format: N = 2^32 - 1 keys at b = 32 (eps = 2^31 - 1), so
  the words section holds W = 2^32 words (FORMAT F2: roundup4(ceil(N b / 32) + 1)) and word
  indices pass 2^32 - 1.  The blob is assembled directly from FORMAT F1/F2 (host sections,
  16 GiB of words filled on the device), not by the encoder: keys K[i] = i in two exact
  segments (slope 1, i.e. slope_fx = 2^32, the longest the F2 guard allows is 2^31 keys), every
  residual u = eps.
"""
from __future__ import annotations

import struct

import numpy as np
import pytest
import torch

from oracle import native as orc
from tests.blobparse import HEADER_FMT, align, parse

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def lc():
    from paper_2412_10770_b200 import lc as _lc
    return _lc


def _dev(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)).to(DEV)


@pytest.mark.parametrize("n", [128 * 40, 1024 * 9, 1024 * 9 + 128, 1024 * 9 + 1, 1024 * 9 + 127,
                               1024 * 33])
@pytest.mark.parametrize("brk", ["q128", "q1024", "q128_plus1", "q256_minus1", "none"])
def test_sparse_fast_path_edges(lc, n, brk):
    keys = (np.arange(n, dtype=np.uint64) * np.uint64(5) + np.uint64(11))
    keys[n // 2:] += np.uint64(3)  # one kink so the unforced fit is not one segment
    fb = np.zeros(n, np.uint8)
    if brk == "q128":
        fb[::128] = 1
    elif brk == "q1024":
        fb[::1024] = 1
    elif brk == "q128_plus1":
        fb[::128] = 1
        fb[129::1024] = 1
    elif brk == "q256_minus1":
        fb[255::256] = 1
    blob = orc.encode(keys, 2, force_break=fb if brk != "none" else None)
    bl = parse(blob)
    assert bl.L * 64 < n  # the sparse instantiation (< 1 segment per 64 keys) decodes it
    v = lc.View(blob, device=DEV)
    out = lc.decode(v)
    torch.cuda.synchronize()
    assert torch.equal(out, _dev(keys))
    assert np.array_equal(orc.decode(blob), keys)
    # spans starting at every chunk take the same path from a different first chunk
    for i0 in range(0, n, 1024 * 4):
        sp = lc.decode_span(v, i0, n)
        torch.cuda.synchronize()
        assert torch.equal(sp, _dev(keys[i0:]))


def _b32_blob_host(key_bits: int):
    """(host bytes of header + starts + params + hint, total blob bytes, words offset, W)."""
    N = (1 << 32) - 1
    eps = (1 << 31) - 1
    b = 32
    starts = np.array([0, 1 << 31, N], np.uint32)
    L = 2
    params = np.array([[0, 1 << 32], [1 << 31, 1 << 32]], np.uint64)  # base = K[s_j], slope 1
    H = (N + 1023) // 1024
    hint = np.where(np.arange(H + 1, dtype=np.int64) * 1024 >= (1 << 31), 1, 0).astype(np.uint32)
    hint[H] = L - 1
    W = ((N * b + 31) // 32 + 1 + 3) // 4 * 4
    o_s = 256
    o_p = align(o_s + 4 * (L + 1))
    o_h = align(o_p + 16 * L)
    o_w = align(o_h + 4 * (H + 1))
    total = o_w + 4 * W
    head = struct.pack(HEADER_FMT, b"LCG1", 1, key_bits, b, eps, 10, N, L, H + 1, W, o_s, o_p,
                       o_h, o_w, total, 0, bytes(36))
    host = bytearray(o_w)
    host[:128] = head
    host[o_s:o_s + starts.nbytes] = starts.tobytes()
    host[o_p:o_p + params.nbytes] = params.tobytes()
    host[o_h:o_h + hint.nbytes] = hint.tobytes()
    return bytes(host), total, o_w, W


@pytest.mark.parametrize("key_bits", [64, 32])
def test_max_words_b32(lc, key_bits):
    N = (1 << 32) - 1
    host, total, o_w, W = _b32_blob_host(key_bits)
    assert W == 1 << 32
    d = torch.empty(total, dtype=torch.uint8, device=DEV)
    d[:o_w].copy_(torch.frombuffer(bytearray(host), dtype=torch.uint8))
    words = d[o_w:].view(torch.int32)
    words.fill_((1 << 31) - 1)  # u_i = eps for every key
    words[N:].zero_()           # the pad word
    v = lc.View(np.frombuffer(host[:128], np.uint8).copy(), device=DEV, d_blob=d, blob_bytes=total)
    dt = torch.int64 if key_bits == 64 else torch.int32

    def want(a, b_):
        return torch.arange(a, b_, dtype=torch.int64, device=DEV).to(dt)

    # decode spans at the start, across the segment boundary 2^31 and at the very end
    for i0, i1 in [(0, 1 << 20), ((1 << 31) - (1 << 20), (1 << 31) + (1 << 20)),
                   (N - (N % 1024) - (1 << 22), N)]:
        out = lc.decode_span(v, i0, i1)
        torch.cuda.synchronize()
        assert torch.equal(out, want(i0, i1)), (i0, i1)
        del out
    probe = np.array([0, 1, (1 << 31) - 1, 1 << 31, N - 1025, N - 65, N - 2, N - 1], np.uint64)
    got = lc.access(v, _dev(probe))
    torch.cuda.synchronize()
    assert got.cpu().numpy().view(np.uint32 if key_bits == 32 else np.uint64).tolist() == \
        probe.tolist()
    rs = np.array([0, (1 << 31) - 32, N - 64, N - 1024], np.uint64)
    for ln in (64, 33):
        rg = lc.range_decode(v, _dev(rs), ln)
        torch.cuda.synchronize()
        for r, s in enumerate(rs.tolist()):
            assert torch.equal(rg[r], want(s, s + ln)), (ln, s)
    del d, words, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", ["sparse", "dense"])
@pytest.mark.parametrize("extra", [0, 1, 777, 8 * 1024 + 5])
def test_launch_shape_threshold(lc, kind, extra):
    """Launches just below and above the long-launch threshold (24 K chunks: the persistent grid
    drops to 2 / 3 CTAs per SM for u64 lists, lc_kernels.cu persistent_grid) with ragged tails:
    every key, and the same list decoded as spans that straddle the threshold."""
    from synth import make_keys
    n = 24 * 1024 * 1024 - 1024 + extra
    keys = make_keys(4 if kind == "sparse" else 2, n + 2048)
    blob = lc.encode(keys, 31 if kind == "sparse" else 127)
    bl = parse(blob)
    assert (bl.L * 64 < keys.size) == (kind == "sparse")
    v = lc.View(blob, device=DEV)
    ref = _dev(keys)
    out = lc.decode(v)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    for i0, i1 in ((0, n), (1024, n + 1024), (2048, keys.size), (0, 24 * 1024 * 1024 - 1)):
        part = lc.decode_span(v, i0, i1)
        torch.cuda.synchronize()
        assert torch.equal(part, ref[i0:i1]), (i0, i1)
