"""Sharded decode: the host-side shard planning of lc_shard_bytes /
lc_decode_host on CPU (no device memory is touched), and on the GPU (-m gpu) shard views that
hold only their span's slices, decoded independently, including two processes on one GPU that
reassemble the list over gloo.

The shard of keys [i0, i1) is defined in include/lc.h from FORMAT F2: hint[i0/1024 ..
ceil(i1/1024)], the segments hint[i0/1024] .. hint[ceil(i1/1024)] (starts and params), and the
residual words [i0 b/32, i1 b/32 + 1)."""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch

from synth import CONFIGS, make_keys
from tests.blobparse import parse


@pytest.fixture(scope="module")
def lc():
    from paper_2412_10770_b200 import lc as _lc
    return _lc


def _shard_bytes(lc, blob, i0, i1):
    nb = C.c_uint64()
    rc = lc._lib.lc_shard_bytes(blob, len(blob), i0, i1, C.byref(nb))
    return rc, int(nb.value)


def _r256(x):
    return (x + 255) // 256 * 256


def _expected_shard_bytes(blob, i0, i1):
    """The slices named in include/lc.h, recomputed from the raw sections (tests/blobparse)."""
    bl = parse(blob)
    c0, c1 = i0 // 1024, (i1 + 1023) // 1024
    j0, j1 = int(bl.hint[c0]), int(bl.hint[c1])
    L = bl.L
    s_lo, s_hi = j0 // 4 * 4, min((j1 + 2 + 3) // 4 * 4, (L + 1 + 3) // 4 * 4)
    p_lo, p_hi = j0 // 4 * 4, j1 + 1
    w = 0 if bl.b == 0 else min(c1 * 32 * bl.b + 4, bl.W) - c0 * 32 * bl.b
    return (_r256(4 * (c1 - c0 + 1)) + _r256(4 * (s_hi - s_lo)) + _r256(16 * (p_hi - p_lo))
            + _r256(4 * w))


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_bytes_cover_the_span(lc, cid, world):
    from paper_2412_10770_b200.shard import shard_spans
    keys = make_keys(cid, 200_003)
    blob = lc.encode(keys, CONFIGS[cid].eps)
    bl = parse(blob)
    total = 0
    for i0, i1 in shard_spans(keys.size, world):
        rc, nb = _shard_bytes(lc, blob, i0, i1)
        assert rc == 0
        assert nb == _expected_shard_bytes(blob, i0, i1)
        # the span's segments are inside the shard: [hint[c0], hint[c1]] covers keys [i0, i1)
        c0, c1 = i0 // 1024, (i1 + 1023) // 1024
        j0, j1 = int(bl.hint[c0]), int(bl.hint[c1])
        assert bl.starts[j0] <= i0 and (j1 + 1 == bl.L or bl.starts[j1 + 1] >= min(i1, keys.size))
        total += nb
    if world > 1:
        # every shard is much smaller than the blob; together about one blob plus alignment
        assert total < len(blob) + world * 4 * 256 + world * 16 * 4 * 256
    assert total >= len(blob) - bl.o_starts - 256


def test_shard_bytes_errors(lc):
    keys = make_keys(2, 50_000)
    blob = lc.encode(keys, 127)
    n = keys.size
    assert _shard_bytes(lc, blob, 1, 2048)[0] == lc.LC_ERR_ARG     # i0 not a multiple of 1024
    assert _shard_bytes(lc, blob, 0, n + 1)[0] == lc.LC_ERR_ARG     # past the end
    assert _shard_bytes(lc, blob, 1024, 1024)[0] == lc.LC_ERR_ARG   # empty
    assert _shard_bytes(lc, blob[:100], 0, n)[0] == lc.LC_ERR_FORMAT
    bl = parse(blob)
    for bad in (bl.L, 0xFFFFFFFF):  # a hint past the last segment
        b2 = bytearray(blob)
        np.frombuffer(b2, np.uint32, bl.n_hint, bl.o_hint)[5] = bad
        assert _shard_bytes(lc, bytes(b2), 0, n)[0] == lc.LC_ERR_FORMAT
        assert _shard_bytes(lc, bytes(b2), 8 * 1024, n)[0] == 0  # slice without it is fine
    b2 = bytearray(blob)
    h = np.frombuffer(b2, np.uint32, bl.n_hint, bl.o_hint)
    h[7] = h[6] - 1 if h[6] else 1  # not non-decreasing
    h[6] = max(int(h[6]), 1)
    assert _shard_bytes(lc, bytes(b2), 0, n)[0] == lc.LC_ERR_FORMAT


def test_decode_host_rejects_corrupt_hint_before_any_copy(lc):
    """lc_decode_host sizes its uploads from the hint values: a corrupt hint must fail with
    LC_ERR_FORMAT before anything is enqueued (fake device pointers are never touched)."""
    keys = make_keys(2, 50_000)
    blob = bytearray(lc.encode(keys, 127))
    bl = parse(bytes(blob))
    np.frombuffer(blob, np.uint32, bl.n_hint, bl.o_hint)[3] = 0xFFFFFFF0
    hb = (C.c_char * len(blob)).from_buffer(blob)
    fake = C.c_void_p(1 << 40)  # 256-byte aligned, never dereferenced
    rc = lc._lib.lc_decode_host(C.addressof(hb), len(blob), fake, fake, C.addressof(hb), None)
    assert rc == lc.LC_ERR_FORMAT


# ----------------------------------------------------------------------------------- GPU
DEV = "cuda:0"


def _dev(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype.itemsize == 8 else a.view(np.int32)).to(DEV)


@pytest.mark.gpu
@pytest.mark.parametrize("cid,n", [(1, 1_000_000), (2, 1_000_003), (3, 700_001), (4, 2_000_000),
                                   (5, 300_000)])
@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_shard_views_decode(lc, cid, n, world):
    from paper_2412_10770_b200 import shard
    keys = make_keys(cid, n)
    blob = lc.encode(keys, CONFIGS[cid].eps)
    ref = _dev(keys)
    for r in range(world):
        v, (i0, i1) = shard.upload_shard(blob, r, world, device=DEV)
        if v is None:
            continue
        assert v.d_blob.numel() == lc.View.shard_bytes(blob, i0, i1)
        out, span = shard.decode_shard(v, r, world)
        torch.cuda.synchronize()
        assert span == (i0, i1)
        assert torch.equal(out, ref[i0:i1])
        # a sub-span inside the shard (1024-aligned start), and one reaching outside
        if i1 - i0 > 2048:
            sub = lc.decode_span(v, i0 + 1024, i1 - 5)
            torch.cuda.synchronize()
            assert torch.equal(sub, ref[i0 + 1024:i1 - 5])
        outside = [(i0, i1 + 1)] if i1 < keys.size else []
        outside += [(i0 - 1024, i1)] if i0 >= 1024 else []
        for a, b in outside:
            with pytest.raises(lc.LcError):
                lc.decode_span(v, a, b)


@pytest.mark.gpu
def test_shard_view_rejected_by_other_calls(lc):
    keys = make_keys(5, 100_000)
    blob = lc.encode(keys, 127)
    v = lc.View.shard(blob, 1024 * 10, 1024 * 60, device=DEV)
    idx = _dev(np.arange(10, dtype=np.uint64))
    for call in (lambda: lc.access(v, idx), lambda: lc.range_decode(v, idx, 64),
                 lambda: lc.quantile(v, idx, 100), lambda: lc.next_geq(v, idx),
                 lambda: v.build_search_index(), lambda: lc.intersect(v, v),
                 lambda: lc.union(v, v)):
        with pytest.raises(lc.LcError) as e:
            call()
        assert e.value.code == lc.LC_ERR_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [3, 4])
def test_full_config_sharded_8(lc, cid):
    """Bench-size lists cut into 8 shards (the strong-scaling path of bench.py --gpus 8), each
    uploaded alone and decoded: every key checked on device."""
    from paper_2412_10770_b200 import shard
    keys = make_keys(cid)
    blob = lc.encode(keys, CONFIGS[cid].eps)
    ref = _dev(keys)
    del keys
    tot = 0
    for r in range(8):
        v, (i0, i1) = shard.upload_shard(blob, r, 8, device=DEV)
        tot += v.d_blob.numel()
        out, _ = shard.decode_shard(v, r, 8)
        torch.cuda.synchronize()
        assert torch.equal(out, ref[i0:i1])
        del v, out
    assert tot < 1.01 * len(blob)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gpu_worker(rank, world, port, n, result_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_10770_b200 import lc as _lc
        from paper_2412_10770_b200 import shard
        keys = make_keys(4, n)
        blob = _lc.encode(keys, CONFIGS[4].eps)
        h_blob = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
        v, (i0, i1) = shard.upload_shard(h_blob, rank, world, device=DEV)
        out, _ = shard.decode_shard(v, rank, world)
        torch.cuda.synchronize()
        part = out.cpu()
        spans = shard.shard_spans(n, world)
        chunk = max(b - a for a, b in spans)
        buf = torch.zeros(chunk, dtype=torch.int64)
        buf[: part.numel()] = part
        bufs = [torch.zeros(chunk, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(bufs, buf)
        whole = np.concatenate([b.numpy()[: e - s] for b, (s, e) in zip(bufs, spans)])
        result_q.put((rank, bool(np.array_equal(whole.view(np.uint64), keys)),
                      int(v.d_blob.numel()), len(blob)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_shards_on_one_gpu():
    """Two processes (world size 2, gloo for the host-side reassembly only), each holding only
    its shard on the GPU (lc_shard_upload) and decoding it with its own kernels."""
    import torch.multiprocessing as mp
    world, n = 2, 3_000_000 + 777
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert all(r[2] < 0.6 * r[3] for r in res)  # each process holds about half the blob
