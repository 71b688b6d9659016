"""N > 1 host logic on CPU (gloo, world size 2, 127.0.0.1): shard planning at hint-block
boundaries, per-rank span decode (here with the oracle, the GPU path uses lc_decode_span on the
same spans), reassembly, and max-over-ranks timing."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_10770_b200.shard import max_over_ranks, shard_spans


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,world", [(1, 1), (1, 2), (1023, 2), (1024, 2), (1025, 2),
                                      (100_000, 3), (5 * 1024, 8), (3 * 1024 + 7, 4)])
def test_shard_spans_tile(n, world):
    spans = shard_spans(n, world)
    assert len(spans) == world
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    for i0, i1 in spans:
        assert (i0 % 1024 == 0 or i0 == i1 == n) and i0 <= i1
    sizes = [(i1 - i0 + 1023) // 1024 for i0, i1 in spans]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, n, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import native as orc
        from synth import make_keys
        keys = make_keys(3, n)
        blob = orc.encode(keys, 255)
        i0, i1 = shard_spans(n, world)[rank]
        part = orc.decode_span(blob, i0, i1)
        # pad to a common length for all_gather
        chunk = max(b - a for a, b in shard_spans(n, world))
        buf = torch.zeros(chunk, dtype=torch.int64)
        buf[: part.size] = torch.from_numpy(part.view(np.int64))
        bufs = [torch.zeros(chunk, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(bufs, buf)
        whole = np.concatenate([b.numpy()[: e - s] for b, (s, e) in zip(bufs, shard_spans(n, world))])
        ok = np.array_equal(whole.view(np.uint64), keys)
        tmax = max_over_ranks(0.5 + rank)
        result_q.put((rank, ok, tmax))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_decode_gloo():
    world, n = 2, 50_000 + 123
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [1.5, 1.5]  # max over ranks of (0.5, 1.5)
