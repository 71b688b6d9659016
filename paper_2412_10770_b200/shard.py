"""Multi-GPU host logic: full decode shards with no exchange step.

The key index space is cut at multiples of 1024 (hint-block boundaries, FORMAT F2), so every
shard is a legal `lc_decode_span`.  Each GPU uploads only its shard of the compressed blob
(`lc_shard_upload`: the span's hint, starts, params and residual-word slices; the straddling
segment is duplicated) and decodes it independently (§IV-E ① "reduce the data
dependencies ... to maximize parallelism").  No collective touches the data path;
`max_over_ranks` is only for timing.
"""
from __future__ import annotations

HINT_BLOCK = 1024


def shard_spans(n: int, world: int) -> list[tuple[int, int]]:
    """Split keys [0, n) into `world` spans [i0, i1) with i0 % 1024 == 0, as even as possible in
    1024-key chunks (the last span may be ragged; spans may be empty when world > chunks)."""
    if n < 0 or world < 1:
        raise ValueError("n >= 0 and world >= 1 required")
    chunks = (n + HINT_BLOCK - 1) // HINT_BLOCK
    base, extra = divmod(chunks, world)
    spans, c = [], 0
    for r in range(world):
        take = base + (1 if r < extra else 0)
        i0, i1 = min(c * HINT_BLOCK, n), min((c + take) * HINT_BLOCK, n)
        spans.append((i0, i1))
        c += take
    return spans


def upload_shard(h_blob, rank: int, world: int, device="cuda", stream=None):
    """This rank's shard view (lc_shard_upload): only the slices its span reads are copied to
    `device`.  Returns (view or None for an empty span, (i0, i1))."""
    from . import lc
    i0, i1 = shard_spans(int(lc.header(h_blob).n), world)[rank]
    if i0 == i1:
        return None, (i0, i1)
    return lc.View.shard(h_blob, i0, i1, device=device, stream=stream), (i0, i1)


def decode_shard(view, rank: int, world: int, out=None, stream=None):
    """Decode this rank's span of the list on its GPU: `view` is the rank's shard view
    (upload_shard) or a whole-blob view (lc_decode_span over the rank's span)."""
    from . import lc
    if view is None:  # empty span
        return None, (0, 0)
    i0, i1 = shard_spans(view.n, world)[rank]
    if view.v.span_hi and view.span != (i0, i1):
        raise ValueError(f"shard view holds {view.span}, rank {rank} of {world} needs {(i0, i1)}")
    return lc.decode_span(view, i0, i1, out=out, stream=stream), (i0, i1)


def max_over_ranks(seconds: float, device=None) -> float:
    """Max of a per-rank duration over the default process group (1 rank: identity)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(seconds)
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
