"""Thin ctypes binding of the C ABI in include/lc.h (argument marshalling only).

Every step of the decode path runs inside liblc.so (host encoder in C++, decode / access /
range kernels in CUDA for sm_100a).  PyTorch is used only for device memory and streams.
There is no fallback: if liblc.so is missing this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# LC_LIB: developer override to A/B another build of the same sources (tools/ only)
LIB_PATH = os.environ.get("LC_LIB") or os.path.join(_PKG, "liblc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (nvcc, sm_100a)")

_lib = C.CDLL(LIB_PATH)

LC_OK, LC_ERR_ARG, LC_ERR_EMPTY, LC_ERR_UNSORTED = 0, -1, -2, -3
LC_ERR_TOO_LARGE, LC_ERR_FORMAT, LC_ERR_ALLOC, LC_ERR_CUDA = -4, -5, -6, -7
LC_FLAG_FREE_INTERCEPT = 1  # FORMAT F7
LC_FLAG_MIN_SEGMENTS = 2    # encoder option: fewest segments (not stored in the blob)


class lc_header(C.Structure):
    _fields_ = [
        ("magic", C.c_char * 4), ("version", C.c_uint16), ("key_bits", C.c_uint8),
        ("res_bits", C.c_uint8), ("eps", C.c_uint32), ("hint_log2", C.c_uint32),
        ("n", C.c_uint64), ("n_seg", C.c_uint64), ("n_hint", C.c_uint64), ("n_words", C.c_uint64),
        ("off_starts", C.c_uint64), ("off_params", C.c_uint64), ("off_hint", C.c_uint64),
        ("off_words", C.c_uint64), ("total_bytes", C.c_uint64), ("flags", C.c_uint32),
        ("reserved", C.c_uint8 * 36),
    ]


assert C.sizeof(lc_header) == 128


class lc_batch(C.Structure):
    _fields_ = [("m", C.c_uint32), ("key_bits", C.c_uint32), ("max_res_bits", C.c_uint32),
                ("sparse", C.c_uint32), ("n_total", C.c_uint64), ("n_chunks", C.c_uint64),
                ("n_small", C.c_uint64), ("small_keys", C.c_uint64), ("payload_bytes", C.c_uint64),
                ("d_lists", C.c_void_p), ("d_chunks", C.c_void_p), ("d_small", C.c_void_p)]


class lc_setop_plan(C.Structure):
    _fields_ = [("n_pairs", C.c_uint32), ("op", C.c_int32), ("short_keys", C.c_uint64),
                ("long_keys", C.c_uint64), ("units", C.c_uint64), ("scratch_bytes", C.c_uint64),
                ("out_keys", C.c_uint64)]


class lc_view(C.Structure):
    _fields_ = [("h", lc_header), ("d_blob", C.c_void_p), ("d_first", C.c_void_p),
                ("d_acc", C.c_void_p), ("span_lo", C.c_uint64), ("span_hi", C.c_uint64), ("sec_base", C.c_uint64 * 4)]


_p, _u64, _u32, _i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32
_sig = {
    "lc_encode": ([_p, _u64, _u32, _u32, C.POINTER(_p), C.POINTER(_u64)], _i32),
    "lc_encode_ex": ([_p, _u64, _u32, _u32, _u32, C.POINTER(_p), C.POINTER(_u64)], _i32),
    "lc_free": ([_p], None),
    "lc_validate": ([_p, _u64], _i32),
    "lc_view_init": ([C.POINTER(lc_view), _p, _p, _u64], _i32),
    "lc_decode": ([C.POINTER(lc_view), _p, _p], _i32),
    "lc_decode_span": ([C.POINTER(lc_view), _u64, _u64, _p, _p], _i32),
    "lc_access": ([C.POINTER(lc_view), _p, _u64, _p, _p, _p], _i32),
    "lc_range_decode": ([C.POINTER(lc_view), _p, _u64, _u32, _p, _p, _p], _i32),
    "lc_quantile": ([C.POINTER(lc_view), _p, _u64, _u64, _i32, _p, _p, _p], _i32),
    "lc_next_geq": ([C.POINTER(lc_view), _p, _u64, _p, _p, _p], _i32),
    "lc_intersect_scratch_bytes": ([C.POINTER(lc_view)], _u64),
    "lc_intersect": ([C.POINTER(lc_view), C.POINTER(lc_view), _p, _u64, _p, _p, _p], _i32),
    "lc_union_scratch_bytes": ([C.POINTER(lc_view), C.POINTER(lc_view)], _u64),
    "lc_search_index_bytes": ([C.POINTER(lc_view)], _u64),
    "lc_search_index_build": ([C.POINTER(lc_view), _p, _p], _i32),
    "lc_access_layout_bytes": ([C.POINTER(lc_view)], _u64),
    "lc_access_layout_build": ([C.POINTER(lc_view), _p, _p], _i32),
    "lc_union": ([C.POINTER(lc_view), C.POINTER(lc_view), _p, _u64, _p, _p, _p], _i32),
    "lc_decode_host": ([_p, _u64, _p, _p, _p, _p], _i32),
    "lc_shard_bytes": ([_p, _u64, _u64, _u64, C.POINTER(_u64)], _i32),
    "lc_shard_upload": ([_p, _u64, _u64, _u64, _p, _u64, C.POINTER(lc_view), _p], _i32),
    "lc_batch_dir_bytes": ([_p, _u64, _p, _u32, C.POINTER(_u64)], _i32),
    "lc_batch_init": ([C.POINTER(lc_batch), _p, _u64, _p, _u32, _p, _p, _p, _u64, _p], _i32),
    "lc_decode_batch": ([C.POINTER(lc_batch), _p, _p, _p], _i32),
    "lc_setop_batch_plan": ([C.POINTER(lc_batch), _p, _p, _u32, _i32, C.POINTER(lc_setop_plan)],
                            _i32),
    "lc_intersect_batch": ([C.POINTER(lc_batch), C.POINTER(lc_setop_plan), _p, _p, _u64, _p, _p,
                            _p, _p], _i32),
    "lc_union_batch": ([C.POINTER(lc_batch), C.POINTER(lc_setop_plan), _p, _p, _u64, _p, _p, _p,
                        _p], _i32),
    "lc_status_str": ([_i32], C.c_char_p),
    "lc_launch_count": ([], _u64),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTS = tuple(_sig)


class LcError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {_lib.lc_status_str(code).decode()} ({code})")
        self.code = code


def _check(code: int, what: str) -> None:
    if code != LC_OK:
        raise LcError(code, what)


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class _On:
    """Stream discipline of one call that launches on `stream` (a torch.cuda.Stream, a raw
    cudaStream_t handle, or None = the current stream).

    When `stream` is a torch stream other than the current one: it first waits for the current
    stream (inputs staged there are ready), every device tensor the call reads or writes is
    marked used on it (record_stream: the caching allocator will not hand that memory to other
    work while the kernels may still run), and tensors allocated inside the `with` block
    (outputs, scratch) are allocated on it, so dropping a scratch right after the call is
    safe.  A raw handle leaves this to the caller."""

    def __init__(self, stream, *tensors):
        import torch
        cur = torch.cuda.current_stream()
        self.handle = _stream(stream)
        self.ts = stream if isinstance(stream, torch.cuda.Stream) else None
        self.other = self.ts is not None and self.ts != cur
        self._ctx = None
        if self.other:
            self.ts.wait_stream(cur)
            self.use(*tensors)

    def use(self, *tensors):
        if self.other:
            for t in tensors:
                if t is not None and getattr(t, "is_cuda", False):
                    t.record_stream(self.ts)
        return tensors[0] if len(tensors) == 1 else tensors

    def __enter__(self):
        if self.other:
            import torch
            self._ctx = torch.cuda.stream(self.ts)
            self._ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self._ctx is not None:
            self._ctx.__exit__(*exc)
        return False


def launch_count() -> int:
    """Kernels launched by liblc.so so far (process-wide counter)."""
    return int(_lib.lc_launch_count())


# ---------------------------------------------------------------------------- host side
def encode(keys: np.ndarray, eps: int, key_bits: int | None = None, free: bool = False,
           min_segments: bool = False) -> bytes:
    """lc_encode / lc_encode_ex: host blob of sorted keys (uint32 or uint64 numpy array);
    anchored greedy (FORMAT F1-F6) or, with free=True, the free-intercept encoder (F7);
    min_segments=True: the fewest segments of that form (LC_FLAG_MIN_SEGMENTS)."""
    k = np.asarray(keys)
    if key_bits is None:
        key_bits = 32 if k.dtype == np.uint32 else 64
    if key_bits == 32 and k.dtype != np.uint32:
        if k.size and int(k.max()) > 0xFFFFFFFF:
            raise LcError(LC_ERR_TOO_LARGE, "lc_encode")
    k = np.ascontiguousarray(k, dtype=np.uint32 if key_bits == 32 else np.uint64)
    out, nb = C.c_void_p(), C.c_uint64()
    _check(_lib.lc_encode_ex(k.ctypes.data if k.size else None, k.size, key_bits, eps,
                             (LC_FLAG_FREE_INTERCEPT if free else 0)
                             | (LC_FLAG_MIN_SEGMENTS if min_segments else 0),
                             C.byref(out), C.byref(nb)),
           "lc_encode_ex")
    try:
        return C.string_at(out.value, nb.value)
    finally:
        _lib.lc_free(out)


def _host_ptr(blob) -> tuple[int, int, object]:
    if isinstance(blob, (bytes, bytearray)):
        buf = (C.c_char * len(blob)).from_buffer_copy(blob) if isinstance(blob, bytes) else \
            (C.c_char * len(blob)).from_buffer(blob)
        return C.addressof(buf), len(blob), buf
    if isinstance(blob, np.ndarray):
        return blob.ctypes.data, blob.nbytes, blob
    # torch CPU tensor
    return blob.data_ptr(), blob.numel() * blob.element_size(), blob


def validate(blob) -> int:
    """lc_validate: 0 (LC_OK) or a negative status."""
    p, n, _keep = _host_ptr(blob)
    return int(_lib.lc_validate(p, n))


def header(blob) -> lc_header:
    p, n, _keep = _host_ptr(blob)
    if n < 128:
        raise LcError(LC_ERR_FORMAT, "header")
    return lc_header.from_buffer_copy(C.string_at(p, 128))


# -------------------------------------------------------------------------- device side
class View:
    """A blob resident on the GPU: lc_view (host header + device pointer) plus the tensor."""

    def __init__(self, blob, device="cuda", d_blob=None, blob_bytes=None):
        """`blob`: the host blob (or at least its 128-byte header when `d_blob`, a device copy
        of `blob_bytes` bytes, is given)."""
        import torch
        raw = bytes(blob) if not isinstance(blob, (bytes, np.ndarray)) else blob
        host = np.frombuffer(raw, np.uint8) if isinstance(raw, bytes) else raw.view(np.uint8)
        if d_blob is None:
            d_blob = torch.from_numpy(host.copy()).to(device)
        self.d_blob = d_blob
        self.d_first = None
        self.d_acc = None
        self.v = lc_view()
        nbytes = host.nbytes if blob_bytes is None else int(blob_bytes)
        _check(_lib.lc_view_init(C.byref(self.v), host.ctypes.data, d_blob.data_ptr(), nbytes),
               "lc_view_init")

    @classmethod
    def shard(cls, h_blob, i0: int, i1: int, device="cuda", stream=None, out=None):
        """lc_shard_upload: a shard view holding only the slices of keys [i0, i1) of the host
        blob h_blob (bytes, numpy uint8 or a pinned CPU uint8 tensor); decode() then writes
        keys [i0, i1).  The host buffer is kept referenced by the view until it is dropped."""
        import torch
        hp, hn, keep = _host_ptr(h_blob)
        nb = C.c_uint64()
        _check(_lib.lc_shard_bytes(hp, hn, i0, i1, C.byref(nb)), "lc_shard_bytes")
        self = cls.__new__(cls)
        self.d_first = None
        self.d_acc = None
        self._host_keep = keep
        with _On(stream) as on:
            if out is None:
                out = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=device)
            on.use(out)
            if out.numel() < nb.value:
                raise ValueError("shard buffer too small")
            self.d_blob = out
            self.v = lc_view()
            _check(_lib.lc_shard_upload(hp, hn, i0, i1, out.data_ptr(), out.numel(),
                                        C.byref(self.v), on.handle), "lc_shard_upload")
        return self

    @staticmethod
    def shard_bytes(h_blob, i0: int, i1: int) -> int:
        hp, hn, _keep = _host_ptr(h_blob)
        nb = C.c_uint64()
        _check(_lib.lc_shard_bytes(hp, hn, i0, i1, C.byref(nb)), "lc_shard_bytes")
        return int(nb.value)

    @property
    def n(self) -> int:
        return int(self.v.h.n)

    @property
    def span(self) -> tuple[int, int]:
        """Keys this view decodes: (0, n), or a shard's (span_lo, span_hi)."""
        if self.v.span_hi:
            return int(self.v.span_lo), int(self.v.span_hi)
        return 0, self.n

    @property
    def key_bits(self) -> int:
        return int(self.v.h.key_bits)

    @property
    def torch_dtype(self):
        import torch
        return torch.int64 if self.key_bits == 64 else torch.int32

    def search_index_bytes(self) -> int:
        return int(_lib.lc_search_index_bytes(C.byref(self.v)))

    def build_search_index(self, stream=None, out=None):
        """lc_search_index_build: allocate the successor-search index (the segments' first keys
        plus every 16th of them, about 8.5 bytes per segment) on the blob's device, build it on
        `stream` and attach it to this view (next_geq / intersect / union then use it)."""
        import torch
        nbytes = self.search_index_bytes()
        with _On(stream, self.d_blob) as on:
            if out is None:
                out = torch.empty(max(nbytes // 8, 1), dtype=torch.int64, device=self.d_blob.device)
            if out.numel() * out.element_size() < nbytes:
                raise ValueError("search index buffer too small")
            self.d_first = on.use(out)
            _check(_lib.lc_search_index_build(C.byref(self.v), self.d_first.data_ptr(), on.handle),
                   "lc_search_index_build")
        return self.d_first

    def access_layout_bytes(self) -> int:
        return int(_lib.lc_access_layout_bytes(C.byref(self.v)))

    def build_access_layout(self, stream=None, out=None):
        """lc_access_layout_build: allocate the access layout (segment-major records: params
        followed by the segment's residual units, 16 (2 L + N b / 128) bytes) on the blob's
        device, build it on `stream` and attach it (access / exact quantiles then use it)."""
        import torch
        nbytes = self.access_layout_bytes()
        with _On(stream, self.d_blob) as on:
            if out is None:
                out = torch.empty(max(nbytes // 8, 2), dtype=torch.int64,
                                  device=self.d_blob.device)
            if out.numel() * out.element_size() < nbytes:
                raise ValueError("access layout buffer too small")
            self.d_acc = on.use(out)
            _check(_lib.lc_access_layout_build(C.byref(self.v), self.d_acc.data_ptr(),
                                               on.handle), "lc_access_layout_build")
        return self.d_acc

    def tensors(self):
        """Device tensors the view's calls read (for stream bookkeeping)."""
        return (self.d_blob, self.d_first, getattr(self, "d_acc", None))

    def out_tensor(self, count: int):
        import torch
        return torch.empty(count, dtype=self.torch_dtype, device=self.d_blob.device)


def _ptr(t) -> int | None:
    return t.data_ptr() if t is not None and t.numel() else None


def decode(view: View, out=None, stream=None):
    """lc_decode: all N keys (or a shard view's span) into a device tensor (int64/int32 storage
    of u64/u32 keys)."""
    with _On(stream, *view.tensors()) as on:
        if out is None:
            lo, hi = view.span
            out = view.out_tensor(hi - lo)
        on.use(out)
        _check(_lib.lc_decode(C.byref(view.v), out.data_ptr(), on.handle), "lc_decode")
    return out


def decode_span(view: View, i0: int, i1: int, out=None, stream=None):
    with _On(stream, *view.tensors()) as on:
        if out is None:
            out = view.out_tensor(max(i1 - i0, 0))
        on.use(out)
        _check(_lib.lc_decode_span(C.byref(view.v), i0, i1, _ptr(out), on.handle),
               "lc_decode_span")
    return out


def access(view: View, idx, out=None, err=None, stream=None):
    """lc_access: Dec(K^c)[idx] for a device int64 tensor of indices."""
    q = idx.numel()
    with _On(stream, *view.tensors(), idx, err) as on:
        if out is None:
            out = view.out_tensor(q)
        on.use(out)
        _check(_lib.lc_access(C.byref(view.v), _ptr(idx), q, _ptr(out) if q else None,
                              err.data_ptr() if err is not None else None, on.handle),
               "lc_access")
    return out


def range_decode(view: View, starts, length: int, out=None, err=None, stream=None):
    """lc_range_decode: out[r, k] = K[starts[r] + k]."""
    q = starts.numel()
    with _On(stream, *view.tensors(), starts, err) as on:
        if out is None:
            out = view.out_tensor(q * length)
        on.use(out)
        _check(_lib.lc_range_decode(C.byref(view.v), _ptr(starts), q, length,
                                    _ptr(out) if q else None,
                                    err.data_ptr() if err is not None else None, on.handle),
               "lc_range_decode")
    return out.view(q, length)


def quantile(view: View, ranks, q: int, exact: bool = True, out=None, err=None, stream=None):
    """lc_quantile: the ranks[t]-th q-quantiles (exact, or the segments-only approximation)."""
    m = ranks.numel()
    with _On(stream, *view.tensors(), ranks, err) as on:
        if out is None:
            out = view.out_tensor(m)
        on.use(out)
        _check(_lib.lc_quantile(C.byref(view.v), _ptr(ranks), m, q, 1 if exact else 0,
                                _ptr(out) if m else None,
                                err.data_ptr() if err is not None else None, on.handle),
               "lc_quantile")
    return out


def next_geq(view: View, x, out_idx=None, out_key=None, stream=None):
    """lc_next_geq: (first index with K[i] >= x_t, that key) for a device int64 tensor of probes."""
    import torch
    m = x.numel()
    with _On(stream, *view.tensors(), x) as on:
        if out_idx is None:
            out_idx = torch.empty(m, dtype=torch.int64, device=x.device)
        if out_key is None:
            out_key = view.out_tensor(m)
        on.use(out_idx, out_key)
        _check(_lib.lc_next_geq(C.byref(view.v), _ptr(x), m, _ptr(out_idx) if m else None,
                                _ptr(out_key) if m else None, on.handle), "lc_next_geq")
    return out_idx, out_key


def ctypes_ref(view: View):
    return C.byref(view.v)


def union_scratch_bytes(a: View, b: View) -> int:
    return int(_lib.lc_union_scratch_bytes(C.byref(a.v), C.byref(b.v)))


def intersect_scratch_bytes(a: View) -> int:
    return int(_lib.lc_intersect_scratch_bytes(C.byref(a.v)))


def intersect(a: View, b: View, scratch=None, out=None, count=None, stream=None):
    """lc_intersect: keys in both lists (pass the shorter list as `a`).  Returns (out, count)
    where out[:count] holds the intersection (count is a device tensor)."""
    import torch
    dev = a.d_blob.device
    need = int(_lib.lc_intersect_scratch_bytes(C.byref(a.v)))
    with _On(stream, *a.tensors(), *b.tensors()) as on:
        if scratch is None:
            scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        if out is None:
            out = a.out_tensor(a.n)
        if count is None:
            count = torch.zeros(1, dtype=torch.int64, device=dev)
        on.use(scratch, out, count)
        _check(_lib.lc_intersect(C.byref(a.v), C.byref(b.v), scratch.data_ptr(),
                                 scratch.numel() * scratch.element_size(), out.data_ptr(),
                                 count.data_ptr(), on.handle), "lc_intersect")
    return out, count


def union(a: View, b: View, scratch=None, out=None, count=None, stream=None):
    """lc_union: sorted keys in either list.  Returns (out, count): out[:count] is the union."""
    import torch
    dev = a.d_blob.device
    need = int(_lib.lc_union_scratch_bytes(C.byref(a.v), C.byref(b.v)))
    with _On(stream, *a.tensors(), *b.tensors()) as on:
        if scratch is None:
            scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        if out is None:
            out = a.out_tensor(a.n + b.n)
        if count is None:
            count = torch.zeros(1, dtype=torch.int64, device=dev)
        on.use(scratch, out, count)
        _check(_lib.lc_union(C.byref(a.v), C.byref(b.v), scratch.data_ptr(),
                             scratch.numel() * scratch.element_size(), out.data_ptr(),
                             count.data_ptr(), on.handle), "lc_union")
    return out, count


def decode_host(h_blob, d_blob, d_out, h_out, stream=None) -> None:
    """lc_decode_host: pinned host blob -> device -> decode -> pinned host keys (async)."""
    with _On(stream, d_blob, d_out) as on:
        _check(_lib.lc_decode_host(h_blob.data_ptr(), h_blob.numel(), d_blob.data_ptr(),
                                   d_out.data_ptr(), h_out.data_ptr(), on.handle),
               "lc_decode_host")


# ------------------------------------------------------------------------------- batches
class Batch:
    """Many lists in one device buffer (lc_batch_init): their blobs packed at 256-byte aligned
    offsets, uploaded once, plus the device directory of the batch (list and chunk records)."""

    def __init__(self, blobs, device="cuda", stream=None, out_off=None):
        import torch
        offs, pos = [], 0
        for bl in blobs:
            offs.append(pos)
            pos += (len(bl) + 255) // 256 * 256
        host = np.zeros(max(pos, 256), np.uint8)
        for o, bl in zip(offs, blobs):
            host[o:o + len(bl)] = np.frombuffer(bl, np.uint8)
        self.blob_off = np.asarray(offs, np.uint64)
        self.m = len(blobs)
        self.host = host
        nb = C.c_uint64()
        _check(_lib.lc_batch_dir_bytes(host.ctypes.data, host.nbytes, self.blob_off.ctypes.data,
                                       self.m, C.byref(nb)), "lc_batch_dir_bytes")
        oo = None if out_off is None else np.ascontiguousarray(out_off, np.uint64)
        with _On(stream) as on:
            self.d_blobs = on.use(torch.from_numpy(host).to(device, non_blocking=False))
            self.d_dir = on.use(torch.empty(max(nb.value, 16), dtype=torch.uint8, device=device))
            self.b = lc_batch()
            _check(_lib.lc_batch_init(C.byref(self.b), host.ctypes.data, host.nbytes,
                                      self.blob_off.ctypes.data, self.m, self.d_blobs.data_ptr(),
                                      None if oo is None else oo.ctypes.data,
                                      self.d_dir.data_ptr(), self.d_dir.numel(), on.handle),
                   "lc_batch_init")
            self.d_work = on.use(torch.zeros(4, dtype=torch.int32, device=device))
        headers = [lc_header.from_buffer_copy(bl[:128]) for bl in blobs]
        self.n = np.array([h.n for h in headers], np.int64)
        self.out_off = (np.concatenate([[0], np.cumsum(self.n)[:-1]]).astype(np.int64)
                        if oo is None else oo.astype(np.int64))

    @property
    def n_total(self) -> int:
        return int(self.b.n_total)

    @property
    def torch_dtype(self):
        import torch
        return torch.int64 if self.b.key_bits == 64 else torch.int32

    def tensors(self):
        return (self.d_blobs, self.d_dir, self.d_work)


def decode_batch(batch: Batch, out=None, stream=None):
    """lc_decode_batch: every list of the batch in one launch; list k's keys at
    out[batch.out_off[k] : batch.out_off[k] + batch.n[k]]."""
    import torch
    with _On(stream, *batch.tensors()) as on:
        if out is None:
            size = int((batch.out_off + batch.n).max()) if batch.m else 0
            out = torch.empty(max(size, 1), dtype=batch.torch_dtype, device=batch.d_blobs.device)
        on.use(out)
        _check(_lib.lc_decode_batch(C.byref(batch.b), out.data_ptr(), batch.d_work.data_ptr(),
                                    on.handle), "lc_decode_batch")
    return out


LC_SETOP_AND, LC_SETOP_OR = 0, 1


class SetopBuffers:
    """One batched AND / OR query batch: its host plan (lc_setop_batch_plan), the pairs on the
    device, and the scratch / output / result arrays (reusable for repeated runs)."""

    def __init__(self, batch: Batch, pairs, op: int):
        import torch
        self.pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        self.h_n = np.ascontiguousarray(batch.n, np.uint64)
        self.op = op
        self.plan = lc_setop_plan()
        _check(_lib.lc_setop_batch_plan(C.byref(batch.b), self.h_n.ctypes.data,
                                        self.pairs.ctypes.data, len(self.pairs), op,
                                        C.byref(self.plan)), "lc_setop_batch_plan")
        dev = batch.d_blobs.device
        self.d_pairs = torch.from_numpy(self.pairs.view(np.int32).reshape(-1).copy()).to(dev)
        self.scratch = torch.empty(max(self.plan.scratch_bytes, 256), dtype=torch.uint8, device=dev)
        self.out = torch.empty(max(self.plan.out_keys, 1), dtype=batch.torch_dtype, device=dev)
        self.out_off = torch.zeros(len(self.pairs) + 1, dtype=torch.int64, device=dev)
        self.counts = torch.zeros(max(len(self.pairs), 1), dtype=torch.int64, device=dev)

    def tensors(self):
        return (self.d_pairs, self.scratch, self.out, self.out_off, self.counts)


def _setop_batch(fn, what, batch: Batch, pairs, op, bufs, stream):
    if bufs is None:
        bufs = SetopBuffers(batch, pairs, op)
    with _On(stream, *batch.tensors(), *bufs.tensors()) as on:
        _check(fn(C.byref(batch.b), C.byref(bufs.plan), bufs.d_pairs.data_ptr(),
                  bufs.scratch.data_ptr(), bufs.scratch.numel(), bufs.out.data_ptr(),
                  bufs.out_off.data_ptr(), bufs.counts.data_ptr(), on.handle), what)
    return bufs


def intersect_batch(batch: Batch, pairs=None, bufs=None, stream=None) -> SetopBuffers:
    """lc_intersect_batch: AND of every pair (a, b) of list indices; pair p's keys at
    bufs.out[bufs.out_off[p] : bufs.out_off[p] + bufs.counts[p]] (packed)."""
    return _setop_batch(_lib.lc_intersect_batch, "lc_intersect_batch", batch, pairs,
                        LC_SETOP_AND, bufs, stream)


def union_batch(batch: Batch, pairs=None, bufs=None, stream=None) -> SetopBuffers:
    """lc_union_batch: OR of every pair; pair p's keys at
    bufs.out[bufs.out_off[p] : bufs.out_off[p] + bufs.counts[p]]."""
    return _setop_batch(_lib.lc_union_batch, "lc_union_batch", batch, pairs, LC_SETOP_OR, bufs,
                        stream)
