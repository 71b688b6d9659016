"""ctypes binding of oracle/lc_oracle.c (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lc_oracle.c")
_LIB = os.path.join(_HERE, "liblc_oracle.so")

U64_MAX = (1 << 64) - 1
GMAX = (1 << 63) - 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, OpenMP for the all-cores baseline timing)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-std=gnu11", "-Wall", "-shared",
                               "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        p = C.c_void_p
        u64, i64, u32, i32 = C.c_uint64, C.c_int64, C.c_uint32, C.c_int32
        L.oracle_width.argtypes = [u64]
        L.oracle_width.restype = u32
        L.oracle_segment_ex.argtypes = [p, u64, u64, u32, u64, p, C.c_int, p, p, p]
        L.oracle_segment_ex.restype = i64
        L.oracle_encode_ex.argtypes = [p, u64, u32, u64, p, C.c_int, C.POINTER(p),
                                       C.POINTER(u64)]
        L.oracle_encode_ex.restype = i32
        L.oracle_segment_free.argtypes = [p, u64, u64, u32, u64, p, p, p]
        L.oracle_segment_free.restype = i64
        L.oracle_encode_free.argtypes = [p, u64, u32, u64, C.POINTER(p), C.POINTER(u64)]
        L.oracle_encode_free.restype = i32
        L.oracle_segment_min.argtypes = [p, u64, u64, C.c_int, u32, u64, p, p, p]
        L.oracle_segment_min.restype = i64
        L.oracle_encode_min.argtypes = [p, u64, u32, u64, i32, C.POINTER(p), C.POINTER(u64)]
        L.oracle_encode_min.restype = i32
        L.oracle_free.argtypes = [p]
        L.oracle_free.restype = None
        L.oracle_decode.argtypes = [p, u64, p]
        L.oracle_decode.restype = i32
        L.oracle_decode_span.argtypes = [p, u64, u64, u64, p]
        L.oracle_decode_span.restype = i32
        L.oracle_decode_mt.argtypes = [p, u64, p, C.POINTER(i32)]
        L.oracle_decode_mt.restype = i32
        L.oracle_access.argtypes = [p, u64, p, u64, p, C.POINTER(u32)]
        L.oracle_access.restype = i32
        L.oracle_predict.argtypes = [p, u64, p, u64, p, C.POINTER(u32)]
        L.oracle_predict.restype = i32
        L.oracle_range.argtypes = [p, u64, p, u64, u32, p, C.POINTER(u32)]
        L.oracle_range.restype = i32
        L.oracle_validate.argtypes = [p, u64]
        L.oracle_validate.restype = i32
        L.oracle_header.argtypes = [p, u64, p]
        L.oracle_header.restype = i32
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def width(eps: int) -> int:
    return int(lib().oracle_width(eps))


def segment(keys, eps: int, F: int = 32, gmax: int = GMAX, force_break=None, slope_mode: int = 0):
    """Greedy anchored cone segmentation (FORMAT F4). Returns (starts, base, slope) u64 arrays."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    n = k.size
    st = np.empty(max(n, 1), np.uint64)
    ba = np.empty(max(n, 1), np.uint64)
    sl = np.empty(max(n, 1), np.uint64)
    fb = None if force_break is None else np.ascontiguousarray(force_break, dtype=np.uint8)
    L = lib().oracle_segment_ex(_ptr(k), n, eps, F, gmax, None if fb is None else _ptr(fb),
                                slope_mode, _ptr(st), _ptr(ba), _ptr(sl))
    if L < 0:
        raise OracleError(L, "segment")
    return st[:L].copy(), ba[:L].copy(), sl[:L].copy()


def segment_free(keys, eps: int, F: int = 32, gmax: int = GMAX):
    """Free-intercept greedy segmentation (FORMAT F7). Returns (starts, base, slope) u64
    arrays, base = beta - eps."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    n = k.size
    st = np.empty(max(n, 1), np.uint64)
    ba = np.empty(max(n, 1), np.uint64)
    sl = np.empty(max(n, 1), np.uint64)
    L = lib().oracle_segment_free(_ptr(k), n, eps, F, gmax, _ptr(st), _ptr(ba), _ptr(sl))
    if L < 0:
        raise OracleError(L, "segment_free")
    return st[:L].copy(), ba[:L].copy(), sl[:L].copy()


def segment_min(keys, eps: int, free: bool = False, F: int = 32, gmax: int = GMAX):
    """Fewest segments (oracle_segment_min: DP over the greedy ends emax(s), F4 or F7 fits).
    Returns (starts, base, slope) u64 arrays."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    n = k.size
    st = np.empty(max(n, 1), np.uint64)
    ba = np.empty(max(n, 1), np.uint64)
    sl = np.empty(max(n, 1), np.uint64)
    L = lib().oracle_segment_min(_ptr(k), n, eps, 1 if free else 0, F, gmax, _ptr(st), _ptr(ba),
                                 _ptr(sl))
    if L < 0:
        raise OracleError(L, "segment_min")
    return st[:L].copy(), ba[:L].copy(), sl[:L].copy()


def encode(keys, eps: int, key_bits: int | None = None, force_break=None,
           slope_mode: int = 0, free: bool = False, min_segments: bool = False) -> bytes:
    """LCG1 blob of `keys`: anchored (FORMAT F1-F6) or, with free=True, free-intercept (F7)."""
    arr = np.asarray(keys)
    if key_bits is None:
        key_bits = 32 if arr.dtype == np.uint32 else 64
    k = np.ascontiguousarray(arr, dtype=np.uint64)
    fb = None if force_break is None else np.ascontiguousarray(force_break, dtype=np.uint8)
    out = C.c_void_p()
    nb = C.c_uint64()
    if min_segments:
        if fb is not None or slope_mode:
            raise ValueError("force_break / slope_mode apply to the greedy anchored encoder only")
        st = lib().oracle_encode_min(_ptr(k) if k.size else None, k.size, key_bits, eps,
                                     1 if free else 0, C.byref(out), C.byref(nb))
    elif free:
        if fb is not None or slope_mode:
            raise ValueError("force_break / slope_mode apply to the anchored encoder only")
        st = lib().oracle_encode_free(_ptr(k) if k.size else None, k.size, key_bits, eps,
                                      C.byref(out), C.byref(nb))
    else:
        st = lib().oracle_encode_ex(_ptr(k) if k.size else None, k.size, key_bits, eps,
                                    None if fb is None else _ptr(fb), slope_mode,
                                    C.byref(out), C.byref(nb))
    if st != 0:
        raise OracleError(st, "encode")
    try:
        return C.string_at(out.value, nb.value)
    finally:
        lib().oracle_free(out)


@dataclass
class Header:
    key_bits: int
    b: int
    eps: int
    hint_log2: int
    n: int
    L: int
    n_hint: int
    W: int
    o_starts: int
    o_params: int
    o_hint: int
    o_words: int
    total: int
    flags: int


def header(blob: bytes) -> Header:
    v = np.zeros(14, np.uint64)
    st = lib().oracle_header(blob, len(blob), _ptr(v))
    if st != 0:
        raise OracleError(st, "header")
    return Header(*[int(x) for x in v])


def _dtype(h: Header):
    return np.uint32 if h.key_bits == 32 else np.uint64


def decode(blob: bytes) -> np.ndarray:
    h = header(blob)
    out = np.empty(h.n, _dtype(h))
    st = lib().oracle_decode(blob, len(blob), _ptr(out))
    if st != 0:
        raise OracleError(st, "decode")
    return out


def decode_span(blob: bytes, i0: int, i1: int) -> np.ndarray:
    h = header(blob)
    out = np.empty(max(i1 - i0, 0), _dtype(h))
    st = lib().oracle_decode_span(blob, len(blob), i0, i1, _ptr(out) if out.size else None)
    if st != 0:
        raise OracleError(st, "decode_span")
    return out


def decode_mt(blob: bytes, out: np.ndarray | None = None):
    """All-cores decode; returns (keys, threads used)."""
    h = header(blob)
    if out is None:
        out = np.empty(h.n, _dtype(h))
    nt = C.c_int32(0)
    st = lib().oracle_decode_mt(blob, len(blob), _ptr(out), C.byref(nt))
    if st != 0:
        raise OracleError(st, "decode_mt")
    return out, int(nt.value)


def access(blob: bytes, idx) -> tuple[np.ndarray, int]:
    h = header(blob)
    ix = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(ix.size, _dtype(h))
    err = C.c_uint32(0)
    st = lib().oracle_access(blob, len(blob), _ptr(ix) if ix.size else None, ix.size,
                             _ptr(out) if out.size else None, C.byref(err))
    if st != 0:
        raise OracleError(st, "access")
    return out, int(err.value)


def predict(blob: bytes, idx) -> tuple[np.ndarray, int]:
    """Segments-only prediction floor(f(i)) for each index (approximate quantiles)."""
    h = header(blob)
    ix = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(ix.size, _dtype(h))
    err = C.c_uint32(0)
    st = lib().oracle_predict(blob, len(blob), _ptr(ix) if ix.size else None, ix.size,
                              _ptr(out) if out.size else None, C.byref(err))
    if st != 0:
        raise OracleError(st, "predict")
    return out, int(err.value)


def quantile_index(n: int, k: int, q: int) -> int:
    """Index of the k-th q-quantile, min(floor(N k / q), N - 1)."""
    return min((n * k) // q, n - 1)


def range_decode(blob: bytes, starts, length: int) -> tuple[np.ndarray, int]:
    h = header(blob)
    s = np.ascontiguousarray(starts, dtype=np.uint64)
    out = np.empty(s.size * length, _dtype(h))
    err = C.c_uint32(0)
    st = lib().oracle_range(blob, len(blob), _ptr(s) if s.size else None, s.size, length,
                            _ptr(out) if out.size else None, C.byref(err))
    if st != 0:
        raise OracleError(st, "range")
    return out.reshape(s.size, length), int(err.value)


def validate(blob: bytes) -> int:
    """0 if the blob is a valid LCG1 blob, else a negative status."""
    return int(lib().oracle_validate(blob, len(blob)))
