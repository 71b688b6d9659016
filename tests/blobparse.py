"""Test-side reader of an LCG1 blob (FORMAT F1/F2), written from FORMAT.md with `struct`.

Independent of both the oracle's C reader and the product's header code: tests use it to
recompute invariants (exact-rational residual bound, ratio from byte counts) from raw bytes.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

HEADER_FMT = "<4sHBBII9QI36s"  # FORMAT F1, 128 bytes (flags at offset 88)
assert struct.calcsize(HEADER_FMT) == 128


@dataclass
class Blob:
    magic: bytes
    version: int
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
    starts: np.ndarray
    base: np.ndarray
    slope: np.ndarray
    hint: np.ndarray
    words: np.ndarray
    flags: int = 0

    @property
    def bias(self) -> int:
        """Decode bias c of FORMAT F3: eps (anchored) or 0 (free intercept, F7)."""
        return 0 if self.flags & 1 else self.eps

    @property
    def beta(self) -> list[int]:
        """Segment intercepts beta_j = floor(f(s_j)) as Python ints (F7 stores beta - eps)."""
        return [int(x) + self.eps - self.bias for x in self.base]


def parse(blob: bytes) -> Blob:
    (magic, version, key_bits, b, eps, hint_log2, n, L, n_hint, W, o_s, o_p, o_h, o_w, total,
     flags, _res) = struct.unpack_from(HEADER_FMT, blob, 0)
    starts = np.frombuffer(blob, np.uint32, L + 1, o_s)
    params = np.frombuffer(blob, np.uint64, 2 * L, o_p).reshape(L, 2)
    hint = np.frombuffer(blob, np.uint32, n_hint, o_h)
    words = np.frombuffer(blob, np.uint32, W, o_w)
    return Blob(magic, version, key_bits, b, eps, hint_log2, n, L, n_hint, W, o_s, o_p, o_h,
                o_w, total, starts, params[:, 0], params[:, 1], hint, words, flags)


def fields(bl: Blob) -> list[int]:
    """Residual fields u_i read bit by bit from the LSB-first stream (FORMAT F3)."""
    bits = np.unpackbits(bl.words.view(np.uint8), bitorder="little")
    out = []
    for i in range(bl.n):
        u = 0
        for t in range(bl.b):
            u |= int(bits[i * bl.b + t]) << t
        out.append(u)
    return out


def align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


def expected_size(n: int, L: int, b: int) -> int:
    """Blob bytes from the section sizes alone (FORMAT F1/F2; P7)."""
    H = (n + 1023) // 1024
    W = ((n * b + 31) // 32 + 1 + 3) // 4 * 4
    off = 256                      # 128-byte header, padded to the first 256-byte boundary
    off = align(off + 4 * (L + 1))  # starts u32[L+1]
    off = align(off + 16 * L)       # params {u64 base, i64 slope}[L]
    off = align(off + 4 * (H + 1))  # hint u32[H+1]
    return off + 4 * W              # words u32[W]
