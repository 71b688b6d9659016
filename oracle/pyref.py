"""Python big-int transliteration of FORMAT F3/F4 (TEST INFRASTRUCTURE ONLY, tiny inputs).

A second, independent reading of the greedy anchored cone (F4) and the decode rule (F3),
written with unbounded Python ints so no 64/128-bit reasoning is involved. Used to
cross-check the C oracle on N <= 1e4; it is not itself a pin (the pins are in
tests/test_oracle_pins.py).
"""
from __future__ import annotations


def width(eps: int) -> int:
    """ceil(log2(2 eps + 1))."""
    return (2 * eps).bit_length()  # smallest b with 2^b >= 2 eps + 1


def segment(K, eps: int, F: int = 32, gmax: int = (1 << 63) - 1):
    """F4 greedy: list of (s, base, slope)."""
    K = [int(x) for x in K]
    n, out, s = len(K), [], 0
    while s < n:
        lo, hi, e = 0, gmax, s + 1
        while e < n:
            d, D = e - s, K[e] - K[s]
            lo2 = max(lo, -((-(D - eps) << F) // d) if D > eps else 0)
            hi2 = min(hi, (((D + eps + 1) << F) - 1) // d, gmax // d)
            if lo2 > hi2:
                break
            lo, hi, e = lo2, hi2, e + 1
        out.append((s, K[s], 0 if e - s == 1 else lo + (hi - lo) // 2))
        s = e
    return out


def decode_segments(segs, residuals, n: int, eps: int, key_bits: int):
    """F3 given decoded segments and residual fields u_i (no bit packing involved)."""
    keys, j = [], 0
    for i in range(n):
        while j + 1 < len(segs) and segs[j + 1][0] <= i:
            j += 1
        s, base, slope = segs[j]
        keys.append((base + ((slope * (i - s)) >> 32) + residuals[i] - eps) % (1 << key_bits))
    return keys


def residuals(K, segs, eps: int):
    """u_i = K[i] - floor(f(i)) + eps (F4 emit step)."""
    out, j = [], 0
    for i, k in enumerate(K):
        while j + 1 < len(segs) and segs[j + 1][0] <= i:
            j += 1
        s, base, slope = segs[j]
        out.append(int(k) - (base + ((slope * (i - s)) >> 32)) + eps)
    return out


def pack(us, b: int) -> list[int]:
    """LSB-first bit stream in little-endian u32 words (FORMAT F2/F3, L8), unpadded."""
    acc = 0
    for i, u in enumerate(us):
        acc |= u << (i * b)
    nw = (len(us) * b + 31) // 32
    return [(acc >> (32 * w)) & 0xFFFFFFFF for w in range(nw)]
