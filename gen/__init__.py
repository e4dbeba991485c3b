"""Seeded synthetic-input generator shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only turns
(seed, stream, index) into pseudo-random 64-bit words with a counter-based
SplitMix64 mix and maps them into [0, p) or 16-bit limbs.  Tests (oracle
side) and bench.py / the GPU parity tests (CUDA side) draw their inputs from
here, so both see identical bytes; a rank of a multi-GPU run draws exactly its
own index range (no scatter).

Two bit-identical backends implement the same integer recipe:
  * numpy uint64 (host), and
  * torch int64 (any device; two's-complement wrap == uint64 wrap, logical
    shifts emulated with masks) -- used to materialise large inputs directly
    in HBM for the bench.  tests/test_gen.py checks the two agree.

Recipe:
  w_i   = mix64(key + (i + 1) * GAMMA),   key = seed ^ (stream * STREAM_MULT)
  p < 2^32 : r_i = floor(w_i * p / 2^64)           (multiply-high, uniform to 2^-32)
  2^32 <= p < 2^62: r_i = (w_i >> 1) mod p         (bias <= p / 2^63)
  p >= 2^62: r_i = w_i - p if w_i >= p else w_i    (bias <= (2^64 - p) / 2^64)
  limbs    : low 16 bits of w_i
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
STREAM_MULT = 0xD1B54A32D192ED03
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def config_seed(k: int) -> int:
    """Config k uses seed 0x14073383_0000000k; operands a/b = streams 1/2."""
    return (0x14073383 << 32) | k


def _key(seed: int, stream: int) -> int:
    return (seed ^ (stream * STREAM_MULT)) & _MASK64


# ------------------------------------------------------------------ numpy
def _mix64_np(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def words(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """count raw 64-bit words for indices [start, start + count)."""
    key = np.uint64(_key(seed, stream))
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
        return _mix64_np(key + idx * np.uint64(GAMMA))


def _map_np(w, p):
    if p < (1 << 32):
        P = np.uint64(p)
        with np.errstate(over="ignore"):
            hi = (w >> np.uint64(32)) * P
            lo = ((w & np.uint64(0xFFFFFFFF)) * P) >> np.uint64(32)
            return ((hi + lo) >> np.uint64(32)).astype(np.uint32)
    P = np.uint64(p)
    if p < (1 << 62):
        return ((w >> np.uint64(1)) % P).astype(np.uint64)
    with np.errstate(over="ignore"):
        return np.where(w >= P, w - P, w).astype(np.uint64)


def residues(seed: int, stream: int, count: int, p: int, start: int = 0,
             chunk: int = 1 << 24) -> np.ndarray:
    """count residues uniform in [0, p): uint32 if p < 2^32 else uint64."""
    out = np.empty(count, dtype=np.uint32 if p < (1 << 32) else np.uint64)
    for off in range(0, count, chunk):
        n = min(chunk, count - off)
        out[off:off + n] = _map_np(words(seed, stream, start + off, n), p)
    return out


def limbs16(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """count uniform 16-bit limbs (little-endian digits of a random integer)."""
    return (words(seed, stream, start, count) & np.uint64(0xFFFF)).astype(np.uint16)


# ------------------------------------------------------------------ torch
def _s64(v: int) -> int:
    v &= _MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _shr(z, k):
    """Logical right shift of an int64 tensor holding uint64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _mix64_t(z):
    z = (z ^ _shr(z, 30)) * _s64(_M1)
    z = (z ^ _shr(z, 27)) * _s64(_M2)
    return z ^ _shr(z, 31)


def words_torch(seed: int, stream: int, start: int, count: int, device):
    import torch
    idx = torch.arange(start + 1, start + 1 + count, dtype=torch.int64, device=device)
    return _mix64_t(_s64(_key(seed, stream)) + idx * _s64(GAMMA))


def residues_torch(seed: int, stream: int, count: int, p: int, device, start: int = 0,
                   chunk: int = 1 << 26):
    """Same values as residues(), materialised on `device` (uint32 for p < 2^32
    returned as torch.int32 bit patterns; uint64 as torch.int64 bit patterns)."""
    import torch
    small = p < (1 << 32)
    out = torch.empty(count, dtype=torch.int32 if small else torch.int64, device=device)
    for off in range(0, count, chunk):
        n = min(chunk, count - off)
        w = words_torch(seed, stream, start + off, n, device)
        if small:
            hi = _shr(w, 32) * p
            lo = _shr((w & 0xFFFFFFFF) * p, 32)
            r = _shr(hi + lo, 32)
            out[off:off + n] = (r - ((r >> 31) << 32)).to(torch.int32)   # to signed 32-bit pattern
        elif p < (1 << 62):
            out[off:off + n] = torch.remainder(_shr(w, 1), p)            # non-negative int64
        else:
            flip = -(1 << 63)
            ge = (w ^ flip) >= (_s64(p) ^ flip)                          # unsigned compare
            out[off:off + n] = torch.where(ge, w - _s64(p), w)
    return out


def limbs16_torch(seed: int, stream: int, count: int, device, start: int = 0):
    """Same values as limbs16(), as torch.int16 bit patterns on `device`."""
    import torch
    w = words_torch(seed, stream, start, count, device) & 0xFFFF
    return (w - ((w >> 15) << 16)).to(torch.int16)
