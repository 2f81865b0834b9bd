"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used for the random-Gaussian policy s ~ N(0, I) (App. C.3 "Randomized Actions",
P:2143-2146) under reading R16: entry j of the action of iteration i at step k is
    (w0, w1, w2, w3) = philox4x32_10(ctr = (j, i, k, 0), key = (seed_lo, seed_hi))
    u1 = ((w0 >> 8) + 1) * 2^-24,  u2 = (w1 >> 8) * 2^-24
    z  = sqrt(-2 ln u1) * cos(2 pi u2)                      (Box–Muller, fp64)
numpy's Philox is the 4x64 variant and is NOT used.  Pinned by the Random123
known-answer vectors in tests/golden/philox4x32_10_kat.txt.
"""
from __future__ import annotations

import math

import numpy as np

_M0 = 0xD2511F53
_M1 = 0xCD9E8D57
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """One block: ctr = 4 uint32, key = 2 uint32 -> 4 uint32 (pure-Python ints)."""
    c0, c1, c2, c3 = (int(c) & _MASK for c in ctr)
    k0, k1 = (int(k) & _MASK for k in key)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> 32, p0 & _MASK
        hi1, lo1 = p1 >> 32, p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & _MASK, lo1, (hi0 ^ c3 ^ k1) & _MASK, lo0
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return c0, c1, c2, c3


def philox4x32_10_vec(c0, c1, c2, c3, k0, k1):
    """Vectorised over numpy uint64 arrays holding uint32 values (same arithmetic)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & _MASK for c in (c0, c1, c2, c3))
    k0 = np.uint64(k0 & _MASK)
    k1 = np.uint64(k1 & _MASK)
    for _ in range(10):
        p0 = np.uint64(_M0) * c0
        p1 = np.uint64(_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(_MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(_MASK)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & np.uint64(_MASK), lo1, (hi0 ^ c3 ^ k1) & np.uint64(_MASK), lo0
        k0 = (k0 + np.uint64(_W0)) & np.uint64(_MASK)
        k1 = (k1 + np.uint64(_W1)) & np.uint64(_MASK)
    return c0, c1, c2, c3


def random_action(seed: int, k: int, i: int, n: int) -> np.ndarray:
    """Action of iteration i (1-based) at step k (1-based), length n (R16)."""
    j = np.arange(n, dtype=np.uint64)
    w0, w1, _, _ = philox4x32_10_vec(j, np.full(n, i, np.uint64), np.full(n, k, np.uint64),
                                     np.zeros(n, np.uint64), seed & _MASK, (seed >> 32) & _MASK)
    u1 = ((w0 >> np.uint64(8)).astype(np.float64) + 1.0) * 2.0 ** -24
    u2 = (w1 >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
