"""Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11).

Test infrastructure only (see oracle/__init__.py).

The paper fixes no random generator; its Router only "selects the final approximate
model at K' based on the Route-Plan" and uniform routing
"distribut[es] prompts randomly to workers".  DESIGN.md reading R18 fixes
the randomness as a counter-based function of (seed, batch_seq, prompt, stream) so
it is reproducible and independent of the number of router GPUs.

Two implementations live here on purpose: ``philox4x32_10`` is the textbook scalar
round function on Python integers, ``philox4x32_10_np`` the same rounds vectorised
on numpy uint64.  Tests pin both to the published Random123 known-answer vectors
and to each other.

Counter layout (R18):
    key = (seed & 0xffffffff, seed >> 32)
    ctr = (p, 0, batch_seq & 0xffffffff, (stream << 24) | ((batch_seq >> 32) & 0xffffff))
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

STREAM_REDIRECT = 1   # O8: per-prompt redirection key
STREAM_UNIFORM = 2    # O9: uniform-mode worker pick


def philox4x32_10(ctr, key):
    """Scalar Philox4x32 with 10 rounds.  ctr: 4 uint32, key: 2 uint32 -> 4 uint32."""
    c0, c1, c2, c3 = (int(v) & MASK32 for v in ctr)
    k0, k1 = (int(v) & MASK32 for v in key)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def _mulhilo_np(a: int, b: np.ndarray):
    prod = np.uint64(a) * b.astype(np.uint64)
    return (prod >> np.uint64(32)), (prod & np.uint64(MASK32))


def philox4x32_10_np(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10 over arrays of counters (same key for all)."""
    c0 = np.asarray(c0, dtype=np.uint64) & np.uint64(MASK32)
    c1 = np.asarray(c1, dtype=np.uint64) & np.uint64(MASK32)
    c2 = np.asarray(c2, dtype=np.uint64) & np.uint64(MASK32)
    c3 = np.asarray(c3, dtype=np.uint64) & np.uint64(MASK32)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 &= MASK32
    k1 &= MASK32
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        hi0, lo0 = _mulhilo_np(PHILOX_M0, c0)
        hi1, lo1 = _mulhilo_np(PHILOX_M1, c2)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return c0, c1, c2, c3


def stream_words(n: int, seed: int, batch_seq: int, stream: int):
    """(w0, w1, w2, w3) of Philox at ctr = (p, 0, batch_lo, stream<<24 | batch_hi) for p < n."""
    p = np.arange(n, dtype=np.uint64)
    c2 = batch_seq & MASK32
    c3 = ((stream & 0xFF) << 24) | ((batch_seq >> 32) & 0xFFFFFF)
    return philox4x32_10_np(p, 0, c2, c3, seed & MASK32, (seed >> 32) & MASK32)


def redirect_keys(n: int, seed: int, batch_seq: int) -> np.ndarray:
    """kappa_p = ((w1 << 32) | w0) >> 4 for the redirection stream (60-bit keys, uint64)."""
    w0, w1, _, _ = stream_words(n, seed, batch_seq, STREAM_REDIRECT)
    return ((w1 << np.uint64(32)) | w0) >> np.uint64(4)


def uniform_words(n: int, seed: int, batch_seq: int) -> np.ndarray:
    """u_p = w0 of the uniform-routing stream (uint32 values in uint64)."""
    w0, _, _, _ = stream_words(n, seed, batch_seq, STREAM_UNIFORM)
    return w0
