"""Adversarial input rows for K1's quantisation (R11: v_hat = bf16_RNE(fp32_RN(v / sqrt(sum v^2)_64))),
built in exact integer / rational arithmetic so the expected values are decided by the definition
alone (tests/test_gpu_k1_exact.py compares the GPU's bytes with oracle.quantize on them).

Every row's sum of squares is an exact integer (times 4^s), so the fp64 norm is the same whatever the
summation order; the rows then put v_i / |v| where a shortcut would go wrong:

* near-midpoint rows: v_0 / |v| within a few fp64 ulp of an fp32 rounding midpoint whose two fp32
  neighbours straddle a bf16 tie (low 16 bits 0x7FFF / 0x8000), so one fp64 ulp decides the bf16
  value.  (An EXACT fp32 midpoint cannot occur in the normal range: v has at most 24 significant bits
  and |v| = 2^e * r, so v / |v| has at most 24 -- or, for odd r > 1, infinitely many.)
* subnormal rows: |v| = 3 * 2^40 exactly and v_j / |v| = (2 c_j + 1) 2^-150 EXACTLY on an fp32
  subnormal rounding midpoint next to a bf16 tie;
* the same rows scaled by 2^100 and 2^-100 (~1e30, ~1e-30).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def _fp32_bits_to_value(bits: int) -> Fraction:
    e = (bits >> 23) & 0xFF
    m = bits & 0x7FFFFF
    assert 0 < e < 255
    return Fraction((1 << 23) | m, 1 << 23) * Fraction(2) ** (e - 127)


def _squares(S: int):
    """Greedy decomposition of a non-negative integer into squares of integers < 2^24."""
    out = []
    while S > 0:
        a = min(math.isqrt(S), (1 << 24) - 1)
        out.append(a)
        S -= a * a
    return out


def near_midpoint_rows(n: int, d: int = 768, seed: int = 0):
    """2n rows [2n, d] float64 (exactly fp32-representable integers): n where the fp64 product
    v_0 * RN(1/|v|) and the fp64 quotient RN(v_0 / |v|) round to different fp32 values (a kernel
    rounding the product would be wrong) and n where they agree; plus that flag per row."""
    rng = np.random.default_rng(seed)
    rows, straddle = [], []
    n_yes = n_no = 0
    while n_yes < n or n_no < n:
        e = int(rng.integers(-5, -1))                    # y in [1/32, 1/2)
        top = int(rng.integers(0, 128))                  # the 7 bf16 mantissa bits
        ybits = ((e + 127) << 23) | (top << 16) | 0x8000   # a bf16 tie in fp32
        y = _fp32_bits_to_value(ybits)
        m = y - Fraction(2) ** (e - 24)                  # fp32 midpoint between y - ulp and y
        x = int(rng.integers(1 << 21, 1 << 22))
        S_f = round(Fraction(x * x) * (1 - m * m) / (m * m))
        ss = x * x + S_f
        if ss >= 1 << 53:
            continue
        norm = math.sqrt(ss)                             # IEEE fp64 sqrt of an exact integer
        q_div = np.float64(x) / np.float64(norm)
        q_mul = np.float64(x) * (np.float64(1.0) / np.float64(norm))
        fill = _squares(S_f)
        if len(fill) + 1 > d or any(a >= 1 << 24 for a in fill):
            continue
        st = bool(np.float32(q_div) != np.float32(q_mul))
        if (st and n_yes >= n) or (not st and n_no >= n):
            continue
        n_yes += st
        n_no += not st
        r = np.zeros(d)
        r[0] = x
        r[1:1 + len(fill)] = fill
        rows.append(r)
        straddle.append(st)
    return np.stack(rows), np.array(straddle)


def subnormal_rows(n: int, d: int = 768, seed: int = 1, per_row: int = 64):
    """Rows [n, d]: (2^40, 2^41, 2^41) fix |v| = 3 * 2^40; per_row further components
    v_j = 3 (2 c_j + 1) 2^-110 make v_j / |v| = (2 c_j + 1) 2^-150, an fp32 subnormal midpoint,
    with c_j = h 2^16 + 0x7FFF, h odd: its fp32 neighbours c_j and c_j + 1 (a bf16 tie, which rounds
    to the even h + 1) give different bf16 values, so a mis-rounded fp32 step shows in the bytes."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, d))
    for i in range(n):
        out[i, :3] = [2.0 ** 40, 2.0 ** 41, 2.0 ** 41]
        h = 2 * rng.integers(0, 1 << 4, per_row) + 1      # odd: c and c + 1 round to different bf16
        c = (h << 16) | 0x7FFF
        sign = rng.choice([-1.0, 1.0], per_row)
        vals = sign * 3.0 * (2 * c + 1).astype(np.float64) * 2.0 ** -110
        out[i, 3:3 + per_row] = vals
    return out


def scaled(rows: np.ndarray, s: int) -> np.ndarray:
    """rows * 2^s (exact in fp32 for the scales used: no overflow / underflow of any component)."""
    out = rows * 2.0 ** s
    assert np.all(np.float32(out) == out), "scale not exact in fp32"
    return out
