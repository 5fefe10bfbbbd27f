"""Pins for O1..O4 (similarity, quantisation, top-k, optimal-K, H_K).

What pins them: SPEC worked examples (tests/golden/spec_examples.json), an independent
bf16 rounding (ml_dtypes) against the oracle's bit trick, the closed-form bf16 error
bound, brute-force sorting with Python's sorted() on tiny inputs, and invariants.
"""
import json
import math
import os

import ml_dtypes
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import route as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
GRID6 = [0, 5, 10, 15, 20, 25]
BANDS6 = [0.65, 0.72, 0.79, 0.86, 0.93]


def _setup(**kw):
    base = dict(grid=GRID6, thresholds=BANDS6, F=[1 / 6] * 6, instance_level=list(range(6)))
    base.update(kw)
    return O.Setup(**base)


def test_spec_nearest_examples():
    rng = np.random.default_rng(0)
    d = 16
    C = rng.standard_normal((10, d)).astype(np.float32)
    # the store contains the query itself
    r = O.route(C[3:4] * 3.0, C, _setup(topk=2))
    assert r.topk_id[0, 0] == 3 and abs(r.topk_score[0, 0] - 1.0) < 1e-12
    # S:161 / S:171: empty store -> cold -> K = 0
    r = O.route(C[:2], np.zeros((0, d), np.float32), _setup(topk=2))
    assert list(r.K) == [0, 0] and np.all(r.topk_id == -1) and np.all(r.flags & O.FLAG_COLD)
    # {e1, e2}, q = normalize(e1+e2): sqrt(2)/2 with either; tie -> lower gid (R10)
    e = np.eye(d, dtype=np.float32)
    q = (e[0] + e[1])[None, :]
    r = O.route(q, e[:2], _setup(topk=2))
    assert list(r.topk_id[0]) == [0, 1]
    assert abs(r.topk_score[0, 0] - math.sqrt(2) / 2) < 1e-15
    assert r.topk_score[0, 0] == r.topk_score[0, 1]


def test_spec_select_optimal_k():
    for ex in SPEC["select_optimal_k"]:
        lv = O.optimal_k_level(np.array([ex["s1"]]), BANDS6, np.array([True]))
        assert GRID6[lv[0]] == ex["K"], ex["cite"]
    assert O.optimal_k_level(np.array([0.99]), BANDS6, np.array([False]))[0] == 0   # cold


@settings(max_examples=100, deadline=None)
@given(st.lists(st.floats(-1, 1), min_size=2, max_size=40))
def test_optimal_k_monotone(s):
    s = np.sort(np.array(s))
    lv = O.optimal_k_level(s, BANDS6, np.ones(len(s), bool))
    assert np.all(np.diff(lv) >= 0)


def test_bf16_rounding_two_implementations():
    rng = np.random.default_rng(1)
    y = np.concatenate([rng.standard_normal(100_000).astype(np.float32),
                        np.array([1.0, -1.0, 0.0, 1.00390625, 1.005859375, 3.0e-39], np.float32)])
    mine = O.bf16_rne_bits(y)
    lib = y.astype(ml_dtypes.bfloat16).view(np.uint16)
    assert np.array_equal(mine, lib)


def test_quantise_error_bound_and_invalid():
    """|s_hat - s_A| <= (2u + u^2) |q||c| with u = 2^-8 (bf16) plus the fp32 step."""
    rng = np.random.default_rng(2)
    P = (rng.standard_normal((50, 768)) * 3).astype(np.float32)
    C = rng.standard_normal((300, 768)).astype(np.float32)
    Pq, pv = O.quantize(P)
    Cq, cv = O.quantize(C)
    assert pv.all() and cv.all()
    u = 2.0 ** -8 + 2.0 ** -24
    err = np.abs(O.similarity_B(Pq, Cq) - O.similarity_A(P, C))
    assert err.max() <= 2 * u + u * u
    # quantised rows are unit up to the bf16 rounding
    assert np.allclose(np.linalg.norm(Pq, axis=1), 1.0, atol=768 * 2 ** -8)
    bad = P.copy()
    bad[0] = 0.0
    bad[1, 5] = np.nan
    bad[2, 7] = np.inf
    q, v = O.quantize(bad)
    assert list(v[:4]) == [False, False, False, True] and np.all(q[:3] == 0)


def test_similarity_closed_forms():
    e = np.eye(4, dtype=np.float32)
    S = O.similarity_A(np.stack([e[0], -2 * e[0]]), np.stack([e[0], e[1]]))
    assert S.tolist() == [[1.0, 0.0], [-1.0, 0.0]]


def _brute_topk(row, gids, k):
    order = sorted(range(len(row)), key=lambda g: (-row[g], gids[g]))[:k]
    ids = [int(gids[g]) for g in order] + [-1] * (k - len(order))
    sc = [float(row[g]) for g in order] + [float("-inf")] * (k - len(order))
    return ids, sc


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 30), st.integers(1, 6), st.integers(0, 2**31 - 1))
def test_topk_matches_bruteforce_with_ties(m, k, seed):
    rng = np.random.default_rng(seed)
    s = np.round(rng.standard_normal((3, m)), 1)         # many exact ties
    gids = np.arange(m) * 3 + 1
    a_i, a_s = O.topk_sorted(s, gids, k)
    b_i, b_s = O.topk_prefiltered(s, gids, k)
    for p in range(3):
        ids, sc = _brute_topk(s[p], gids, k)
        assert list(a_i[p]) == ids and list(b_i[p]) == ids
        assert list(a_s[p]) == sc


@settings(max_examples=40, deadline=None)
@given(st.integers(2, 40), st.integers(1, 8), st.integers(1, 39), st.integers(0, 2**31 - 1))
def test_merge_of_parts_equals_whole(m, k, cut, seed):
    cut = min(cut, m - 1)
    rng = np.random.default_rng(seed)
    s = np.round(rng.standard_normal((4, m)), 1)
    g = np.arange(m)
    whole = O.topk_sorted(s, g, k)
    a = O.topk_sorted(s[:, :cut], g[:cut], k)
    b = O.topk_sorted(s[:, cut:], g[cut:], k)
    mi, ms = O.merge_topk(*a, *b, k)
    assert np.array_equal(mi, whole[0]) and np.array_equal(ms, whole[1])


def test_histogram_counts():
    lv = np.array([0, 2, 2, 5, 0, 2])
    assert O.histogram(lv, 6).tolist() == [2, 0, 3, 0, 0, 1]


def test_k1_adversarial_rows_are_what_they_claim():
    """The adversarial K1 inputs (tests/k1_adversarial.py) pinned by exact rational arithmetic: integer
    sums of squares (order-free norms), the straddle flag really separates the fp64 product from the
    quotient under fp32 rounding, and the subnormal quotients sit EXACTLY on fp32 midpoints whose two
    neighbours round to different bf16 values."""
    import math
    from fractions import Fraction

    from oracle import route as O
    from tests.k1_adversarial import near_midpoint_rows, subnormal_rows

    mid, straddle = near_midpoint_rows(16)
    for r, st in zip(mid, straddle):
        ss = sum(int(v) ** 2 for v in r)
        assert ss == int(np.sum(r * r)) and ss < 2 ** 53
        norm = math.sqrt(ss)
        assert (np.float32(r[0] / norm) != np.float32(r[0] * (1.0 / norm))) == st
    sub = subnormal_rows(2, per_row=8)
    for r in sub:
        norm = Fraction(3) * 2 ** 40
        assert sum(Fraction(float(v)) ** 2 for v in r[:3]) == norm ** 2
        for v in r[3:11]:
            q = abs(Fraction(float(v))) / norm
            units = q / Fraction(1, 2 ** 149)                    # fp32 subnormal spacing
            assert units.denominator == 2 and (units.numerator // 2) & 0xFFFF == 0x7FFF
        q, _ = O.quantize(r[None, :].astype(np.float32))
        # fp32 ties to even (c + 1 = h 2^16 + 0x8000), then that bf16 tie rounds to even: h + 1 units
        b = (q[0, 3:11].astype(np.float32).view(np.uint32) >> 16) & 0x7FFF
        h = (np.abs(r[3:11]) / 3 * 2.0 ** 110 - 1) / 2 / 2 ** 16
        assert np.array_equal(b, np.floor(h).astype(np.uint32) + 1)
