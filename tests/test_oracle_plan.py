"""Pins for O5..O7 (apportionment, Eq. 1 plan, D_Q).

What pins them: SPEC S:236-238 worked examples (golden), exhaustive enumeration on tiny
instances (exact rationals), scipy HiGHS LP, the cut-based closed form for linear D,
and the apportionment invariants (sum f = N, |f - N F| < 1, F = h/N recovers h).
"""
import json
import os

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import route as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
C_LIN = O.default_degradation()


def test_spec_plan_examples():
    for ex in SPEC["plan_routes"]:
        grid, h, f = ex["grid"], ex["h"], ex["f"]
        N = sum(h)
        xb, ties = O.plan_bruteforce(h, f, grid, C_LIN)
        xl = O.plan_lp(h, f, grid, C_LIN)
        assert np.array_equal(xb, xl), ex["cite"]
        assert ties == 1
        if "x" in ex:
            assert xb.tolist() == ex["x"], ex["cite"]
        assert abs(O.d_q(xb, grid, C_LIN, N) - ex["D_Q"]) <= 1e-12 + 1e-9 * ex["D_Q"], ex["cite"]


def test_degradation_linear_anchor():
    """R6 / S:50: a 25-step over-skip costs 0.15 (quality 0.85, P:129 'at just 85%')."""
    D = O.degradation_matrix([0, 25], C_LIN)
    assert D.tolist() == [[0.0, C_LIN[25]], [0.0, 0.0]] and abs(C_LIN[25] - 0.15) < 1e-15


@st.composite
def tiny_instance(draw):
    nK = draw(st.integers(2, 4))
    grid = sorted(draw(st.sets(st.integers(1, 49), min_size=nK - 1, max_size=nK - 1)))
    grid = [0] + grid
    N = draw(st.integers(0, 7))
    h = [0] * nK
    f = [0] * nK
    for _ in range(N):
        h[draw(st.integers(0, nK - 1))] += 1
        f[draw(st.integers(0, nK - 1))] += 1
    convex = draw(st.booleans())
    return grid, h, f, convex


def _convex_c(seed):
    rng = np.random.default_rng(seed)
    inc = np.sort(rng.uniform(0, 0.01, 50))
    c = np.concatenate([[0.0], np.cumsum(inc)[:49]])
    return c


@settings(max_examples=150, deadline=None)
@given(tiny_instance(), st.integers(0, 1000))
def test_lp_equals_bruteforce(inst, seed):
    grid, h, f, convex = inst
    c = _convex_c(seed) if convex else C_LIN
    xb, ties = O.plan_bruteforce(h, f, grid, c)
    assert ties == 1                       # R7: (D, sum dK^2) has a unique optimum
    xl = O.plan_lp(h, f, grid, c)
    assert np.array_equal(xb, xl)
    assert xb.sum(axis=1).tolist() == h and xb.sum(axis=0).tolist() == f


@settings(max_examples=100, deadline=None)
@given(st.integers(2, 10), st.integers(1, 5000), st.integers(0, 2**31 - 1))
def test_lp_dq_matches_linear_closed_form(nK, N, seed):
    rng = np.random.default_rng(seed)
    grid = [0] + sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
    h = np.bincount(rng.integers(0, nK, N), minlength=nK)
    f = np.bincount(rng.integers(0, nK, N), minlength=nK)
    x = O.plan_lp(h, f, grid, C_LIN)
    got = O.d_q(x, grid, C_LIN, N)
    want = O.dq_linear_closed_form(h, f, grid, 0.006, N)
    assert abs(got - want) <= 1e-12 + 1e-9 * want


def test_identity_when_h_equals_f():
    rng = np.random.default_rng(5)
    for _ in range(20):
        h = rng.integers(0, 50, 6)
        x = O.plan_lp(h, h, [0, 5, 10, 15, 20, 25], C_LIN)
        assert np.array_equal(x, np.diag(h))


def test_all_upgrade_costs_zero():
    """S:238 / acceptance 10: when every move can be an upgrade (K' <= K), D_Q = 0."""
    h = [0, 0, 10]
    for f in ([10, 0, 0], [3, 3, 4], [0, 5, 5]):
        x = O.plan_lp(h, f, [0, 10, 25], C_LIN)
        assert O.d_q(x, [0, 10, 25], C_LIN, 10) == 0.0


def test_apportion_examples():
    assert O.apportion([0.2, 0.3, 0.5], 10).tolist() == [2, 3, 5]
    assert O.apportion([0.5, 0.5], 1).tolist() == [1, 0]           # tie -> lower index
    assert O.apportion([1 / 3] * 3, 3).tolist() == [1, 1, 1]
    assert O.apportion([0.25, 0.0, 0.75], 3).tolist() == [1, 0, 2]  # q = (.75, 0, 2.25)
    assert O.apportion([0.6, 0.4], 0).tolist() == [0, 0]


@settings(max_examples=300, deadline=None)
@given(st.integers(1, 200_000), st.lists(st.integers(0, 1000), min_size=2, max_size=16))
def test_apportion_invariants(N, wts):
    if sum(wts) == 0:
        wts[0] = 1
    F = [w / sum(wts) for w in wts]
    f = O.apportion(F, N)
    assert int(f.sum()) == N
    assert np.all(np.abs(f - N * np.array(F)) < 1)
    assert np.all(f[np.array(F) == 0] == 0)


@settings(max_examples=300, deadline=None)
@given(st.lists(st.integers(0, 5000), min_size=2, max_size=16))
def test_apportion_recovers_h(h):
    N = sum(h)
    if N == 0:
        return
    F = [v / N for v in h]
    assert O.apportion(F, N).tolist() == h
