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


# ------------------------------------------------------------------------------------------------
# R37 (NEXT f4): the exact plan for an arbitrary, non-convex degradation table
# ------------------------------------------------------------------------------------------------
def _concave_c():
    """c(t) = min(1, 0.09 t): c(10) = 0.9, c(20) = 1.0 -- concave, non-decreasing, in [0, 1]."""
    return np.minimum(1.0, 0.09 * np.arange(50))


def test_r37_hand_example_where_nw_corner_is_suboptimal():
    """Eq. 1 with a concave D: two prompts at K = {0, 10}, targets at {10, 20}.  The NW-corner
    (monotone) coupling moves both by 10 steps, D = 0.9 + 0.9 = 1.8; sending the K = 0 prompt to 20 and
    keeping the other costs D = 1.0 -- the exact optimum (NW is suboptimal on arbitrary
    tables)."""
    grid, c = [0, 10, 20], _concave_c()
    assert not O.is_convex(c)
    h, f = [1, 1, 0], [0, 1, 1]
    want = [[0, 0, 1], [0, 1, 0], [0, 0, 0]]
    cI = O.degradation_int(c)
    xb, ties = O.plan_int_bruteforce(h, f, grid, cI)
    assert xb.tolist() == want and ties == 1
    assert O.plan_int_lp(h, f, grid, cI).tolist() == want
    assert O.plan_for(h, f, grid, c).tolist() == want
    assert abs(O.d_q(xb, grid, c, 2) - 0.5) < 1e-15                       # D_Q = 1.0 / N
    nw = O.plan_lp(h, f, grid, O.default_degradation())                     # the convex-table plan
    assert nw.tolist() == [[0, 1, 0], [0, 0, 1], [0, 0, 0]] and O.d_q(nw, grid, c, 2) > 0.89


def test_r37_degradation_int_is_round_half_even():
    c = np.zeros(50)
    c[1] = 0.5 * 2.0 ** -24          # exactly half a unit: ties to even -> 0
    c[2] = 1.5 * 2.0 ** -24          # -> 2
    c[3] = 2.5 * 2.0 ** -24          # -> 2
    c[4] = 0.3
    c[5:] = 1.0
    cI = O.degradation_int(c)
    assert cI[:4].tolist() == [0, 0, 2, 2] and cI[4] == round(0.3 * 2 ** 24) and cI[5] == 2 ** 24


def _r37_instances(rng, n, nK_max=4, N_max=8):
    """Random small instances: random grids and tables, plus arithmetic grids with step tables, where
    (D, Q) ties occur and the lexicographic rule decides."""
    for it in range(n):
        if it % 2:
            nK = 4
            grid = [0, 5, 10, 15] if it % 4 == 1 else [0, 10, 20, 30]
            steps = np.sort(rng.choice([0.0, 0.25, 0.5, 1.0], 3))
            c = np.zeros(50)
            c[1:] = steps[np.minimum(np.arange(1, 50) // 11, 2)]
        else:
            nK = int(rng.integers(2, nK_max + 1))
            grid = [0] + sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
            c = np.concatenate([[0.0], np.sort(rng.uniform(0, 1, 49))])
        N = int(rng.integers(1, N_max + 1))
        h = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        f = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        yield grid, c, h, f


def r37_tie_instances(n_ties: int, seed: int = 4):
    """Arithmetic grids with step tables, searched (seeded, bounded) until n_ties instances have
    several (D, Q)-optimal plans, where only the lexicographic row-major rule decides."""
    rng = np.random.default_rng(seed)
    found = []
    for it in range(50_000):
        grid = [0, 5, 10, 15] if it % 2 else [0, 10, 20, 30]
        steps = np.sort(rng.choice([0.0, 0.25, 0.5, 1.0], 3))
        c = np.zeros(50)
        c[1:] = steps[np.minimum(np.arange(1, 50) // 11, 2)]
        N = int(rng.integers(2, 11))
        h = rng.multinomial(N, rng.dirichlet(np.ones(4)))
        f = rng.multinomial(N, rng.dirichlet(np.ones(4)))
        if O.plan_int_bruteforce(h, f, grid, O.degradation_int(c))[1] > 1:
            found.append((grid, c, h, f))
            if len(found) == n_ties:
                return found
    raise AssertionError("no tie instances found")


def test_r37_lp_equals_bruteforce_with_ties():
    """Exhaustive search (the definition) = the phased LP on 300 random instances and on instances
    with several (D, Q)-optimal plans, decided by the lexicographic row-major rule on both sides."""
    rng = np.random.default_rng(37)
    for grid, c, h, f in list(_r37_instances(rng, 300)) + r37_tie_instances(6):
        cI = O.degradation_int(c)
        xb, nt = O.plan_int_bruteforce(h, f, grid, cI)
        xl = O.plan_int_lp(h, f, grid, cI)
        assert np.array_equal(xb, xl), (grid, h.tolist(), f.tolist())


def test_r37_agrees_with_r7_on_exactly_linear_tables():
    """Where both rules apply -- a linear table whose integer image is exactly linear (c = t / 64) --
    R37's plan is R7's unique optimum (the NW-corner plan; LP and brute force)."""
    rng = np.random.default_rng(7)
    c = np.arange(50) / 64.0
    cI = O.degradation_int(c)
    assert np.all(np.diff(cI, 2) == 0)
    for _ in range(60):
        nK = int(rng.integers(2, 7))
        grid = [0] + sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
        N = int(rng.integers(1, 40))
        h = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        f = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        assert np.array_equal(O.plan_int_lp(h, f, grid, cI), O.plan_lp(h, f, grid, c))


def test_r37_never_worse_than_nw_and_often_better():
    """SURVEY V2 in integer form: on arbitrary tables the exact plan's D is <= the NW-corner plan's,
    strictly lower on a good share of instances (what makes the solver worth having)."""
    rng = np.random.default_rng(2)
    better = 0
    for _ in range(100):
        nK = int(rng.integers(3, 9))
        grid = [0] + sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
        c = np.concatenate([[0.0], np.sort(rng.uniform(0, 1, 49))])
        cI = O.degradation_int(c)
        N = int(rng.integers(5, 200))
        h = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        f = rng.multinomial(N, rng.dirichlet(np.ones(nK)))
        x = O.plan_int_lp(h, f, grid, cI)
        hc, fc = np.concatenate([[0], np.cumsum(h)]), np.concatenate([[0], np.cumsum(f)])
        nw = np.array([[max(0, min(hc[i + 1], fc[j + 1]) - max(hc[i], fc[j])) for j in range(nK)]
                       for i in range(nK)])
        D = lambda y: sum(int(y[i, j]) * int(cI[grid[j] - grid[i]]) for i in range(nK) for j in range(nK)
                          if grid[j] > grid[i])
        assert D(x) <= D(nw)
        better += D(x) < D(nw)
    assert better >= 20


def test_dq_continuous_pins():
    """D_Q_LP (pas_plan_stats; the Eq. 1 optimum on unrounded masses): the S:237 fractional example
    {0, 25}, H = (.5, .5), F = (.25, .75) -> 0.0375; H = F -> 0; all mass upgraded (F below H) -> 0;
    and for linear D it equals the cut closed form divided by N on masses that are multiples of 1/N."""
    c = O.default_degradation()
    assert abs(O.dq_continuous([0.5, 0.5], [0.25, 0.75], [0, 25], c) - 0.0375) < 1e-12
    assert abs(O.dq_continuous([0.2, 0.3, 0.5], [0.2, 0.3, 0.5], [0, 10, 25], c)) < 1e-12
    assert abs(O.dq_continuous([0.0, 0.0, 1.0], [0.5, 0.5, 0.0], [0, 10, 25], c)) < 1e-12
    h, f, N = [3, 5, 2], [1, 2, 7], 10
    ref = O.dq_linear_closed_form(h, f, [0, 10, 25], 0.006, N)
    assert abs(O.dq_continuous([v / N for v in h], [v / N for v in f], [0, 10, 25], c) - ref) < 1e-12


def test_is_convex_pins():
    assert O.is_convex(O.default_degradation())                          # linear
    assert O.is_convex(np.concatenate([[0.0], np.cumsum(np.linspace(0.001, 0.02, 49))]))   # increasing steps
    assert not O.is_convex(np.minimum(1.0, 0.09 * np.arange(50)))       # concave cap
    c = np.zeros(50)
    c[1:] = 0.5                                                          # a jump: non-convex
    assert not O.is_convex(c)
