"""Pins for the f4 controller oracle (oracle/controller.py, R33-R36).

What pins it (none retypes the enumerator's own scoring):
  * SPEC S:226-228 worked examples (tests/golden/spec_controller.json);
  * an exact-rational brute force (fractions.Fraction, no rounding anywhere) on random small
    instances: same assignment wherever the exact optimum is not within 2^-38 of the runner-up;
  * the HiGHS MILP (scipy.optimize.milp) of the same lexicographic problem -- the formulation class
    the paper uses (via Proteus) -- on random instances up to W = 64: same S* and q*;
  * the HiGHS LP of the Query Fraction Solver for a fixed assignment: the greedy fill's q is its
    optimum;
  * Sum n = W, F_K lambda <= n_K rate_K, sum F = S, F_route sums to 1.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import controller as C

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_controller.json")))
GRID6 = [0, 5, 10, 15, 20, 25]
LIN = [0.006 * t for t in range(50)]


def _service(grid, per_step_us=100_000, marginal=0.3, bstar=4, T=50):
    """SPEC S:75 service(K, b) = (T - K) per_step (1 + marginal (b - 1)), in integer us."""
    return [int(round((T - K) * per_step_us * (1 + marginal * (bstar - 1)))) for K in grid]


def _random_instance(rng, Wmax, nKmax):
    nK = int(rng.integers(2, nKmax + 1))
    grid = sorted(rng.choice(np.arange(1, 40), nK - 1, replace=False).tolist())
    grid = [0] + grid
    W = int(rng.integers(1, Wmax + 1))
    H = rng.dirichlet(np.ones(nK)).tolist()
    bstar = int(rng.integers(1, 5))
    svc = _service(grid, per_step_us=int(rng.integers(20_000, 200_000)), bstar=bstar)
    r = C.rates(svc, bstar)
    lam = float(rng.choice([0.0, rng.uniform(0.01, 1.3) * W * max(r)]))
    c = [0.0] + np.cumsum(rng.uniform(0, 0.02, 49)).tolist()
    return W, lam, H, svc, bstar, grid, c


def test_spec_low_load_all_k0():
    g = GOLD["low_load"]
    svc = _service(GRID6)
    res = C.solve(g["W"], g["lambda"], g["H"], svc, 4, GRID6, LIN)
    assert res["n"] == g["expect_n"] and res["F"][0] == 1.0 and sum(res["F"][1:]) == 0.0


def test_spec_peak_load_all_k25():
    g = GOLD["peak_load"]
    grid = [0, 25]
    svc = _service(grid)
    r = C.rates(svc, 4)
    for mult in (1.0, 1.5, 10.0):
        res = C.solve(g["W"], mult * g["W"] * r[1], g["H"], svc, 4, grid, LIN)
        assert res["n"] == g["expect_n"]


def test_spec_mixed_equals_exhaustive():
    g = GOLD["mixed"]
    grid = [0, 25]
    svc = _service(grid)
    r = C.rates(svc, 4)
    lam = 0.5 * (g["W"] * r[0] + g["W"] * r[1])
    res = C.solve(g["W"], lam, g["H"], svc, 4, grid, LIN)
    ex = C.solve_exact(g["W"], lam, g["H"], svc, 4, grid, LIN)
    assert res["n"] == ex["n"]
    assert 0 < res["n"][0] < g["W"]              # a genuinely mixed assignment
    assert res["S"] == 1.0


def _exact_margin(W, lam, H, svc, bstar, grid, c, n_best):
    """Gap between the exact optimum and the best assignment that differs from it in (S, q)."""
    r = [Fraction(bstar) * 10**6 / Fraction(int(s)) for s in svc]
    a = [Fraction(1) - sum((Fraction(H[i]) * Fraction(c[K - grid[i]]) for i in range(len(grid))
                            if grid[i] < K), Fraction(0)) for K in grid]
    order = sorted(range(len(grid)), key=lambda k: (-a[k], k))
    vals = []
    for n in C.compositions(W, len(grid)):
        if lam == 0:
            S, cap = Fraction(1), [None if n[k] else Fraction(0) for k in range(len(grid))]
        else:
            cap = [Fraction(n[k]) * r[k] / Fraction(lam) for k in range(len(grid))]
            S = min(Fraction(1), sum(cap, Fraction(0)))
        filled = q = Fraction(0)
        for k in order:
            t = S - filled if cap[k] is None else min(cap[k], S - filled)
            filled += t
            q += t * a[k]
        vals.append((S, q))
    vals = sorted(set(vals), reverse=True)
    if len(vals) < 2:
        return 1.0
    (S0, q0), (S1, q1) = vals[0], vals[1]
    return float(S0 - S1) if S0 != S1 else float(q0 - q1)


def test_float_enumeration_equals_exact_rationals():
    rng = np.random.default_rng(2502)
    checked = 0
    for _ in range(200):
        W, lam, H, svc, bstar, grid, c = _random_instance(rng, 8, 4)
        got = C.solve(W, lam, H, svc, bstar, grid, c)
        ex = C.solve_exact(W, lam, H, svc, bstar, grid, c)
        if got["n"] != ex["n"]:
            # only a near-tie below the 2^-40 comparison grid may differ (R35)
            assert _exact_margin(W, lam, H, svc, bstar, grid, c, ex["n"]) < 2.0 ** -38
            continue
        checked += 1
        assert abs(got["S"] - float(ex["S"])) < 1e-12 and abs(got["q"] - float(ex["q"])) < 1e-12
    assert checked >= 190


def test_vectorized_equals_loops():
    rng = np.random.default_rng(7)
    for _ in range(40):
        W, lam, H, svc, bstar, grid, c = _random_instance(rng, 12, 5)
        a = C.solve(W, lam, H, svc, bstar, grid, c)
        b = C.solve_vectorized(W, lam, H, svc, bstar, grid, c)
        assert a["n"] == b["n"] and a["S"] == b["S"] and a["q"] == b["q"] and a["F"] == b["F"]


def _milp(W, lam, H, svc, bstar, grid, c):
    """The lexicographic problem as two HiGHS MILPs: max S, then max q at S >= S* (R33-R35)."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    nK = len(grid)
    r = C.rates(svc, bstar)
    a = C.agnostic_quality(H, grid, c)
    # variables: n_0..n_{nK-1} (integer), F_0..F_{nK-1}
    A, lo, hi = [], [], []
    for k in range(nK):            # lambda F_k - r_k n_k <= 0
        row = np.zeros(2 * nK)
        row[k], row[nK + k] = -r[k], lam
        A.append(row); lo.append(-np.inf); hi.append(0.0)
    row = np.zeros(2 * nK); row[:nK] = 1
    A.append(row); lo.append(W); hi.append(W)
    row = np.zeros(2 * nK); row[nK:] = 1
    A.append(row); lo.append(0.0); hi.append(1.0)
    integ = np.r_[np.ones(nK), np.zeros(nK)]
    bounds = Bounds(np.zeros(2 * nK), np.r_[np.full(nK, W), np.ones(nK)])
    obj1 = np.r_[np.zeros(nK), -np.ones(nK)]
    r1 = milp(obj1, constraints=LinearConstraint(np.array(A), lo, hi), integrality=integ, bounds=bounds)
    S = -r1.fun
    A2, lo2, hi2 = A + [np.r_[np.zeros(nK), np.ones(nK)]], lo + [S - 1e-9], hi + [1.0]
    obj2 = np.r_[np.zeros(nK), -np.array(a)]
    r2 = milp(obj2, constraints=LinearConstraint(np.array(A2), lo2, hi2), integrality=integ, bounds=bounds)
    return S, -r2.fun


@pytest.mark.parametrize("seed", range(12))
def test_enumeration_matches_milp(seed):
    rng = np.random.default_rng(100 + seed)
    W, lam, H, svc, bstar, grid, c = _random_instance(rng, 24, 5)
    if seed < 2:       # the SPEC scale: W = 64, |grid| = 6
        W, grid = 64, GRID6
        H = rng.dirichlet(np.ones(6)).tolist()
        svc = _service(grid, bstar=bstar)
        lam = float(rng.uniform(0.3, 1.1) * W * max(C.rates(svc, bstar)))
    if lam == 0.0:
        lam = 1e-3
    got = C.solve_vectorized(W, lam, H, svc, bstar, grid, c)
    S, q = _milp(W, lam, H, svc, bstar, grid, c)
    assert abs(got["S"] - S) < 1e-7 and abs(got["q"] - q) < 1e-7, (got, S, q)


def test_greedy_fill_is_the_lp_optimum():
    from scipy.optimize import linprog
    rng = np.random.default_rng(3)
    for _ in range(100):
        W, lam, H, svc, bstar, grid, c = _random_instance(rng, 12, 6)
        if lam == 0.0:
            continue
        n = list(next(iter(C.compositions(W, len(grid)))))
        rng.shuffle(n)
        r = C.rates(svc, bstar)
        a = C.agnostic_quality(H, grid, c)
        S, q, F = C.evaluate(n, r, a, lam)
        cap = [n[k] * r[k] / lam for k in range(len(grid))]
        res = linprog(-np.array(a), A_eq=np.ones((1, len(grid))), b_eq=[S],
                      bounds=[(0, cap[k]) for k in range(len(grid))], method="highs")
        assert abs(-res.fun - q) < 1e-9


def test_invariants():
    rng = np.random.default_rng(11)
    for _ in range(60):
        W, lam, H, svc, bstar, grid, c = _random_instance(rng, 10, 5)
        res = C.solve(W, lam, H, svc, bstar, grid, c)
        r = C.rates(svc, bstar)
        assert sum(res["n"]) == W and len(res["instance_level"]) == W
        assert res["instance_level"] == sorted(res["instance_level"])
        assert abs(sum(res["F"]) - res["S"]) < 1e-12 and abs(sum(res["F_route"]) - 1.0) < 1e-12
        for k in range(len(grid)):
            assert res["F"][k] * lam <= res["n"][k] * r[k] * (1 + 1e-12) + 1e-15
            assert res["F"][k] == 0.0 or res["n"][k] > 0
