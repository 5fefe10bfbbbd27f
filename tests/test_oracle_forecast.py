"""Pins of oracle/forecast.py (R21-R24) against things other than itself:
SPEC worked examples, a linear-programming solver, closed-form counts, exact marginals, statistics."""
import math

import numpy as np
import pytest

from oracle import forecast as fc
from oracle import route

GRID6 = [0, 5, 10, 15, 20, 25]


# ---------------- R21 predictor: SPEC S:202-213, S:323-330 examples ----------------

def test_predict_hk_spec_examples():
    p = fc.Predictor(2, 1000)
    p.record([0] * 7)
    assert list(p.predict()) == [1.0, 0.0]                     # window all K=0 -> {0: 1.0}
    p = fc.Predictor(2, 1000)
    p.record([0, 0, 1, 1])
    assert list(p.predict()) == [0.5, 0.5]                     # [0,0,25,25] -> {0: .5, 25: .5}
    assert list(fc.Predictor(2, 10).predict()) == [0.5, 0.5]   # empty, grid {0,25} -> uniform


def test_record_optimal_k_spec_examples():
    p = fc.Predictor(2, 4)
    p.record([0, 0, 0])
    p.record([1])
    assert list(p.predict()) == [0.75, 0.25]                   # append 25 to zeros(3), W=4
    p.record([0] * 10)
    assert p.counts()[1] == 4                                  # full window stays W
    q = fc.Predictor(6, 1)
    q.record([3, 5, 2])
    assert list(q.predict()) == [0, 0, 1, 0, 0, 0]             # W=1 -> last observation


# ---------------- l2_hist_error: SPEC S:533-540 examples ----------------

def test_l2_hist_error_spec_examples():
    assert fc.l2_hist_error([0.3, 0.7], [0.3, 0.7]) == 0.0
    assert fc.l2_hist_error([1.0, 0.0], [0.0, 1.0]) == pytest.approx(math.sqrt(2), abs=1e-15)
    assert fc.l2_hist_error([0.6, 0.4], [0.5, 0.5]) == pytest.approx(math.sqrt(0.02), abs=1e-15)
    with pytest.raises(ValueError):
        fc.l2_hist_error([1.0], [0.5, 0.5])


# ---------------- R22 plan: SPEC S:236-238 in fractional form, LP, marginals ----------------

def test_plan_spec_examples_fractional():
    c = route.default_degradation()
    # H == F -> identity, D_Q = 0
    Hc = fc.cumulative_H([2, 1, 1], 4, 3)
    Fc = fc.cumulative_F([0.5, 0.25, 0.25])
    assert Hc == Fc
    x = fc.coupling(Hc, Fc)
    assert np.all(x == np.diag(np.diag(x)))
    assert fc.dq_plan(Hc, Fc, [0, 10, 25], c) == 0.0
    # {0,25}, H = (.5,.5), F = (.25,.75), D(25,0) = 0.15 -> D_Q = 0.0375 exactly
    Hc = fc.cumulative_H([1, 1], 2, 2)
    Fc = fc.cumulative_F([0.25, 0.75])
    assert fc.dq_plan(Hc, Fc, [0, 25], c) == pytest.approx(0.0375, abs=1e-15)
    rows = fc.plan_rows(Hc, Fc)
    assert list(rows[0]) == [0.5, 0.5] and list(rows[1]) == [0.0, 1.0]
    # {0,10,25}, H = (.2,.3,.5), F = (.5,.2,.3): only upgrades -> D_Q = 0
    Hc = fc.cumulative_H([2, 3, 5], 10, 3)
    Fc = fc.cumulative_F([0.5, 0.2, 0.3])
    assert fc.dq_plan(Hc, Fc, [0, 10, 25], c) == 0.0


def test_plan_equals_lp_optimum_on_fractions():
    """The fixed-point monotone coupling attains the Eq. 1 LP optimum on (H, F) (HiGHS)."""
    rng = np.random.default_rng(21)
    for trial in range(60):
        nK = int(rng.integers(2, 7))
        grid = sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
        grid = [0] + grid
        if trial % 2:
            c = route.default_degradation()
        else:   # a convex, non-linear table
            t = np.arange(route.T_TOTAL, dtype=np.float64)
            c = 0.002 * t + 0.0004 * t * t
        n = int(rng.integers(1, 2000))
        cnt = rng.multinomial(n, rng.dirichlet(np.ones(nK)))
        F = rng.dirichlet(np.ones(nK))
        Hc = fc.cumulative_H(cnt, n, nK)
        Fc = fc.cumulative_F(F)
        got = fc.dq_plan(Hc, Fc, grid, c)
        lp = route.dq_continuous(cnt / n, F, grid, c)
        assert got == pytest.approx(lp, abs=nK * nK * 2.0 ** -31 + 1e-12), (trial, got, lp)


def test_coupling_marginals_exact():
    rng = np.random.default_rng(22)
    for _ in range(200):
        nK = int(rng.integers(1, 11))
        n = int(rng.integers(0, 5000))
        cnt = rng.multinomial(n, np.ones(nK) / nK) if n else np.zeros(nK, np.int64)
        F = rng.dirichlet(np.ones(nK)) * (rng.random(nK) > 0.3)
        if F.sum() == 0:
            F[0] = 1.0
        F = F / F.sum()
        Hc = fc.cumulative_H(cnt, n, nK)
        Fc = fc.cumulative_F(F)
        x = fc.coupling(Hc, Fc)
        assert Hc[-1] == fc.ONE and Fc[-1] == fc.ONE
        assert list(x.sum(axis=1)) == [Hc[i + 1] - Hc[i] for i in range(nK)]
        assert list(x.sum(axis=0)) == [Fc[j + 1] - Fc[j] for j in range(nK)]
        for j in range(nK):                      # no mass where F has none
            if F[j] == 0:
                assert x[:, j].sum() == 0
        if n:                                    # fixed point within one unit of the exact masses
            for i in range(nK):
                assert abs((Hc[i + 1] - Hc[i]) - cnt[i] * fc.ONE / n) <= 1.0


# ---------------- R23 sampling ----------------

def test_words_per_level_matches_plan_rows():
    """The closed-form word counts reproduce P(K'_j|K_i) = x_ij / H_i to within 1 word."""
    rng = np.random.default_rng(23)
    for _ in range(100):
        nK = int(rng.integers(2, 8))
        n = int(rng.integers(1, 3000))
        cnt = rng.multinomial(n, rng.dirichlet(np.ones(nK)))
        Hc = fc.cumulative_H(cnt, n, nK)
        Fc = fc.cumulative_F(rng.dirichlet(np.ones(nK)))
        x = fc.coupling(Hc, Fc)
        for i in range(nK):
            w = Hc[i + 1] - Hc[i]
            cnts = fc.words_per_level(Hc, Fc, i)
            if w == 0:
                assert cnts.sum() == 0
                continue
            assert cnts.sum() == fc.ONE
            for j in range(nK):
                assert abs(int(cnts[j]) - int(x[i, j]) * fc.ONE / w) <= 1.0


def test_sampler_agrees_with_closed_form_on_reduced_words():
    """sample() puts word u in level j iff the closed-form interval says so: check u at the
    interval ends computed by the closed form (every boundary word and its neighbour)."""
    Hc = fc.cumulative_H([3, 5, 7, 1], 16, 4)
    Fc = fc.cumulative_F([0.1, 0.45, 0.05, 0.4])
    for i in range(4):
        w = Hc[i + 1] - Hc[i]
        cnts = fc.words_per_level(Hc, Fc, i)
        start = 0
        for j in range(4):
            if cnts[j] == 0:
                continue
            for u in (start, start + cnts[j] - 1):   # first and last word of level j
                pos = Hc[i] + ((u * w) >> 32)
                jj = 0
                while jj < 3 and Fc[jj + 1] <= pos:
                    jj += 1
                assert jj == j
            start += cnts[j]


def test_route_prompt_spec_examples():
    c = route.default_degradation()
    # row {25: 1.0} -> always 25: F puts all mass on K=25
    Hc = fc.cumulative_H([5, 5], 10, 2)
    Fc = fc.cumulative_F([0.0, 1.0])
    kp, _ = fc.sample(np.array([0, 1] * 500), Hc, Fc, seed=7, batch_seq=0)
    assert np.all(kp == 1)
    # row {0: .5, 25: .5}, 10k samples -> 5000 +- 150: H all at 25, F = (.5, .5)
    Hc = fc.cumulative_H([0, 1000], 1000, 2)
    Fc = fc.cumulative_F([0.5, 0.5])
    kp, unf = fc.sample(np.ones(10_000, np.int64), Hc, Fc, seed=0x5EED2502, batch_seq=3)
    assert abs(int(np.sum(kp == 0)) - 5000) <= 150 and not unf.any()
    # determinism: same seed and batch -> same output
    kp2, _ = fc.sample(np.ones(10_000, np.int64), Hc, Fc, seed=0x5EED2502, batch_seq=3)
    assert np.array_equal(kp, kp2)
    assert fc.dq_plan(Hc, Fc, [0, 25], c) == 0.0


def test_unforecast_class_goes_to_coupling_point():
    # forecast all K=0, a K=25 prompt arrives: width 0 -> pos = Hc = 2^32 - 1 (clamped) -> last level
    Hc = fc.cumulative_H([4, 0], 4, 2)
    Fc = fc.cumulative_F([0.3, 0.7])
    kp, unf = fc.sample(np.array([1, 1, 0]), Hc, Fc, seed=1, batch_seq=0)
    assert list(unf) == [True, True, False] and list(kp[:2]) == [1, 1]
    # F with no mass at the last level: never routed there
    Hc = fc.cumulative_H([4, 0, 0], 4, 3)
    Fc = fc.cumulative_F([0.5, 0.5, 0.0])
    kp, _ = fc.sample(np.array([2] * 50 + [0] * 50), Hc, Fc, seed=2, batch_seq=0)
    assert not np.any(kp == 2)


def test_sampling_frequencies_match_plan_rows():
    rng = np.random.default_rng(24)
    cnt = np.array([300, 100, 250, 50, 200, 100])
    Hc = fc.cumulative_H(cnt, 1000, 6)
    F = np.array([0.05, 0.05, 0.10, 0.10, 0.20, 0.50])
    Fc = fc.cumulative_F(F)
    rows = fc.plan_rows(Hc, Fc)
    levels = rng.integers(0, 6, 120_000)
    kp, _ = fc.sample(levels, Hc, Fc, seed=99, batch_seq=5)
    for i in range(6):
        m = levels == i
        n = int(m.sum())
        for j in range(6):
            p = rows[i][j]
            got = int(np.sum(kp[m] == j))
            assert abs(got - n * p) <= 5 * math.sqrt(n * p * (1 - p)) + 1, (i, j, got, n * p)


def test_stationary_stretch_l1_below_003():
    """SPEC invariant: over a 10k-prompt stationary stretch the realised K' marginal is within
    L1 0.03 of F; and the L2 forecast error is small once the W = 1000 window is full."""
    rng = np.random.default_rng(25)
    H = np.array([0.30, 0.10, 0.25, 0.05, 0.20, 0.10])
    F = [0.05, 0.05, 0.10, 0.10, 0.20, 0.50]
    s = route.Setup(grid=GRID6, thresholds=[0.65, 0.72, 0.79, 0.86, 0.93], F=F,
                    instance_level=[0, 1, 2, 3, 4, 5, 5, 5], bstar=4)
    fr = fc.ForecastRouter(6, 1000, replan_every=1)
    kps = []
    l2s = []
    for b in range(14):
        s.batch_seq = b
        level = rng.choice(6, size=1000, p=H)
        out = fr.batch(level, s, route)
        if b >= 4:
            kps.append(out["level_prime"])
            l2s.append(out["l2"])
    kp = np.concatenate(kps)
    realised = np.bincount(kp, minlength=6) / len(kp)
    assert np.sum(np.abs(realised - np.array(F))) < 0.03
    assert max(l2s) < 0.08 and np.mean(l2s) < 0.05


def test_forecast_router_replan_period_and_window():
    s = route.Setup(grid=[0, 10, 25], thresholds=[0.7, 0.9], F=[0.2, 0.3, 0.5], instance_level=[0, 1, 2, 2])
    fr = fc.ForecastRouter(3, 8, replan_every=3)
    outs = []
    for b in range(7):
        s.batch_seq = b
        outs.append(fr.batch(np.array([b % 3] * 5), s, route))
    assert [o["replanned"] for o in outs] == [True, False, False, True, False, False, True]
    assert outs[0]["plan_n"] == 0 and outs[0]["n_unforecast"] == 0   # empty window: uniform forecast
    assert outs[3]["plan_n"] == 8 and list(outs[3]["plan_counts"]) == [0, 3, 5]   # last 8 of 0x5,1x5,2x5
    s.F = [0.5, 0.3, 0.2]                           # F change forces a rebuild
    s.batch_seq = 7
    assert fr.batch(np.array([0] * 5), s, route)["replanned"]


def test_forecast_downstream_matches_exact_path_bookkeeping():
    """Route-and-batch after the i.i.d. K' is the same O9/O10 as the exact path: buckets are a
    permutation, per-instance FIFO, K' counts = column sums of the realised moves."""
    rng = np.random.default_rng(26)
    s = route.Setup(grid=GRID6, thresholds=[0.65, 0.72, 0.79, 0.86, 0.93], F=[0.1, 0.1, 0.15, 0.15, 0.2, 0.3],
                    instance_level=[0, 0, 1, 2, 3, 4, 5, 5], bstar=4)
    fr = fc.ForecastRouter(6, 1000)
    for b in range(3):
        s.batch_seq = b
        level = rng.integers(0, 6, 777)
        out = fr.batch(level, s, route)
        assert sorted(out["bucket_prompts"].tolist()) == list(range(777))
        assert list(out["f"]) == [int(np.sum(out["level_prime"] == j)) for j in range(6)]
        assert out["x"].sum() == 777 and list(out["x"].sum(axis=1)) == list(out["h"])
        assert out["D_Q"] == pytest.approx(fc.dq_realized(level, out["level_prime"], s.grid, s.c))
