"""Pins for O8..O10 (redirection, route-and-batch, buckets) and the composite route().

What pins them: the worked example W1 (tests/golden/w1.json), exact per-(i,j) counts equal
to the plan x, 'no redirection when H = F', the multinomial bound of S:312, a chi-square
uniformity check of the rank sampler, FIFO and size rules of S:320-334.
"""
import json
import os

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import route as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
W1 = json.load(open(os.path.join(GOLD, "w1.json")))
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))


def _w1_setup(mode, bstar):
    return O.Setup(grid=W1["grid"], thresholds=[0.7, 0.9], F=W1["F"],
                   instance_level=W1["instance_level"], bstar=bstar, mode=mode,
                   seed=W1["seed"], batch_seq=W1["batch_seq"])


def test_w1_greedy_and_uniform():
    lv = np.array(W1["levels"])
    for mode, bstar, key in ((O.GREEDY, 2, "greedy_bstar2"), (O.UNIFORM, 1, "uniform")):
        for solver in ("brute", "lp"):
            d = O.downstream(lv, _w1_setup(mode, bstar), solver)
            assert d["h"].tolist() == W1["h"] and d["f"].tolist() == W1["f"]
            assert d["x"].tolist() == W1["x"] and d["D_Q"] == W1["D_Q"]
            assert d["rank"].tolist() == W1["class_rank"]
            got = [[int(lv[p]), int(d["level_prime"][p]), int(d["instance"][p]), int(d["slot"][p])]
                   for p in range(len(lv))]
            assert got == W1[key]


@st.composite
def batch(draw):
    nK = draw(st.integers(2, 6))
    N = draw(st.integers(1, 300))
    seed = draw(st.integers(0, 2**32 - 1))
    rng = np.random.default_rng(seed)
    lv = rng.integers(0, nK, N)
    w = rng.random(nK) + 0.01
    F = (w / w.sum()).tolist()
    return nK, lv, F, seed


@settings(max_examples=80, deadline=None)
@given(batch(), st.sampled_from([1, 2, 4]), st.sampled_from([O.GREEDY, O.UNIFORM]))
def test_realised_counts_equal_plan(b, bstar, mode):
    nK, lv, F, seed = b
    grid = [5 * i for i in range(nK)]
    inst_level = list(range(nK)) + [nK - 1, 0]
    s = O.Setup(grid=grid, thresholds=[0.5 + 0.05 * i for i in range(nK - 1)], F=F,
                instance_level=inst_level, bstar=bstar if mode == O.GREEDY else 1, mode=mode,
                seed=seed, batch_seq=seed % 7)
    d = O.downstream(lv, s)
    x = d["x"]
    kp = d["level_prime"]
    for i in range(nK):
        for j in range(nK):
            assert int(np.sum((lv == i) & (kp == j))) == int(x[i, j])
    # K' counts equal f exactly (north_star: within one prompt of N F(K))
    assert np.array_equal(np.bincount(kp, minlength=nK), d["f"])
    assert np.all(np.abs(d["f"] - len(lv) * np.array(F)) < 1)
    # every instance serves only its own level; FIFO slots 0..c-1 in prompt order
    for w in range(len(inst_level)):
        mine = np.nonzero(d["instance"] == w)[0]
        assert np.all(kp[mine] == inst_level[w])
        assert sorted(d["slot"][mine].tolist()) == list(range(len(mine)))
        assert np.all(np.diff(d["slot"][mine]) > 0)                    # S:333 FIFO
    off, bp = d["offsets"], d["bucket_prompts"]
    assert sorted(bp.tolist()) == list(range(len(lv)))
    for w in range(len(inst_level)):
        seg = bp[off[w]:off[w + 1]]
        assert np.all(d["instance"][seg] == w) and np.all(np.diff(seg) > 0)


def test_no_redirection_when_h_equals_f():
    rng = np.random.default_rng(3)
    lv = rng.integers(0, 6, 1000)
    h = np.bincount(lv, minlength=6)
    s = O.Setup(grid=[0, 5, 10, 15, 20, 25], thresholds=[0.6] * 5, F=(h / 1000).tolist(),
                instance_level=list(range(6)))
    d = O.downstream(lv, s)
    assert np.array_equal(d["level_prime"], lv)


def test_route_prompt_row_25_always_25():
    """a plan row {25: 1.0} always gives 25."""
    lv = np.zeros(50, dtype=np.int64)
    s = O.Setup(grid=[0, 25], thresholds=[0.8], F=[0.0, 1.0], instance_level=[0, 1])
    d = O.downstream(lv, s)
    assert np.all(d["level_prime"] == 1)


def test_uniform_pick_is_multinomial():
    ex = SPEC["pick_worker_uniform"]
    lv = np.zeros(ex["n"], dtype=np.int64)
    s = O.Setup(grid=[0, 5], thresholds=[0.8], F=[1.0, 0.0], instance_level=[0] * ex["W"],
                mode=O.UNIFORM, bstar=1, seed=11)
    d = O.downstream(lv, s)
    counts = np.bincount(d["instance"], minlength=ex["W"])
    assert np.all(np.abs(counts - ex["mean"]) <= ex["tol"]), counts


def test_greedy_fills_bstar_batches():
    """b* = 4 -> batches of 4 in FIFO order; instance I_j[0] is filled first (R13)."""
    lv = np.zeros(10, dtype=np.int64)
    s = O.Setup(grid=[0, 5], thresholds=[0.8], F=[1.0, 0.0], instance_level=[0, 0, 1], bstar=4)
    d = O.downstream(lv, s)
    assert d["instance"].tolist() == [0, 0, 0, 0, 1, 1, 1, 1, 0, 0]
    assert d["slot"].tolist() == [0, 1, 2, 3, 0, 1, 2, 3, 4, 5]


def test_rank_sampler_uniform_over_seeds():
    """The member of a 6-prompt class that lands at rank 0 is uniform over seeds (chi^2)."""
    lv = np.zeros(6, dtype=np.int64)
    x = np.array([[6]])
    hits = np.zeros(6)
    for seed in range(3000):
        _, rank = O.redirect(lv, x, seed, 0)
        hits[int(np.argmin(rank))] += 1
    exp = 3000 / 6
    chi2 = float(np.sum((hits - exp) ** 2 / exp))
    assert chi2 < 20.5   # 5 dof, p ~ 1e-3


def test_determinism_and_batch_dependence():
    lv = np.random.default_rng(0).integers(0, 3, 200)
    x = np.array([[30, 20, 10], [0, 60, 10], [0, 0, 70]])
    lv = np.repeat([0, 1, 2], [60, 70, 70])
    a, _ = O.redirect(lv, x, 5, 1)
    b, _ = O.redirect(lv, x, 5, 1)
    c, _ = O.redirect(lv, x, 5, 2)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_route_on_synthetic_c1():
    """Composite O1..O10 on the C1 workload: invariants hold end to end."""
    import torch  # noqa: F401  (synth uses torch CPU generators)
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C1"]
    w = Workload(cfg)
    C = w.cache_rows(0, cfg.M).numpy()
    P = w.prompts(cfg.N).numpy()
    s = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=cfg.F,
                instance_level=cfg.instance_level, bstar=cfg.bstar, topk=cfg.topk)
    r = O.route(P, C, s)
    assert r.h.sum() == cfg.N and r.f.sum() == cfg.N
    assert np.all(np.diff(r.topk_score, axis=1) <= 0)
    S = O.similarity_A(P, C)
    assert np.allclose(r.topk_score[:, 0], S.max(axis=1))
    assert np.array_equal(r.topk_id[:, 0], S.argmax(axis=1))
    assert np.array_equal(np.bincount(r.level_prime, minlength=6), r.f)


def test_tier_a_flags_margins_pinned():
    """Flag bits 4 / 8 (north_star: margins below 2e-2 reported, not failed) on hand-built score rows
    just inside and just outside the margin, k = 1 (the next score comes from s1_next), sentinels,
    and the invalid / cold precedence (R16)."""
    from oracle import route as O
    thr = [0.65, 0.72, 0.79, 0.86, 0.93]
    t = np.asarray(thr, np.float32).astype(np.float64)
    eps = 1e-4
    sc = np.array([
        [0.50, 0.50 - 0.02 + eps],      # top-1 margin just below 2e-2        -> 4
        [0.50, 0.50 - 0.02 - eps],      # just above                          -> 0
        [t[2] + 0.02 - eps, 0.0],       # s1 just inside the band above t_2   -> 8
        [t[2] + 0.02 + eps, 0.0],       # just outside                        -> 0
        [t[4] - 0.02 + eps, 0.0],       # just below the top threshold        -> 8
        [t[0] - 0.02 - eps, 0.0],       # far below the lowest threshold      -> 0
        [t[1] + 0.005, t[1] - 0.001],   # both                                -> 12
        [0.40, -np.inf],                # M = 1: no second score              -> 0
        [0.40, 0.39],                   # invalid prompt: only 1
        [0.99, 0.98],
    ])
    valid = np.array([True] * 8 + [False, True])
    f = O.tier_a_flags(sc, np.full(10, -np.inf), thr, valid, cold=False)
    assert f.tolist() == [4, 0, 8, 0, 8, 0, 12, 0, 1, 4]
    # k = 1: the margin is taken against s1_next
    f1 = O.tier_a_flags(sc[:2, :1], np.array([0.50 - 0.02 + eps, 0.50 - 0.02 - eps]), thr, valid[:2], cold=False)
    assert f1.tolist() == [4, 0]
    # cold cache: 2 for valid prompts, 1 for invalid ones, never 4 / 8
    fc = O.tier_a_flags(sc, np.full(10, -np.inf), thr, valid, cold=True)
    assert fc.tolist() == [2] * 8 + [1, 2]
