"""CPU pins of the GPU-vs-oracle parity protocol itself (tests/parity.py): the whole-cache Tier-B
check (SURVEY 8(c).6 S1/S2 "internally") must accept a correct fp32-accumulating result and reject
the plausible kernel bugs it exists to catch -- a lost candidate (a skipped tile or range boundary),
two swapped ids, a score off by more than TAU_B, a level flipped away from a threshold -- and it
must grade most positions on the synth-v1 workload (the Tier-A rule alone grades ~2 %)."""
import numpy as np
import pytest

from oracle import route as O
from synth import BLOCK, CONFIGS, Workload

from .parity import (TAU_B, Report, check_levels_tier_b, check_topk_tier_b, oracle_topk_ab)


def _fp32_topk(Pq, Cq, k):
    """A stand-in for the GPU: fp32 accumulation of the bf16 products (sgemm), top-k by (s desc, g asc)."""
    S = (Pq.astype(np.float32) @ Cq.astype(np.float32).T).astype(np.float64)
    n, m = S.shape
    ids = np.full((n, k), -1, dtype=np.int64)
    sc = np.full((n, k), -np.inf)
    for p in range(n):
        o = np.lexsort((np.arange(m), -S[p]))[:k]
        ids[p, :len(o)] = o
        sc[p, :len(o)] = S[p, o]
    return ids, sc


@pytest.fixture(scope="module")
def problem():
    cfg = CONFIGS["C2"]
    M = 3 * BLOCK // 4 + 777          # one ragged chunk
    w = Workload(cfg, device="cpu", M=M)
    P = w.prompts(160).numpy()
    C = w.cache_rows(0, M).numpy()
    r = oracle_topk_ab(P, [(0, C[:20000]), (20000, C[20000:])], cfg.topk, workers=4)
    Pq, _ = O.quantize(P)
    Cq, _ = O.quantize(C)
    gi, gs = _fp32_topk(Pq, Cq, cfg.topk)
    return cfg, P, C, r, gi, gs


def test_streamed_two_tier_scan_equals_whole_matrix(problem):
    """The chunked, thread-pooled scan = the oracle's top-k of the whole score matrices."""
    cfg, P, C, r, _, _ = problem
    k1 = cfg.topk + 1
    ia, sa = O.topk_sorted(O.similarity_A(P, C), np.arange(len(C)), k1)
    Pq, _ = O.quantize(P)
    Cq, _ = O.quantize(C)
    ib, sb = O.topk_sorted(O.similarity_B(Pq, Cq), np.arange(len(C)), k1)
    assert np.array_equal(r["ids_A"], ia) and np.array_equal(r["sc_A"], sa)
    assert np.array_equal(r["ids_B"], ib) and np.array_equal(r["sc_B"], sb)


def test_correct_fp32_result_passes_and_grades_most_positions(problem):
    cfg, P, C, r, gi, gs = problem
    rep = Report()
    rep.positions = int(np.isfinite(gs).sum())
    check_topk_tier_b(gi, gs, r["ids_B"], r["sc_B"], rep, floor=0.9)
    assert rep.frac_B() >= 0.9 and rep.max_score_err_B < TAU_B / 2
    usable = r["valid"]
    check_levels_tier_b(O.optimal_k_level(gs[:, 0], cfg.thresholds, usable), r["sc_B"][:, 0], usable,
                        cfg.thresholds, rep)
    assert rep.levels_B >= 0.98 * len(gi)


def _graded_position(r, k):
    sb = r["sc_B"]
    prev = np.concatenate([np.full((len(sb), 1), np.inf), sb[:, :k - 1]], axis=1)
    marg = np.minimum(prev - sb[:, :k], sb[:, :k] - sb[:, 1:k + 1])
    p, m = np.argwhere(marg >= 2 * TAU_B)[len(sb) // 2]
    return int(p), int(m)


def test_lost_candidate_is_caught(problem):
    """A candidate dropped (a skipped tail tile, a lost range boundary): the list shifts up."""
    cfg, _, _, r, gi, gs = problem
    p, m = _graded_position(r, cfg.topk)
    bi, bs = gi.copy(), gs.copy()
    bi[p, m:-1], bs[p, m:-1] = gi[p, m + 1:], gs[p, m + 1:]
    bi[p, -1], bs[p, -1] = r["ids_B"][p, cfg.topk], r["sc_B"][p, cfg.topk]
    with pytest.raises(AssertionError):
        check_topk_tier_b(bi, bs, r["ids_B"], r["sc_B"], Report())


def test_swapped_ids_and_score_offsets_are_caught(problem):
    cfg, _, _, r, gi, gs = problem
    p, m = _graded_position(r, cfg.topk)
    q = m + 1 if m + 1 < cfg.topk else m - 1
    bi = gi.copy()
    bi[p, [m, q]] = bi[p, [q, m]]
    with pytest.raises(AssertionError):
        check_topk_tier_b(bi, gs, r["ids_B"], r["sc_B"], Report())
    bs = gs.copy()
    bs[p, m] += 1.5 * TAU_B
    with pytest.raises(AssertionError):
        check_topk_tier_b(gi, bs, r["ids_B"], r["sc_B"], Report())


def test_level_flip_away_from_threshold_is_caught(problem):
    cfg, _, _, r, gi, gs = problem
    usable = r["valid"]
    lev = O.optimal_k_level(gs[:, 0], cfg.thresholds, usable)
    t = np.asarray(cfg.thresholds, np.float32).astype(np.float64)
    far = np.nonzero(np.min(np.abs(r["sc_B"][:, :1] - t[None, :]), axis=1) >= 1e-3)[0]
    bad = lev.copy()
    bad[far[0]] = (bad[far[0]] + 1) % len(cfg.grid)
    with pytest.raises(AssertionError):
        check_levels_tier_b(bad, r["sc_B"][:, 0], usable, cfg.thresholds, Report())


def test_floor_fails_a_vacuous_check(problem):
    """With every position a near-tie (all scores equal) nothing is graded and the floor trips."""
    cfg, _, _, r, gi, gs = problem
    flat = np.zeros_like(r["sc_B"])
    with pytest.raises(AssertionError):
        check_topk_tier_b(gi, np.zeros_like(gs), r["ids_B"], flat, Report(), floor=0.5)
