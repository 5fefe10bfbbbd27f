"""NEXT f4's second half on the GPU: the exact route plan for arbitrary, non-convex degradation tables
(R37; PAPER.md P:89 leaves D's form open, Eq. 1 P:96 puts no convexity on it; SPEC S:264 asks for the
exact optimum).  K5's one-CTA min-cost-flow + lexicographic canonicalisation vs the oracle's
exhaustive search (<= 4 levels) and phased HiGHS LPs (<= 16 levels), bit for bit, plus the whole
routing path downstream of a non-convex plan."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import route as O
from synth import CONFIGS, Workload

from .parity import Report, check_downstream
from .test_oracle_plan import _r37_instances, r37_tie_instances

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _thresholds(nK):
    return [0.2 + 0.045 * m for m in range(nK - 1)]


def _cands(levels, thr, k=4):
    """Candidate lists [1][N][k] whose top-1 score lies mid-band of each prompt's level."""
    t = [-1.0] + list(thr) + [1.0]
    s1 = np.array([(t[l] + t[l + 1]) / 2 if 0 < l < len(thr) else (t[1] - 0.05 if l == 0 else t[-2] + 0.01)
                   for l in levels], dtype=np.float32)
    N = len(levels)
    sc = np.stack([s1 - 0.3 - 0.01 * m for m in range(k)], axis=1).astype(np.float32)
    sc[:, 0] = s1
    gid = np.arange(N * k, dtype=np.int32).reshape(N, k)
    pairs = np.stack([sc.view(np.int32), gid], axis=-1).reshape(1, N, k, 2)
    return torch.from_numpy(np.ascontiguousarray(pairs)).to(DEV)


class _Planner:
    """One context routing synthetic candidate lists: any (grid, c, h, f) instance in one call."""

    def __init__(self, pas, N_max):
        self.pas = pas
        self.r = pas.Router(d=768, topk=4, max_batch=N_max, max_rows_per_rank=1, device=0)
        self.r.load_cache(Workload(CONFIGS["C1"], device=DEV, M=1).cache_rows(0, 1).contiguous())

    def plan(self, grid, c, h, f, out_needed=False):
        nK, N = len(grid), int(sum(h))
        thr = _thresholds(nK)
        self.r.set_bands(grid, thr)
        self.r.set_degradation(list(c))
        F = [v / N for v in f]
        F[-1] = 1.0 - sum(F[:-1])
        self.r.set_fractions(F, list(range(nK)), 2, 0)
        levels = np.repeat(np.arange(nK), h)
        np.random.default_rng(N).shuffle(levels)
        o = self.r.alloc_out(N)
        self.pas.pas_route_from_candidates(self.r.ctx, _cands(levels, thr), 1, N, o)
        torch.cuda.synchronize()
        st = self.r.stats()
        assert st["h"] == list(h) and st["f"] == list(f), (st["h"], st["f"], list(h), list(f))
        return st, o, levels, F, thr


def test_nonconvex_plan_matches_bruteforce(pas):
    """300 random instances (<= 4 levels, N <= 8) and instances with (D, Q) ties: x == exhaustive search."""
    pl = _Planner(pas, 16)
    rng = np.random.default_rng(37)
    n = 0
    for grid, c, h, f in list(_r37_instances(rng, 300)) + r37_tie_instances(6):
        if O.is_convex(c):
            continue
        st, *_ = pl.plan(grid, c, h, f)
        want, _ = O.plan_int_bruteforce(h, f, grid, O.degradation_int(c))
        assert st["x"] == want.tolist(), (grid, list(h), list(f))
        assert st["plan_solver_iters"] >= 0 and np.isnan(st["D_Q_LP"])
        assert abs(st["D_Q"] - O.d_q(want, grid, c, int(sum(h)))) <= 1e-12
        n += 1
    assert n >= 150
    pl.r.close()


def test_nonconvex_plan_matches_lp_up_to_16_levels(pas):
    """Up to 16 levels and 131,072 prompts (the C5 peak batch): x == the phased HiGHS LP, D_Q within
    1e-5 relative (north_star)."""
    pl = _Planner(pas, 131072)
    rng = np.random.default_rng(1616)
    for case in range(16):
        nK = int(rng.integers(5, 17))
        grid = [0] + sorted(rng.choice(np.arange(1, 50), nK - 1, replace=False).tolist())
        kind = case % 3
        if kind == 0:     # arbitrary non-decreasing table
            c = np.concatenate([[0.0], np.sort(rng.uniform(0, 1, 49))])
        elif kind == 1:   # concave
            c = np.minimum(1.0, rng.uniform(0.05, 0.2) * np.sqrt(np.arange(50)))
        else:             # steps
            c = np.zeros(50)
            c[1:] = np.sort(rng.choice([0.1, 0.3, 0.6, 1.0], 49))
        if O.is_convex(c):
            continue
        N = int(rng.choice([97, 4096, 131072]))
        h = rng.multinomial(N, rng.dirichlet(np.ones(nK) * 0.7))
        f = rng.multinomial(N, rng.dirichlet(np.ones(nK) * 0.7))
        st, *_ = pl.plan(grid, c, h, f)
        want = O.plan_int_lp(h, f, grid, O.degradation_int(c))
        assert st["x"] == want.tolist(), (case, nK, N)
        ref = O.d_q(want, grid, c, N)
        assert abs(st["D_Q"] - ref) <= 1e-5 * abs(ref) + 1e-15
        print(f"case {case}: nK={nK} N={N} iters={st['plan_solver_iters']} plan_ms={st['stage_ms'][3]:.3f}")
    pl.r.close()


def test_nonconvex_table_end_to_end(pas):
    """C2 (4,096 prompts vs 100k rows, skewed H_K vs F_K) with a concave table: the whole path --
    K, plan, K', instances, slots, batch lists -- bit-exact vs the oracle teacher-forced on the GPU's K."""
    cfg = CONFIGS["C2"]
    N, M = cfg.N, 20_000
    w = Workload(cfg, device=DEV, M=M)
    C_ = w.cache_rows(0, M).contiguous()
    P = w.prompts(N)
    c = list(np.minimum(1.0, 0.09 * np.arange(50)))
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_degradation(c)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    r.load_cache(C_)
    out = r.route(P)
    torch.cuda.synchronize()
    st = r.stats()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    lev = np.searchsorted(np.asarray(cfg.grid), g["K"])
    setup = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=cfg.F, instance_level=cfg.instance_level,
                    bstar=cfg.bstar, mode=cfg.mode, c=np.asarray(c), topk=cfg.topk, seed=cfg.route_seed)
    d = check_downstream(g, lev, setup, st, Report(), len(cfg.instance_level))
    nw_D = O.d_q(O.plan_lp(d["h"], d["f"], cfg.grid, O.default_degradation()), cfg.grid, c, N)
    print(f"concave c: D_Q {st['D_Q']:.6f} (NW-corner plan would give {nw_D:.6f}), iters {st['plan_solver_iters']}")
    assert st["D_Q"] <= nw_D + 1e-15
    r.close()


def test_degradation_validation(pas):
    r = pas.Router(d=768, topk=4, max_batch=8, max_rows_per_rank=1, device=0)
    r.set_bands([0, 25], [0.9])
    E = pas.PasError
    with pytest.raises(E) as ei:
        r.set_degradation([0.0] + [2.0] * 49)                    # non-convex above 1
    assert ei.value.status == -6
    with pytest.raises(E) as ei:
        r.set_degradation([0.0, 0.5, 0.4] + [0.5] * 47)          # decreasing
    assert ei.value.status == -6
    r.set_degradation([0.0] + [0.5] * 49)                        # non-convex, accepted
    with pytest.raises(E) as ei:
        r.set_forecast(100, 1)                                   # forecast mode needs a convex c
    assert ei.value.status == -6
    r.set_degradation([0.006 * t for t in range(50)])
    r.set_forecast(100, 1)
    with pytest.raises(E) as ei:
        r.set_degradation([0.0] + [0.5] * 49)
    assert ei.value.status == -6
    r.close()
