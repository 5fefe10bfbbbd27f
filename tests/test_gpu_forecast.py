"""GPU parity of the forecast-driven mode (R21-R24) vs oracle/forecast.py.

Batch after batch, teacher-forced on the GPU's optimal-K levels (their own parity is covered by
test_gpu_parity.py), the oracle's ForecastRouter and the CUDA path must agree bit for bit on K',
instance, slot, buckets, the window state, the fixed-point plan (Hc, Fc), the realised moves and
counts, and exactly on D_Q (realised), the plan's D_Q and the L2 forecast error (same fp64
operations in the same order on both sides).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import forecast as OF
from oracle import route as O
from synth import CONFIGS, Workload

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _router(pas, cfg, N, M, mode=None, bstar=None):
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=max(M, 1), device=0,
                   seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar if bstar is None else bstar,
                    cfg.mode if mode is None else mode)
    return r


def _check_batch(g, st, ref, grid, W, N):
    grid = np.asarray(grid)
    assert np.array_equal(g["K_prime"], grid[ref["level_prime"]]), "K' differs"
    assert np.array_equal(g["instance"], ref["instance"]), "instance differs"
    assert np.array_equal(g["slot"], ref["slot"]), "slot differs"
    assert np.array_equal(g["bucket_offsets"][:W + 1], ref["offsets"]), "bucket offsets differ"
    assert np.array_equal(g["bucket_prompts"], ref["bucket_prompts"]), "bucket prompts differ"
    assert st["forecast"] == 1
    assert st["h"] == ref["h"].tolist()
    assert st["x"] == ref["x"].tolist(), "realised moves differ"
    assert st["f"] == ref["f"].tolist()
    assert st["fc_replanned"] == int(ref["replanned"])
    assert st["fc_plan_n"] == ref["plan_n"] and st["fc_plan_counts"] == list(ref["plan_counts"])
    assert st["fc_Hc"] == ref["Hc"] and st["fc_Fc"] == ref["Fc"], "fixed-point plan differs"
    assert st["n_unforecast"] == ref["n_unforecast"]
    assert st["D_Q"] == ref["D_Q"], (st["D_Q"], ref["D_Q"])
    assert st["D_Q_LP"] == ref["D_Q_plan"], (st["D_Q_LP"], ref["D_Q_plan"])
    assert st["fc_l2_error"] == ref["l2"], (st["fc_l2_error"], ref["l2"])
    assert sum(st["bucket_count"]) == N


def _run_stream(pas, name, N, M, batches, window, replan_every=1, mode=None, bstar=None, F_at=None):
    cfg = CONFIGS[name]
    w = Workload(cfg, device=DEV, M=max(M, 1000))     # M = 0: prompts drawn as usual, cache left cold
    r = _router(pas, cfg, N, M, mode, bstar)
    if M:
        r.load_cache(w.cache_rows(0, M).contiguous())
    r.set_forecast(window, replan_every)
    s = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=list(cfg.F), instance_level=cfg.instance_level,
                bstar=cfg.bstar if bstar is None else bstar, mode=cfg.mode if mode is None else mode,
                topk=cfg.topk, seed=cfg.route_seed)
    fr = OF.ForecastRouter(len(cfg.grid), window, replan_every)
    P_all = w.prompts(N * batches)
    l2 = []
    for b in range(batches):
        if F_at is not None and b == F_at[0]:
            s.F = list(F_at[1])
            r.set_fractions(s.F, cfg.instance_level, s.bstar, s.mode)
        out = r.route(P_all[b * N:(b + 1) * N].contiguous())
        torch.cuda.synchronize()
        st = r.stats()
        g = {k: v.cpu().numpy() for k, v in out.items()}
        level = np.searchsorted(np.asarray(cfg.grid), g["K"])
        s.batch_seq = b
        ref = fr.batch(level, s, O)
        _check_batch(g, st, ref, cfg.grid, len(cfg.instance_level), N)
        assert st["fc_window_n"] == min(window, N * (b + 1))
        l2.append(st["fc_l2_error"])
    r.close()
    return l2


def test_forecast_c2_window1000_every_batch(pas):
    l2 = _run_stream(pas, "C2", N=600, M=7000, batches=5, window=1000)
    print("l2 per batch", l2)
    assert l2[0] > 0 and max(l2[2:]) < 0.2     # empty window (uniform) first, then a real forecast


def test_forecast_replan_period_and_F_change(pas):
    _run_stream(pas, "C2", N=300, M=5000, batches=7, window=700, replan_every=3,
                F_at=(4, [0.30, 0.10, 0.10, 0.10, 0.10, 0.30]))


def test_forecast_uniform_mode(pas):
    _run_stream(pas, "C1", N=64, M=1000, batches=4, window=50, mode=1, bstar=1)


def test_forecast_window_smaller_than_batch_and_cold_cache(pas):
    _run_stream(pas, "C2", N=500, M=0, batches=3, window=128)       # cold: every K = 0


def test_forecast_off_returns_to_exact_plan(pas):
    cfg = CONFIGS["C2"]
    N, M = 400, 4000
    w = Workload(cfg, device=DEV, M=M)
    r = _router(pas, cfg, N, M)
    r.load_cache(w.cache_rows(0, M).contiguous())
    P = w.prompts(N)
    r.set_forecast(100)
    r.route(P)
    r.set_forecast(0)
    r.set_seed(cfg.route_seed, 0)
    out = r.route(P)
    torch.cuda.synchronize()
    st = r.stats()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    level = np.searchsorted(np.asarray(cfg.grid), g["K"])
    s = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=cfg.F, instance_level=cfg.instance_level,
                bstar=cfg.bstar, mode=cfg.mode, topk=cfg.topk, seed=cfg.route_seed, batch_seq=0)
    d = O.downstream(level, s)
    assert st["forecast"] == 0
    assert np.array_equal(g["K_prime"], np.asarray(cfg.grid)[d["level_prime"]])
    assert np.array_equal(g["instance"], d["instance"]) and np.array_equal(g["slot"], d["slot"])
    r.close()


def test_forecast_large_batch_from_candidates(pas):
    """200,000 prompts through pas_route_from_candidates (many blocks tally the moves)."""
    cfg = CONFIGS["C4"]
    N, k, S = 200_000, cfg.topk, 1
    g = torch.Generator(device=DEV).manual_seed(11)
    sc = torch.rand(S, N, k, generator=g, device=DEV) * 0.8 + 0.2
    sc, _ = torch.sort(sc, dim=-1, descending=True)
    gid = torch.randint(0, 1 << 30, (S, N, k), generator=g, device=DEV, dtype=torch.int32)
    cand = torch.stack([sc.view(torch.int32), gid], dim=-1).contiguous()
    r = pas.Router(d=cfg.d, topk=k, max_batch=N, max_rows_per_rank=1, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    r.load_cache(Workload(cfg, device=DEV, M=1).cache_rows(0, 1).contiguous())
    r.set_forecast(1000, 1)
    s = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=list(cfg.F), instance_level=cfg.instance_level,
                bstar=cfg.bstar, mode=cfg.mode, topk=k, seed=cfg.route_seed)
    fr = OF.ForecastRouter(len(cfg.grid), 1000, 1)
    o = r.alloc_out(N)
    s1 = sc[0, :, 0].cpu().numpy().astype(np.float64)
    level = O.optimal_k_level(s1, cfg.thresholds, np.ones(N, bool))
    for b in range(2):
        pas.pas_route_from_candidates(r.ctx, cand, S, N, o)
        torch.cuda.synchronize()
        st = r.stats()
        gh = {kk: v.cpu().numpy() for kk, v in o.items()}
        assert np.array_equal(np.searchsorted(np.asarray(cfg.grid), gh["K"]), level)
        s.batch_seq = b
        ref = fr.batch(level, s, O)
        _check_batch(gh, st, ref, cfg.grid, len(cfg.instance_level), N)
    r.close()


def test_set_forecast_validation(pas):
    cfg = CONFIGS["C1"]
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=8, max_rows_per_rank=8, device=0)
    with pytest.raises(pas.PasError):
        r.set_forecast(10)                   # bands first
    r.set_bands(cfg.grid, cfg.thresholds)
    for bad in ((-1, 1), (10, 0), (pas.PAS_MAX_FORECAST_WINDOW + 1, 1)):
        with pytest.raises(pas.PasError):
            r.set_forecast(*bad)
    r.set_forecast(10, 2)
    r.set_forecast(0)
    r.close()
