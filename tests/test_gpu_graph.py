"""CUDA-graph replay of the whole batch (pas_set_graph): the
batch-varying state (Philox batch_seq, LRU tick, K2 epoch) lives on the device, so replaying a captured
batch is exactly the eager batch -- checked byte for byte over sequences that change prompts in place,
fractions, the cache (inserts), the seed, and the modes the graph serves."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from synth import CONFIGS, Workload

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _router(pas, cfg, N, M, mode=None, bstar=None, topk=None):
    r = pas.Router(d=cfg.d, topk=topk or cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar if bstar is None else bstar, cfg.mode if mode is None else mode)
    return r


def _run(pas, graph, cfg, N, M, steps, mode=None, bstar=None, topk=None):
    """Route a scripted sequence; returns per-batch host outputs + stats + the LRU stamps."""
    w = Workload(cfg, device=DEV, M=M + 4096)
    C_ = w.cache_rows(0, M).contiguous()
    r = _router(pas, cfg, N, M + 4096, mode, bstar, topk)
    r.load_cache(C_)
    if graph:
        pas.pas_set_graph(r.ctx, True)
    emb = torch.empty(N, cfg.d, device=DEV)
    out = r.alloc_out(N)
    res = []
    for b, act in enumerate(steps):
        if act == "fractions":   # half of the mass onto the first level that has an instance
            F = [0.5 * f for f in cfg.F]
            F[min(cfg.instance_level)] += 0.5
            r.set_fractions(F, cfg.instance_level, cfg.bstar if bstar is None else bstar,
                            cfg.mode if mode is None else mode)
        elif act == "insert":
            r.insert(w.cache_rows(M, M + min(N, 1000)).contiguous())
        elif act == "seed":
            r.set_seed(cfg.route_seed ^ 0x1234, 7)
        P = w.prompts(N, batch=b)
        if b == 1:
            P[3] = 0.0
        emb.copy_(P)                       # same buffer every batch: the captured graph reads it
        r.route(emb, out)
        torch.cuda.synchronize()
        st = r.stats()
        stamps = torch.empty(M + 4096, dtype=torch.int32, device=DEV)
        pas.pas_cache_stamps(r.ctx, stamps)
        torch.cuda.synchronize()
        res.append(({k: v.cpu().numpy().copy() for k, v in out.items()},
                    {k: st[k] for k in ("h", "f", "x", "D_Q", "n_invalid", "n_near_top1", "n_redirected")},
                    stamps.cpu().numpy()))
    launches = pas.pas_last_launch_count(r.ctx)
    r.close()
    return res, launches


@pytest.mark.parametrize("name,N,M,mode,bstar,topk", [("C1", 64, 1000, 0, 4, 8), ("C1", 64, 1000, 1, 1, 8),
                                                      ("C2", 4096, 100_000, 0, 4, 8), ("C3", 700, 20_000, 0, 3, 5)])
def test_graph_replay_equals_eager(pas, name, N, M, mode, bstar, topk):
    cfg = CONFIGS[name]
    steps = ["", "", "fractions", "", "insert", "", "seed", ""]
    eager, _ = _run(pas, False, cfg, N, M, steps, mode, bstar, topk)
    graph, launches = _run(pas, True, cfg, N, M, steps, mode, bstar, topk)
    W = len(cfg.instance_level)
    for b, ((go, gs, gst), (eo, es, est)) in enumerate(zip(graph, eager)):
        for key in go:
            a, c = go[key], eo[key]
            if key == "bucket_offsets":
                a, c = a[:W + 1], c[:W + 1]
            assert np.array_equal(a, c), (b, key)
        assert gs == es, b
        assert np.array_equal(gst, est), b
    assert launches > 0


def test_graph_latency_c1(pas):
    """C1 (64 prompts vs 1,000 rows): one replay vs the eager launches, device time per batch."""
    cfg = CONFIGS["C1"]
    N, M = cfg.N, cfg.M
    w = Workload(cfg, device=DEV, M=M)
    r = _router(pas, cfg, N, M)
    r.load_cache(w.cache_rows(0, M).contiguous())
    emb = w.prompts(N).contiguous()
    out = r.alloc_out(N)
    res = {}
    for graph in (False, True):
        pas.pas_set_graph(r.ctx, graph)
        for _ in range(20):
            r.route(emb, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(500):
            r.route(emb, out)
        e1.record()
        torch.cuda.synchronize()
        res[graph] = e0.elapsed_time(e1) / 500 * 1e3
    print(f"C1 per batch: eager {res[False]:.1f} us, graph {res[True]:.1f} us")
    r.close()


@pytest.mark.parametrize("N,M,topk,mode,bstar,nonconvex,cold", [
    (64, 1000, 8, 0, 4, False, False), (64, 1000, 8, 1, 1, False, False), (1, 1, 8, 0, 4, False, False),
    (700, 20_000, 16, 0, 3, False, False), (1024, 150_000, 5, 0, 4, True, False), (333, 4000, 1, 1, 1, False, False),
    (100, 0, 8, 0, 4, False, True)])
def test_small_path_equals_multi_kernel_chain(pas, monkeypatch, N, M, topk, mode, bstar, nonconvex, cold):
    """The one-CTA latency path (k_small.cu) vs the multi-kernel chain it replaces (PAS_SMALL_MAX=0),
    byte for byte: outputs, plan stats, flags counters, LRU stamps -- incl. many cache ranges (S > 1),
    k = 1 / 16, uniform mode, a non-convex table, invalid prompts and a cold cache."""
    cfg = CONFIGS["C2"]
    res = []
    for small in (True, False):
        if not small:
            monkeypatch.setenv("PAS_SMALL_MAX", "0")
        w = Workload(cfg, device=DEV, M=max(M, 1))
        r = _router(pas, cfg, N, max(M, 1), mode, bstar, topk)
        if nonconvex:
            r.set_degradation(list(np.minimum(1.0, 0.09 * np.arange(50))))
            r.set_fractions(cfg.F, cfg.instance_level, bstar, mode)
        if not cold:
            r.load_cache(w.cache_rows(0, M).contiguous())
        P = w.prompts(N)
        if N > 10:
            P[7] = 0.0
            P[9, 3] = float("nan")
        out = r.route(P.contiguous())
        torch.cuda.synchronize()
        st = r.stats()
        stamps = torch.empty(max(M, 1), dtype=torch.int32, device=DEV)
        pas.pas_cache_stamps(r.ctx, stamps)
        torch.cuda.synchronize()
        res.append(({k: v.cpu().numpy() for k, v in out.items()}, st, stamps.cpu().numpy()))
        r.close()
    monkeypatch.delenv("PAS_SMALL_MAX")
    (a, sa, ta), (b, sb, tb) = res
    W = len(cfg.instance_level)
    for key in a:
        x, y = (a[key][:W + 1], b[key][:W + 1]) if key == "bucket_offsets" else (a[key], b[key])
        assert np.array_equal(x, y), key
    for key in ("h", "f", "x", "D_Q", "n_invalid", "n_near_top1", "n_near_threshold", "n_redirected",
                "n_upgraded", "n_downgraded", "bucket_count"):
        assert sa[key] == sb[key], key
    assert np.array_equal(ta, tb)
