"""GPU parity of the f2 cache maintenance (R25-R27) vs oracle/cache.py.

A stream of batches on a small store: route (the GPU's top-k checked against the oracle on the
store's CURRENT contents with the parity protocol), touch (teacher-forced on the GPU's top-1 ids,
which the protocol has just checked), insert the vanilla-served prompts (LRU eviction, slot reuse),
and compare the gids handed out and the full stamp array bit for bit, batch after batch.  Also:
explicit inserts with eviction, invalid rows (nothing changes), re-retrieval of inserted rows
(insert v then nearest(v) = 1), and G = 2 virtual shards = G = 1.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import cache as OC
from oracle import route as O
from synth import CONFIGS, Workload

from .parity import Report, check_topk

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _router(pas, cfg, N, cap, world=1, rank=0):
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=cap, device=0, rank=rank, world=world,
                   seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    return r


def _stamps(pas, r, n):
    t = torch.zeros(n, dtype=torch.int32, device=DEV)
    pas.pas_cache_stamps(r.ctx, t)
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def _oracle_topk(store, P, k):
    g, rows = store.contents()
    S = O.similarity_A(np.where(O.row_valid(P)[:, None], P, 1.0), rows)
    ids, sc = O.topk_sorted(S, g, k + 1)
    return ids, sc


def test_lru_stream_vanilla_inserts(pas):
    cfg = CONFIGS["C2"]            # most prompts want K = 0 -> many vanilla inserts
    N, cap, M0 = 256, 1280, 1250
    w = Workload(cfg, device=DEV, M=4000)
    r = _router(pas, cfg, N, cap)
    store = OC.LruStore(capacity=cap, d=cfg.d)
    C0 = w.cache_rows(0, M0).contiguous()
    r.load_cache(C0)
    store.load(C0.cpu().numpy())
    P_all = w.prompts(N * 6)
    k = cfg.topk
    evicted_total = 0
    for b in range(6):
        P = P_all[b * N:(b + 1) * N].contiguous()
        out = r.route(P)
        torch.cuda.synchronize()
        g = {kk: v.cpu().numpy() for kk, v in out.items()}
        Ph = P.cpu().numpy()
        valid = O.row_valid(Ph)
        o_ids, o_sc = _oracle_topk(store, Ph, k)
        rep = Report()
        check_topk(g["topk_id"].reshape(N, k), g["topk_score"].reshape(N, k), o_ids, o_sc, rep)
        store.touch(g["topk_id"].reshape(N, k)[:, 0], valid)            # teacher-forced top-1
        gids = torch.full((N,), -7, dtype=torch.int32, device=DEV)
        n = r.insert_vanilla(P, out["K_prime"], gids)
        torch.cuda.synchronize()
        lev_p = np.searchsorted(np.asarray(cfg.grid), g["K_prime"])
        rows, idx = OC.vanilla_rows(Ph, lev_p, valid)
        used_before = store.used
        exp = store.insert(rows) if len(rows) else []
        evicted_total += len(rows) - (store.used - used_before)
        got = gids.cpu().numpy()
        assert n == len(rows)
        assert np.all(got[np.setdiff1d(np.arange(N), idx)] == -1)
        assert list(got[idx]) == exp, f"batch {b}: gids differ"
        st = _stamps(pas, r, store.used)
        assert all(st[gg] == store.stamp[gg] for gg in store.stamp), f"batch {b}: stamps differ"
        assert pas.pas_cache_size(r.ctx)[0] == store.used
    assert evicted_total > 0                                            # the stream did wrap the store
    # the last inserted rows are retrieved as their own nearest entries
    Plast = P_all[5 * N:].contiguous()
    out = r.route(Plast)
    torch.cuda.synchronize()
    top1 = out["topk_id"].view(N, k)[:, 0].cpu().numpy()
    s1 = out["topk_score"].view(N, k)[:, 0].cpu().numpy()
    mine = got >= 0
    assert np.all(top1[mine] == got[mine]) and np.all(s1[mine] > 0.999)
    r.close()


def test_lru_explicit_insert_and_invalid_rows(pas):
    cfg = CONFIGS["C1"]
    cap = 300
    w = Workload(cfg, device=DEV, M=2000)
    r = _router(pas, cfg, 256, cap)
    store = OC.LruStore(capacity=cap, d=cfg.d)
    for b, n in enumerate((200, 180, 256, 90)):
        rows = w.cache_rows(b * 300, b * 300 + n).contiguous()
        out = torch.empty(n, dtype=torch.int32, device=DEV)
        r.insert(rows, out)
        exp = store.insert(rows.cpu().numpy())
        assert list(out.cpu().numpy()) == exp
        if b == 1:                                  # a routed batch between inserts touches entries
            P = w.prompts(64)
            o = r.route(P)
            torch.cuda.synchronize()
            store.touch(o["topk_id"].view(64, -1)[:, 0].cpu().numpy(), O.row_valid(P.cpu().numpy()))
    st = _stamps(pas, r, cap)
    assert all(st[g] == store.stamp[g] for g in store.stamp)
    bad = w.cache_rows(0, 10).contiguous()
    bad[3, 5] = float("nan")
    with pytest.raises(pas.PasError) as ei:
        r.insert(bad)
    assert ei.value.status == -10
    assert np.array_equal(_stamps(pas, r, cap), st)            # nothing inserted, nothing evicted
    with pytest.raises(pas.PasError):
        r.insert(w.cache_rows(0, 257).contiguous())            # > max_batch
    r.close()


def test_lru_virtual_shards_match_single_gpu(pas):
    """G = 2 contexts (round-robin slots) doing the same loads, routes and inserts stay identical
    to G = 1: same gids, same stamps, same routing outputs."""
    cfg = CONFIGS["C2"]
    N, cap = 200, 900
    w = Workload(cfg, device=DEV, M=3000)
    one = _router(pas, cfg, N, cap)
    two = [_router(pas, cfg, N, cap // 2 + 1, world=2, rank=rk) for rk in range(2)]
    C0 = w.cache_rows(0, 850).contiguous()
    for r in [one] + two:
        r.load_cache(C0)
    P_all = w.prompts(N * 4)
    k = cfg.topk
    for b in range(4):
        P = P_all[b * N:(b + 1) * N].contiguous()
        ref = one.route(P)
        cands = torch.empty(2, N * k, dtype=torch.int64, device=DEV)
        for rk, r in enumerate(two):
            pas.pas_route_local(r.ctx, P, cands[rk])
        outs = []
        for r in two:                               # every rank merges all N (and touches)
            o = r.alloc_out(N)
            pas.pas_route_from_candidates(r.ctx, cands, 2, N, o)
            outs.append(o)
        torch.cuda.synchronize()
        for o in outs:
            for key in ("K", "K_prime", "instance", "slot", "topk_id", "topk_score"):
                assert torch.equal(o[key], ref[key]), (b, key)
        g1 = torch.full((N,), -1, dtype=torch.int32, device=DEV)
        n1 = one.insert_vanilla(P, ref["K_prime"], g1)
        for r, o in zip(two, outs):
            g2 = torch.full((N,), -1, dtype=torch.int32, device=DEV)
            n2 = r.insert_vanilla(P, o["K_prime"], g2)
            assert n2 == n1 and torch.equal(g2, g1), b
    n = pas.pas_cache_size(one.ctx)[0]
    s1 = _stamps(pas, one, n)
    for r in two:
        assert np.array_equal(_stamps(pas, r, n), s1)
    for r in [one] + two:
        r.close()
