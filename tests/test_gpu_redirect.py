"""GPU parity of K6 (redirection by split-rank selection, csrc/k_redirect.cu) at large batch sizes.

The GPU's K' must equal the oracle's O8 (oracle/route.py redirect: Philox keys, a full lexsort by
(class, kappa, p), rank within class, X-interval lookup) bit for bit, on batches big enough that the
selection uses many buckets per class (kb = 12..16), with skewed level mixes, empty classes and tiny
plan entries (several split ranks inside one bucket), greedy and uniform.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import philox
from oracle import route as O
from synth import CONFIGS

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _candidates(level_scores, k):
    """Candidate lists whose top-1 score is given (so the optimal-K level is known)."""
    N = len(level_scores)
    s1 = torch.tensor(level_scores, dtype=torch.float32, device=DEV)
    sc = torch.stack([s1 - 1e-3 * j for j in range(k)], dim=1)[None]
    gid = torch.arange(N * k, dtype=torch.int32, device=DEV).view(1, N, k)
    return torch.stack([sc.contiguous().view(torch.int32), gid], dim=-1).contiguous()


@pytest.mark.parametrize("fallback", [0, 1])
@pytest.mark.parametrize("N,probs,F,mode", [
    (200_000, [0.6, 0.05, 0.05, 0.05, 0.05, 0.2], [0.05, 0.05, 0.1, 0.1, 0.2, 0.5], 0),
    (1 << 22, [0.02, 0.03, 0.15, 0.2, 0.25, 0.35], [0.5, 1e-5, 1e-5, 2e-5, 0.2, 0.29996], 0),
    (1 << 22, [0.0, 0.5, 0.0, 0.0, 0.0, 0.5], [0.25, 0.25, 0.0, 0.25, 0.0, 0.25], 1),
    (3001, [0.3, 0.1, 0.1, 0.1, 0.1, 0.3], [0.1, 0.1, 0.2, 0.2, 0.2, 0.2], 0),
    (300_007, [0.1, 0.2, 0.1, 0.2, 0.1, 0.3], [0.3, 0.1, 0.1, 0.1, 0.1, 0.3], 1),
])
def test_k6_large_batches(pas, N, probs, F, mode, fallback, monkeypatch):
    """fallback 0: the windowed split search (k6_fused + zone select / apply; N >= 2^18) or, below that,
    the exact histogram path alone; 1: the exact path forced (PAS_K6_FALLBACK) -- all bit-exact vs the
    oracle's full sort."""
    if fallback:
        monkeypatch.setenv("PAS_K6_FALLBACK", "1")
    cfg = CONFIGS["C4"]
    k = cfg.topk
    rng = np.random.default_rng(N + mode)
    level = rng.choice(6, size=N, p=np.asarray(probs) / np.sum(probs))
    # a top-1 score in the middle of each level's band (bands: 0.65/0.72/0.79/0.86/0.93)
    mid = np.array([0.30, 0.685, 0.755, 0.825, 0.895, 0.97])
    cand = _candidates(mid[level].tolist(), k)
    inst = [0, 1, 2, 3, 4, 5, 5, 0]
    bstar = 4 if mode == 0 else 1
    r = pas.Router(d=cfg.d, topk=k, max_batch=N, max_rows_per_rank=1, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(F, inst, bstar, mode)
    r.load_cache(torch.ones(1, cfg.d, device=DEV))      # a warm cache: K comes from the candidates
    o = r.alloc_out(N, optional=False)
    o["bucket_offsets"] = torch.empty(pas.PAS_MAX_INSTANCES + 1, dtype=torch.int32, device=DEV)
    o["bucket_prompts"] = torch.empty(N, dtype=torch.int32, device=DEV)
    for b in range(2):
        pas.pas_route_from_candidates(r.ctx, cand, 1, N, o)
        torch.cuda.synchronize()
        st = r.stats()
        assert st["k6_fallback"] == fallback          # the windowed path decides every prompt itself
        K = o["K"].cpu().numpy()
        Kp = o["K_prime"].cpu().numpy()
        assert np.array_equal(np.searchsorted(np.asarray(cfg.grid), K), level)
        h = O.histogram(level, 6)
        f = O.apportion(F, N)
        x = O.plan_lp(h, f, cfg.grid, O.default_degradation())
        assert st["x"] == x.tolist()
        kp, _ = O.redirect(level, x, cfg.route_seed, b)
        assert np.array_equal(np.searchsorted(np.asarray(cfg.grid), Kp), kp), f"batch {b}: K' differs"
        if mode == 1:   # uniform: the instance is drawn at the K' level (R14)
            u = philox.uniform_words(N, cfg.route_seed, b).astype(np.uint64)
            I = O.instance_lists(inst, 6)
            nj = np.array([len(I[j]) for j in range(6)], dtype=np.uint64)[kp]
            pick = ((u * nj) >> np.uint64(32)).astype(np.int64)
            want = np.array([I[j][q] if len(I[j]) else -1 for j, q in zip(kp, pick)])
            assert np.array_equal(o["instance"].cpu().numpy(), want)
        # K7 on every prompt (the rank kernel's tiles, its persistent walk over > 740 tiles at 2^22,
        # ragged tails): instance, slot and the batch lists vs the oracle
        wi, ws = O.route_and_batch(kp, inst, bstar, mode, cfg.route_seed, b)
        assert np.array_equal(o["instance"].cpu().numpy(), wi), f"batch {b}: instance differs"
        assert np.array_equal(o["slot"].cpu().numpy(), ws), f"batch {b}: slot differs"
        off, pr = O.buckets(wi, ws, len(inst))
        assert np.array_equal(o["bucket_offsets"][:len(inst) + 1].cpu().numpy(), off)
        assert np.array_equal(o["bucket_prompts"].cpu().numpy(), pr)
    r.close()
