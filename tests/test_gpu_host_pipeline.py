"""Pipelined host-buffer routing (pas_route_batch_host_async; include/pas.h): a stream of batches
issued without waiting -- copies of one batch overlapping the routing of its neighbours through two
staging slots -- delivers, batch for batch, exactly what the synchronous pas_route_batch_host delivers
on an identically configured context (same Philox batch sequence, same LRU ticks)."""
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


def _router(pas, cfg, N, M, w):
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    r.load_cache(w.cache_rows(0, M).contiguous())
    return r


@pytest.mark.parametrize("name,N,M,sizes", [("C2", 1000, 5000, [1000, 1000, 333, 1000, 1, 777, 1000]),
                                            ("C1", 64, 1000, [64] * 6)])
def test_pipelined_host_routing_equals_sync(pas, name, N, M, sizes):
    cfg = CONFIGS[name]
    w = Workload(cfg, device=DEV, M=M)
    sync_r, pipe_r = _router(pas, cfg, N, M, w), _router(pas, cfg, N, M, w)
    ins = [w.prompts(n, batch=b).cpu().pin_memory() for b, n in enumerate(sizes)]
    want, got = [], []
    for x in ins:
        o = {k: v.pin_memory() for k, v in sync_r.alloc_out(x.shape[0], device="cpu").items()}
        pas.pas_route_batch_host(sync_r.ctx, x, o)
        want.append({k: v.clone() for k, v in o.items()})
    stream = torch.cuda.current_stream()
    pas.pas_route_host_begin(pipe_r.ctx, stream)
    for x in ins:   # every batch keeps its own pinned input and outputs alive until the end
        o = {k: v.pin_memory() for k, v in pipe_r.alloc_out(x.shape[0], device="cpu").items()}
        pas.pas_route_batch_host_async(pipe_r.ctx, x, o, stream)
        got.append(o)
    pas.pas_route_host_end(pipe_r.ctx, stream)
    torch.cuda.synchronize()
    W = len(cfg.instance_level)
    for b, (g, e) in enumerate(zip(got, want)):
        for k in e:
            a, c = g[k].numpy(), e[k].numpy()
            if k == "bucket_offsets":
                a, c = a[:W + 1], c[:W + 1]
            assert np.array_equal(a, c), f"batch {b} ({sizes[b]} prompts): {k} differs"
    sync_r.close()
    pipe_r.close()


def test_pipelined_host_routing_errors(pas):
    """The pipelined call validates like the synchronous one (no batch enqueued on an error)."""
    cfg = CONFIGS["C1"]
    w = Workload(cfg, device=DEV, M=1000)
    r = _router(pas, cfg, 64, 1000, w)
    big = torch.zeros(65, cfg.d).pin_memory()
    o = {k: v.pin_memory() for k, v in r.alloc_out(65, device="cpu").items()}
    with pytest.raises(pas.PasError):
        pas.pas_route_batch_host_async(r.ctx, big, o)          # N > max_batch
    x = w.prompts(64).cpu().pin_memory()
    o = {k: v.pin_memory() for k, v in r.alloc_out(64, device="cpu").items()}
    pas.pas_route_host_begin(r.ctx)
    pas.pas_route_batch_host_async(r.ctx, x, o)                # the context still routes
    pas.pas_route_host_end(r.ctx)
    torch.cuda.synchronize()
    assert o["K"].numpy().min() >= 0
    r.close()
