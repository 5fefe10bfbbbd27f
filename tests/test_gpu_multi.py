"""The world > 1 path on real GPUs: torchrun at G = 2, 4, 8 (as many as the box
has) through pas_route_batch with a real G-rank NCCL communicator, both collective modes, every output
byte-identical to G = 1 (R18, R19).  Self-skips on a box with fewer than two GPUs; the single-GPU
coverage of the same code is test_nccl_collective_path_single_rank (1-rank communicator) and the
virtual-shard tests."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_routing_on_g_gpus_matches_one(G, tmp_path):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < G:
        pytest.skip(f"needs {G} GPUs, this box has {n}")
    from paper_2502_06798_b200 import build
    build.build()
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + G), os.path.join(ROOT, "tests", "mgpu_worker.py"),
           str(tmp_path)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert f"nranks {G}" in p.stdout + p.stderr or "nRanks" in p.stdout + p.stderr
    for r in range(G):
        res = json.load(open(tmp_path / f"rank{r}.json"))
        assert res["world"] == G and res["checked"] == 4 and not res["mismatches"], res


def test_explicit_collectives_single_rank_communicator(tmp_path):
    """PAS_COLL_EXPLICIT through a 1-rank NCCL communicator on one GPU: slice merge (the whole batch),
    N2 all-reduce, N3 all-gather, unpack -- byte-identical to the direct path, LRU stamps included."""
    import numpy as np

    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C2"]
    N, M = 1000, 7000
    dev = torch.device("cuda", 0)
    w = Workload(cfg, device=dev, M=M)
    C_ = w.cache_rows(0, M).contiguous()
    P = w.prompts(N)
    P[3] = 0.0
    outs, stamps = [], []
    for mode in (None, pas.PAS_COLL_FOLDED, pas.PAS_COLL_EXPLICIT):
        nid = None if mode is None else pas.pas_nccl_unique_id()
        r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, world=1, nccl_id=nid,
                       seed=cfg.route_seed)
        r.set_bands(cfg.grid, cfg.thresholds)
        r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
        r.load_cache(C_)
        if mode is not None:
            pas.pas_set_collectives(r.ctx, mode)
        o = r.route(P)
        st_ = torch.empty(M, dtype=torch.int32, device=dev)
        pas.pas_cache_stamps(r.ctx, st_)
        torch.cuda.synchronize()
        outs.append(({k: v.cpu().numpy() for k, v in o.items()}, r.stats()))
        stamps.append(st_.cpu().numpy())
        r.close()
    W = len(cfg.instance_level)
    for (g, st), s_ in zip(outs[1:], stamps[1:]):
        for key in g:
            a, b = g[key], outs[0][0][key]
            if key == "bucket_offsets":
                a, b = a[:W + 1], b[:W + 1]
            assert np.array_equal(a, b), key
        for key in ("h", "f", "x", "D_Q", "n_invalid", "n_near_top1", "n_near_threshold"):
            assert st[key] == outs[0][1][key], key
        assert np.array_equal(s_, stamps[0])
