"""The N > 1 path on CPU (world_size 2, gloo): the bootstrap and timing helpers bench.py uses, and
the sharding design itself -- every rank takes the exact top-k of its round-robin shard, the [N x k]
candidate lists are all-gathered (here over gloo, on the GPU over NCCL inside libpas), and the
merge of the gathered lists equals the single-GPU top-k (the oracle computes each rank's part)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_06798_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import route as O
        from synth import CONFIGS, Workload
        # (1) bootstrap: rank 0's id reaches every rank
        nid = pdist.bootstrap_nccl_id(rank, make_id=lambda: bytes(range(128)))
        assert nid == bytes(range(128))
        # (2) max over ranks
        assert pdist.max_over_ranks(float(rank + 1)) == float(world)
        # (3) sharded exact top-k + all-gather + merge == the whole-cache top-k
        cfg = CONFIGS["C1"]
        M, N, k = 997, 24, 8
        w = Workload(cfg, M=M)
        C = w.cache_rows(0, M).numpy()
        P = w.prompts(N).numpy()
        mine = np.arange(rank, M, world)                         # gid g on rank g % world
        assert len(mine) == pdist.shard_rows(M, world, rank)
        ids, sc = O.topk_sorted(O.similarity_A(P, C[mine]), mine, k)
        pack = torch.from_numpy(np.concatenate([sc, ids.astype(np.float64)], axis=1))
        gathered = [torch.empty_like(pack) for _ in range(world)]
        dist.all_gather(gathered, pack)
        mi, ms = gathered[0][:, k:].numpy().astype(np.int64), gathered[0][:, :k].numpy()
        for g in gathered[1:]:
            mi, ms = O.merge_topk(mi, ms, g[:, k:].numpy().astype(np.int64), g[:, :k].numpy(), k)
        wi, ws = O.topk_sorted(O.similarity_A(P, C), np.arange(M), k)
        assert np.array_equal(mi, wi) and np.array_equal(ms, ws)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


def test_shard_arithmetic():
    for M in (0, 1, 7, 100, 101):
        for G in (1, 2, 3, 8):
            rows = [pdist.shard_rows(M, G, r) for r in range(G)]
            assert sum(rows) == M
            gids = sorted(pdist.local_to_global(l, G, r) for r in range(G) for l in range(rows[r]))
            assert gids == list(range(M))


def _worker_explicit(rank, world, port, q):
    """The explicit-N2 exchange (pas_set_collectives(PAS_COLL_EXPLICIT)) over gloo: N1
    all-gather of every rank's shard top-k, a merge of this rank's slice of ceil(N / G) prompts only, N2
    all-reduce of the slice H_K, N3 all-gather of the slice results padded to ceil(N / G) rows (the
    in-place layout libpas uses), unpacked to the first N rows -- equal to the folded form (every rank
    merging all N) and to the single-GPU result."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import route as O
        from synth import CONFIGS, Workload
        cfg = CONFIGS["C1"]
        M, N, k = 613, 25, 8                                   # N not a multiple of G
        w = Workload(cfg, M=M)
        C = w.cache_rows(0, M).numpy()
        P = w.prompts(N).numpy()
        mine = np.arange(rank, M, world)
        ids, sc = O.topk_sorted(O.similarity_A(P, C[mine]), mine, k)
        pack = torch.from_numpy(np.concatenate([sc, ids.astype(np.float64)], axis=1))
        gathered = [torch.empty_like(pack) for _ in range(world)]
        dist.all_gather(gathered, pack)                        # N1
        Ns = (N + world - 1) // world
        lo, hi = rank * Ns, min(N, (rank + 1) * Ns)
        mi, ms = gathered[0][lo:hi, k:].numpy().astype(np.int64), gathered[0][lo:hi, :k].numpy()
        for g in gathered[1:]:                                 # the slice merge
            mi, ms = O.merge_topk(mi, ms, g[lo:hi, k:].numpy().astype(np.int64), g[lo:hi, :k].numpy(), k)
        lev = O.optimal_k_level(ms[:, 0], cfg.thresholds, np.ones(hi - lo, bool)) if hi > lo else np.zeros(0, int)
        h = torch.from_numpy(O.histogram(lev, len(cfg.grid)))
        dist.all_reduce(h)                                     # N2
        rec = np.zeros((Ns, 2 * k + 1))                        # slice results, padded to Ns rows
        rec[:hi - lo, :k], rec[:hi - lo, k:2 * k], rec[:hi - lo, 2 * k] = ms, mi, lev
        parts = [torch.empty(Ns, 2 * k + 1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(rec))          # N3
        allr = torch.cat(parts).numpy()[:N]
        wi, ws = O.topk_sorted(O.similarity_A(P, C), np.arange(M), k)
        wl = O.optimal_k_level(ws[:, 0], cfg.thresholds, np.ones(N, bool))
        assert np.array_equal(allr[:, k:2 * k].astype(np.int64), wi) and np.array_equal(allr[:, :k], ws)
        assert np.array_equal(allr[:, 2 * k].astype(np.int64), wl)
        assert h.numpy().tolist() == O.histogram(wl, len(cfg.grid)).tolist()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_explicit_n2_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_explicit, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res
