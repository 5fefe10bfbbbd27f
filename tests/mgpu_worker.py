"""One rank of the multi-GPU check (tests/test_gpu_multi.py launches it with torchrun, one process per
GPU): the sharded cache on G real B200s through pas_route_batch with a real G-rank NCCL communicator,
in both collective modes, must give every output byte-identical to a world = 1 context on the same GPU
(shard invariance, R18 / R19), and a bad cache row owned by any rank must be rejected by all.
Writes <out_dir>/rank<r>.json."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out_dir = sys.argv[1]
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2502_06798_b200 import dist as pdist
    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload

    cfg = CONFIGS["C2"]
    N, M = 3001, 50_003
    w = Workload(cfg, device=dev, M=M)
    C_ = w.cache_rows(0, M).contiguous()
    batches = [w.prompts(N, batch=b).contiguous() for b in range(2)]
    batches[0][5] = 0.0                                  # an invalid prompt
    res = {"rank": rank, "world": world, "mismatches": [], "checked": 0}

    def mk(G, r, nid):
        ro = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=pdist.shard_rows(M, G, r),
                        device=local, rank=r, world=G, nccl_id=nid, seed=cfg.route_seed)
        ro.set_bands(cfg.grid, cfg.thresholds)
        ro.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
        return ro

    ref = mk(1, 0, None)
    ref.load_cache(C_)
    want = []
    for P in batches:
        o = ref.route(P)
        torch.cuda.synchronize()
        want.append(({k: v.cpu().numpy() for k, v in o.items()}, ref.stats()))
    ref.close()
    W = len(cfg.instance_level)
    for mode in (pas.PAS_COLL_FOLDED, pas.PAS_COLL_EXPLICIT):
        r = mk(world, rank, pdist.bootstrap_nccl_id(rank))
        bad = C_[:64].clone()
        bad[world - 1 + world * 3, 7] = float("nan")     # owned by the last rank
        try:
            r.load_cache(bad)
            res["mismatches"].append("bad row accepted")
        except pas.PasError as e:
            if e.status != -10:
                res["mismatches"].append(f"bad row: status {e.status}")
        r.load_cache(C_[:20_000])
        r.load_cache(C_[20_000:])
        pas.pas_set_collectives(r.ctx, mode)
        for b, P in enumerate(batches):
            o = r.route(P)
            torch.cuda.synchronize()
            st = r.stats()
            g = {k: v.cpu().numpy() for k, v in o.items()}
            ref_out, ref_st = want[b]
            for key in g:
                a, c = g[key], ref_out[key]
                if key == "bucket_offsets":
                    a, c = a[:W + 1], c[:W + 1]
                if not np.array_equal(a, c):
                    res["mismatches"].append(f"mode {mode} batch {b} {key}")
            for key in ("h", "f", "x", "D_Q", "n_invalid", "n_near_top1", "n_near_threshold", "bucket_count"):
                if st[key] != ref_st[key]:
                    res["mismatches"].append(f"mode {mode} batch {b} stats {key}")
            res["checked"] += 1
        r.close()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
