"""N2 folded vs explicit on one GPU.

(a) The merge work each form does per rank at G = 8: the folded form merges all N prompts' 8 candidate
    lists (pas_route_from_candidates, S = 8, N prompts); the explicit form merges a slice of N / 8
    (S = 8, N / 8 prompts).  Device time of the merge + optimal-K stage (stage_ms[2]).
(b) The explicit form's extra collective launches (N2 ncclAllReduce of H_K, N3 ncclAllGather of the
    slice results, one NCCL group) and the unpack kernel, through a 1-rank communicator: the
    pas_route_batch stage-2 time in PAS_COLL_EXPLICIT vs PAS_COLL_FOLDED.  With one rank NCCL moves no
    bytes over NVLink, so this is the launch / latency floor of the extra steps, not their G = 8 cost.
Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import statistics

    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C5"]
    dev = torch.device("cuda", 0)
    k, S = cfg.topk, 8
    out = {}
    g = torch.Generator(device=dev).manual_seed(3)
    for N in (16384, 131072):
        for n in (N, N // S):
            sc = torch.rand(S, n, k, generator=g, device=dev) * 0.8 + 0.2
            sc, _ = torch.sort(sc, dim=-1, descending=True)
            gid = torch.randint(0, 1 << 30, (S, n, k), generator=g, device=dev, dtype=torch.int32)
            cand = torch.stack([sc.view(torch.int32), gid], dim=-1).contiguous()
            r = pas.Router(d=cfg.d, topk=k, max_batch=n, max_rows_per_rank=1, device=0)
            r.set_bands(cfg.grid, cfg.thresholds)
            r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
            r.load_cache(Workload(cfg, device=dev, M=1).cache_rows(0, 1).contiguous())
            o = r.alloc_out(n)
            t = []
            for i in range(30):
                pas.pas_route_from_candidates(r.ctx, cand, S, n, o)
                t.append(r.stats()["stage_ms"][2])
            out[f"merge_S8_N{n}_of_{N}"] = statistics.median(t[5:])
            r.close()
    for name, M, N in (("C2", 100_000, 4096), ("C4-slice", 1_000_000, 65536)):
        w = Workload(CONFIGS["C2"], device=dev, M=M)
        C_ = w.cache_rows(0, M).contiguous()
        P = w.prompts(N)
        for mode in (pas.PAS_COLL_FOLDED, pas.PAS_COLL_EXPLICIT):
            r = pas.Router(d=768, topk=k, max_batch=N, max_rows_per_rank=M, device=0, world=1,
                           nccl_id=pas.pas_nccl_unique_id())
            r.set_bands(cfg.grid, cfg.thresholds)
            r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
            r.load_cache(C_)
            pas.pas_set_collectives(r.ctx, mode)
            o = r.alloc_out(N)
            t = []
            for i in range(30):
                r.route(P, o)
                t.append(r.stats()["stage_ms"][2])
            out[f"{name}_stage2_{'explicit' if mode else 'folded'}"] = statistics.median(t[5:])
            r.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
