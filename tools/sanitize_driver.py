"""Workloads for compute-sanitizer (tools/sanitize.sh): small, every kernel family of the path.
  c1        C1 (64 x 1,000): K1, K2 (CTA-pair tile, static ranges + leash), the one-CTA latency path
  c1chain   C1 with PAS_SMALL_MAX=0: merge/select, K5, the six K6 kernels, K7 count/scan/rank
  c2        C2 (4,096 x 100,000): K2 dynamic schedule (parked lists, epoch-tagged chunk counters)
  dyn       3 batches, 2,200 x 90,017, k = 16, forced into 2-step chunks (the inter-CTA protocol)
  graph     C1 replayed 5x as a CUDA graph
  plan      a non-convex table (the one-CTA min-cost solver)
  lru       inserts with eviction (k_lru) + vanilla inserts
Each run ends with torch.cuda.synchronize() and prints "ok <name>"."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(name):
    import numpy as np
    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload
    dev = torch.device("cuda", 0)

    def router(cfg, N, M, topk=None):
        r = pas.Router(d=cfg.d, topk=topk or cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, seed=cfg.route_seed)
        r.set_bands(cfg.grid, cfg.thresholds)
        r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
        return r

    if name in ("c1", "c1chain", "graph"):
        cfg = CONFIGS["C1"]
        w = Workload(cfg, device=dev)
        r = router(cfg, cfg.N, cfg.M)
        r.load_cache(w.cache_rows(0, cfg.M).contiguous())
        P = w.prompts(cfg.N).contiguous()
        P[3] = 0.0
        if name == "graph":
            pas.pas_set_graph(r.ctx, True)
        out = r.alloc_out(cfg.N)
        for _ in range(5 if name == "graph" else 2):
            r.route(P, out)
        torch.cuda.synchronize()
        r.stats()
    elif name == "c2":
        cfg = CONFIGS["C2"]
        w = Workload(cfg, device=dev)
        r = router(cfg, cfg.N, cfg.M)
        for b in range(w.n_blocks()):
            r.load_cache(w.cache_block(b).contiguous())
        r.route(w.prompts(cfg.N).contiguous())
        torch.cuda.synchronize()
        r.stats()
    elif name == "dyn":
        cfg = CONFIGS["C2"]
        w = Workload(cfg, device=dev, M=90_017)
        r = router(cfg, 2200, 90_017, topk=16)
        r.load_cache(w.cache_rows(0, 90_017).contiguous())
        for b in range(3):
            r.route(w.prompts(2200, batch=b).contiguous())
        torch.cuda.synchronize()
        assert r.stats()["k2_chunk_tiles"] > 0
    elif name == "plan":
        cfg = CONFIGS["C2"]
        w = Workload(cfg, device=dev, M=5000)
        r = router(cfg, 2000, 5000)
        r.set_degradation(list(np.minimum(1.0, 0.09 * np.arange(50))))
        r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
        r.load_cache(w.cache_rows(0, 5000).contiguous())
        r.route(w.prompts(2000).contiguous())
        torch.cuda.synchronize()
        r.stats()
    elif name == "lru":
        cfg = CONFIGS["C2"]
        w = Workload(cfg, device=dev, M=3000)
        r = router(cfg, 1000, 1000)
        r.load_cache(w.cache_rows(0, 900).contiguous())
        out = r.route(w.prompts(1000).contiguous())
        r.insert(w.cache_rows(900, 1300).contiguous())
        r.insert_vanilla(w.prompts(1000).contiguous(), out["K_prime"])
        torch.cuda.synchronize()
    else:
        raise SystemExit(f"unknown workload {name}")
    torch.cuda.synchronize()
    print("ok", name, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "chain":
        os.environ["PAS_SMALL_MAX"] = "0"
    if sys.argv[1] == "c1chain":
        os.environ["PAS_SMALL_MAX"] = "0"
    if sys.argv[1] == "dyn":
        os.environ["PAS_K2_DYN_MIN_STEPS"] = "2"
        os.environ["PAS_K2_DYN_MB"] = "40"
    main(sys.argv[1])
