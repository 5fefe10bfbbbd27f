#!/usr/bin/env python
"""Sweeps behind BASELINE's metric "prompts scheduled/s vs cache size" on one B200.

  --kind cache   N = 16,384 prompts vs M in {1k, 100k, 1M, 10M, 50M} (SURVEY 8(d) "sweep" row)
  --kind shard   C4 (65,536 prompts) against one rank's share of the 10M cache at G = 1, 2, 4, 8: the K2
                 work of one router GPU under row sharding, measured on one B200 (the NCCL all-gather of
                 8 N k G bytes and the G-way merge are NOT included: a per-rank share, not a multi-GPU run)
  --kind load    C5: N = 256 .. 131,072 (x2) vs a 50M-entry cache, F(K) recomputed before every
                 batch from the previous batch's H_K (F_b = (1 - l_b) h_{b-1} / N_{b-1} + l_b e_{K=25},
                 l_b = log2(N_b / 256) / 9), the pas_set_fractions call timed
                 with the batch.

Device time with CUDA events per batch (median of --steps), stage split from pas_plan_stats.  One
JSON object per line.  The cache is generated on the GPU block by block (synth-v1).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", choices=["cache", "load", "shard"], default="cache")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--max-cache", type=int, default=50_000_000)
    ap.add_argument("--ns", type=str, default="", help="comma-separated N values for --kind load")
    ap.add_argument("--prewarm-s", type=float, default=0.0,
                    help="route the largest batch for this many seconds first (steady clocks / power)")
    args = ap.parse_args()
    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload, c5_fractions

    dev = torch.device("cuda", 0)
    if args.kind in ("cache", "shard"):
        cfg = CONFIGS["C4"]
        N = 16384
        sizes = [m for m in (1_000, 100_000, 1_000_000, 10_000_000, 50_000_000) if m <= args.max_cache]
        if args.kind == "shard":      # one rank's share of C4 at G = 1, 2, 4, 8 (round-robin rows)
            N = cfg.N
            sizes = [(cfg.M + g - 1) // g for g in (1, 2, 4, 8)]
        for M in sizes:
            w = Workload(cfg, device=dev, M=M)
            r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=M, device=0, seed=cfg.route_seed)
            r.set_bands(cfg.grid, cfg.thresholds)
            r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
            t0 = time.perf_counter()
            for b in range(w.n_blocks()):
                r.load_cache(w.cache_block(b).contiguous())
            load_s = time.perf_counter() - t0
            P = w.prompts(N)
            out = r.alloc_out(N)
            ms = []
            k2 = []
            for i in range(args.warmup + args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r.route(P, out)
                e1.record()
                e1.synchronize()
                if i >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
                    k2.append(r.stats()["stage_ms"][1])
            med = statistics.median(ms)
            tf = 2.0 * N * M * cfg.d / (statistics.median(k2) / 1e3) / 1e12
            print(json.dumps({"kind": args.kind, "N": N, "M": M, "prompts_per_s": N / (med / 1e3), "ms_median": med,
                              "ms_p10": sorted(ms)[max(0, len(ms) // 10)], "ms_p90": sorted(ms)[min(len(ms) - 1, (9 * len(ms)) // 10)],
                              "k2_tflops": tf, "cache_load_s": round(load_s, 2)}), flush=True)
            r.close()
            del w, P, out
            torch.cuda.empty_cache()
    else:
        cfg = CONFIGS["C5"]
        M = min(cfg.M, args.max_cache)
        Ns = [int(x) for x in args.ns.split(",")] if args.ns else [256 << i for i in range(10)]
        w = Workload(cfg, device=dev, M=M)
        r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=Ns[-1], max_rows_per_rank=M, device=0, seed=cfg.route_seed)
        r.set_bands(cfg.grid, cfg.thresholds)
        nK = len(cfg.grid)
        F = [1.0 / nK] * nK
        r.set_fractions(F, cfg.instance_level, cfg.bstar, cfg.mode)
        t0 = time.perf_counter()
        for b in range(w.n_blocks()):
            r.load_cache(w.cache_block(b).contiguous())
        load_s = time.perf_counter() - t0
        Pall = w.prompts(Ns[-1])
        if args.prewarm_s > 0:          # untimed: reach the steady power / clock state first
            out = r.alloc_out(Ns[-1])
            t_end = time.perf_counter() + args.prewarm_s
            while time.perf_counter() < t_end:
                r.route(Pall, out)
                torch.cuda.synchronize()
        prev_h, prev_N = None, None
        for N in Ns:
            P = Pall[:N].contiguous()
            out = r.alloc_out(N)
            ms = []
            for i in range(args.warmup + args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if prev_h is not None:          # controller update from the previous batch's H_K
                    F = c5_fractions(prev_h, prev_N, N)
                    r.set_fractions(F, cfg.instance_level, cfg.bstar, cfg.mode)
                r.route(P, out)
                e1.record()
                st = r.stats()                  # syncs; H_K of this batch feeds the next F
                prev_h, prev_N = st["h"], N
                if i >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
            med = statistics.median(ms)
            print(json.dumps({"kind": "load", "N": N, "M": M, "prompts_per_s": N / (med / 1e3), "ms_median": med,
                              "stage_ms": st["stage_ms"][:7], "D_Q": st["D_Q"], "F": [round(f, 4) for f in F],
                              "h": st["h"], "cache_load_s": round(load_s, 2)}), flush=True)
        r.close()


if __name__ == "__main__":
    main()
