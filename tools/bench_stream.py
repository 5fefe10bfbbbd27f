#!/usr/bin/env python
"""Streaming-kernel benchmark (K1, K3/K4, K6, K7 at sizes where the HBM roofline is
meaningful, >= 1 GB moved).

  * K1 (normalise + quantise) through pas_cache_load: M fp32 rows -> bf16 store (CUDA events).
  * K3+K4 (merge + optimal-K + H_K), K5, K6, K7 through pas_route_from_candidates on N synthetic
    prompts with S candidate lists each (no GEMM), stage times from pas_plan_stats.

Per-kernel GB/s come from the ncu launch list of this script (tools/gpu_stream.sh) divided into the
algorithmic bytes printed here.  Prints one JSON object.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def algorithmic_bytes(N, S, k, d, W, M):
    """Bytes each kernel must move at minimum (reads + writes), per launch."""
    return {
        "k_normalize (cache insert, fp32 in)": M * d * (4 + 2),
        "k_merge_select_thr": N * (S * k * 8 + k * 8 + 4 + 1 + 1),
        "k6_fused": N * (1 + 4 + 1),           # level byte read; K' (int32) + K7 class byte written (+ K7's tile counts)
        "k6_hist (fallback only)": N * (1 + 8 + 4),
        "k6_assign (fallback only)": N * (1 + 8 + 4 + 1),
        "k_cls_count (fallback only)": N * 1,
        "k_cls_rank": N * (1 + 4 + 4 + 4),     # class byte; instance, slot, bucket-list entry
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=1 << 26)
    ap.add_argument("--sources", type=int, default=1)
    ap.add_argument("--cache", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload

    cfg = CONFIGS["C4"]
    dev = torch.device("cuda", 0)
    N, S, k, d, M = args.prompts, args.sources, cfg.topk, cfg.d, args.cache
    out = {"N": N, "S": S, "k": k, "M_insert": M}

    # ---- K1 via cache insert -------------------------------------------------------------
    r = pas.Router(d=d, topk=k, max_batch=1, max_rows_per_rank=M, device=0)
    w = Workload(cfg, device=dev, M=M)
    rows = w.cache_rows(0, M).contiguous()
    times = []
    for _ in range(args.reps):
        pas.pas_cache_clear(r.ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r.load_cache(rows)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    t = min(times)
    out["cache_insert_ms"] = t
    out["cache_insert_GBps_incl_sync"] = M * d * 6 / (t / 1e3) / 1e9
    r.close()
    del rows

    # ---- K3..K7 via pas_route_from_candidates ----------------------------------------------
    g = torch.Generator(device=dev).manual_seed(7)
    sc = torch.rand(S, N, k, generator=g, device=dev) * 0.8 + 0.2
    sc, _ = torch.sort(sc, dim=-1, descending=True)
    gid = torch.randint(0, 1 << 30, (S, N, k), generator=g, device=dev, dtype=torch.int32)
    cand = torch.stack([sc.view(torch.int32), gid], dim=-1).contiguous()      # [S][N][k] x {f32, i32}
    del sc, gid
    rt = pas.Router(d=d, topk=k, max_batch=N, max_rows_per_rank=1, device=0)
    rt.set_bands(cfg.grid, cfg.thresholds)
    rt.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    rows1 = w.cache_rows(0, 1).contiguous()
    rt.load_cache(rows1)                      # non-empty cache (M_total > 0)
    o = rt.alloc_out(N)
    stage = None
    for _ in range(args.reps):
        pas.pas_route_from_candidates(rt.ctx, cand, S, N, o)
        st = rt.stats()
        if stage is None or st["stage_ms"][6] < stage[6]:
            stage = st["stage_ms"]
    out["stage_ms"] = dict(zip(["-", "-", "merge_optimalK", "plan", "redirect", "route_and_batch", "total"],
                               stage[:7]))
    out["h"] = st["h"]
    out["k6_fallback"] = st["k6_fallback"]
    out["algorithmic_bytes"] = algorithmic_bytes(N, S, k, d, len(cfg.instance_level), M)
    out["merge_GBps"] = out["algorithmic_bytes"]["k_merge_select_thr"] / (stage[2] / 1e3) / 1e9
    rt.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
