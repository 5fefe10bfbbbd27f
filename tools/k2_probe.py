#!/usr/bin/env python
"""One K2 shape on one B200: N prompts vs an M-row cache (synth-v1, C5 recipe), routed --reps
times; prints K2's device time and TFLOP/s per rep (stage_ms[1]).  For ncu captures of a single
K2 launch at shapes the bench does not cover (e.g. the mid-N points of the C5 load curve)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=2048)
    ap.add_argument("--M", type=int, default=20_000_000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload

    cfg = CONFIGS["C5"]
    dev = torch.device("cuda", 0)
    w = Workload(cfg, device=dev, M=args.M)
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=args.N, max_rows_per_rank=args.M, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions([1.0 / len(cfg.grid)] * len(cfg.grid), cfg.instance_level, cfg.bstar, cfg.mode)
    for b in range(w.n_blocks()):
        r.load_cache(w.cache_block(b).contiguous())
    P = w.prompts(args.N)
    out = r.alloc_out(args.N)
    for i in range(args.reps):
        r.route(P, out)
        st = r.stats()
        ms = st["stage_ms"][1]
        print(json.dumps({"rep": i, "N": args.N, "M": args.M, "k2_ms": ms,
                          "tflops": 2.0 * args.N * args.M * cfg.d / (ms / 1e3) / 1e12}), flush=True)
    r.close()


if __name__ == "__main__":
    main()
