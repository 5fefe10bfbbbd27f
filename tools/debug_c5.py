"""Debug: Tier-B consistency of K2's (score, id) pairs at C5 sizes (no oracle).  For sampled prompts of
each batch, recompute the fp64 dot of the bf16-quantised prompt and cache rows of the returned ids."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import route as O  # noqa: E402  (test infrastructure)
from paper_2502_06798_b200 import pas  # noqa: E402
from synth import BLOCK, CONFIGS, Workload, c5_fractions  # noqa: E402

cfg = CONFIGS["C5"]
M = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.M
Ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 2048, 16384]
dev = torch.device("cuda", 0)
w = Workload(cfg, device=dev, M=M)
r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=max(Ns), max_rows_per_rank=M, device=0, seed=cfg.route_seed)
r.set_bands(cfg.grid, cfg.thresholds)
r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
for b in range(w.n_blocks()):
    r.load_cache(w.cache_block(b).contiguous())
rng = np.random.default_rng(5)
prev_h = prev_N = None
for bi, N in enumerate(Ns):
    P = w.prompts(N, batch=bi)
    idx = np.sort(rng.choice(N, min(N, 64), replace=False))
    F = c5_fractions(prev_h, prev_N, N)
    r.set_fractions(F, cfg.instance_level, cfg.bstar, cfg.mode)
    out = r.route(P)
    torch.cuda.synchronize()
    st = r.stats()
    prev_h, prev_N = st["h"], N
    k = cfg.topk
    gid = out["topk_id"].cpu().numpy().reshape(N, k)[idx]
    gsc = out["topk_score"].cpu().numpy().reshape(N, k)[idx]
    rows = w.rows_at(torch.from_numpy(np.maximum(gid, 0).reshape(-1))).cpu().numpy().reshape(len(idx), k, -1)
    Pq, _ = O.quantize(P[torch.from_numpy(idx)].cpu().numpy())
    Cq, _ = O.quantize(rows.reshape(-1, cfg.d))
    sb = np.einsum("pd,pkd->pk", Pq, Cq.reshape(len(idx), k, -1))
    err = np.abs(gsc - sb)
    print(f"N={N} R={st['k2_ranges']} T={st['k2_chunk_tiles']} CS={st['k2_chunk_steps']} max Tier-B err {err.max():.3g}",
          flush=True)
    for p, m in zip(*np.nonzero(err > 2e-5)):
        g = int(gid[p, m])
        blk = w.cache_block(g // BLOCK)[g % BLOCK].cpu().numpy()
        same = np.array_equal(blk, rows[p, m])
        print(f"  prompt {idx[p]} pos {m} gid {g} score {gsc[p, m]:.6f} tierB {sb[p, m]:.6f} rows_at==block {same}"
              f" row {gid[p].tolist()} scores {np.round(gsc[p], 5).tolist()}", flush=True)
r.close()
