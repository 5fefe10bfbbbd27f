"""Times the f4 assignment solver (pas_solve_assignment) on one GPU against the paper's 100 ms
budget ("for a cluster with tens of GPUs, the solver time is within 100 ms") and the
oracle's NumPy enumeration on the host.  Prints one JSON line per (W, levels)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import controller as OC                      # noqa: E402  (baseline timing only)
from paper_2502_06798_b200 import pas                    # noqa: E402

GRIDS = {6: [0, 5, 10, 15, 20, 25], 10: list(range(0, 50, 5))}


def main():
    rows = []
    for nK, W in ((6, 16), (6, 32), (6, 64), (10, 16), (10, 32)):
        grid = GRIDS[nK]
        thr = [0.6 + 0.03 * i for i in range(nK - 1)]
        svc = [int(round((50 - K) * 100_000 * 1.9)) for K in grid]
        H = [1.0 / nK] * nK
        lam = 0.7 * W * max(OC.rates(svc, 4))
        r = pas.Router(d=768, topk=8, max_batch=64, max_rows_per_rank=16, device=0)
        r.set_bands(grid, thr)
        for _ in range(3):
            g = r.solve_assignment(W, lam, H, svc, 4)      # warm-up
        ms = []
        for _ in range(10):
            t0 = time.perf_counter()
            g = r.solve_assignment(W, lam, H, svc, 4)
            ms.append(((time.perf_counter() - t0) * 1e3, g["solve_ms"]))
        r.close()
        host = None
        if OC.n_compositions(W, nK) <= 12_000_000:
            t0 = time.perf_counter()
            o = OC.solve_vectorized(W, lam, H, svc, 4, grid, [0.006 * t for t in range(50)])
            host = time.perf_counter() - t0
            assert o["n"] == g["n"]
        row = dict(levels=nK, W=W, assignments=g["candidates"], n=g["n"], served=g["S"],
                   device_ms_median=sorted(m[1] for m in ms)[5], call_ms_median=sorted(m[0] for m in ms)[5],
                   oracle_numpy_s=host, host_cores=len(os.sched_getaffinity(0)))
        print(json.dumps(row))
        rows.append(row)


if __name__ == "__main__":
    main()
