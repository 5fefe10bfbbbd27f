"""C1 (64 prompts vs 1,000 rows) latency: device time per batch with the batch replayed as a CUDA graph
and enqueued far ahead of the device (no host gaps), and eagerly.  Also the ncu target for the C1
launch list.  Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(reps=int(os.environ.get("REPS", "400"))):
    import torch

    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C1"]
    N = int(os.environ.get("C1_N", cfg.N))   # batch size override (tiny low-load batches)
    dev = torch.device("cuda", 0)
    w = Workload(cfg, device=dev)
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=cfg.M, device=0, seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    r.load_cache(w.cache_rows(0, cfg.M).contiguous())
    emb = w.prompts(N).contiguous()
    out = r.alloc_out(N)
    res = {}
    for graph in (False, True):
        pas.pas_set_graph(r.ctx, graph)
        for _ in range(10):
            r.route(emb, out)
        torch.cuda.synchronize()
        # enqueue ahead: a long host-side sleep kernel is not available, so time many back-to-back
        # batches with one pair of events; the host enqueue rate bounds this from above
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(50_000_000)   # ~25 ms of GPU spin: the host queues the batches meanwhile
        e0.record()
        for _ in range(reps):
            r.route(emb, out)
        e1.record()
        torch.cuda.synchronize()
        res["graph" if graph else "eager"] = e0.elapsed_time(e1) / reps * 1e3
    res["unit"] = "us per batch (device, back to back)"
    print(json.dumps(res))
    r.close()


if __name__ == "__main__":
    main()
