#!/usr/bin/env python
"""bench.py -- prompts routed per second through libpas on 1..8 B200s (BASELINE.json metric).

One step = one pas_route_batch of the whole hot path (normalise, similarity GEMM + top-k, merge
(+ NCCL all-gather for G > 1), optimal-K + H_K, Eq. 1 plan, redirection, route-and-batch) on one
batch of synthetic prompts resident in HBM.  Default workload: C4 (BASELINE configs[3]): 65,536
prompts vs a 10M-entry cache, the cache row-sharded over the G = --gpus router GPUs (strong
scaling: total work is fixed).  Launch for G > 1:
    python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus G
Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle (oracle/) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prompts scheduled/s vs cache size at 1/2/4/8 B200; % of TC/HBM peak"
UNIT = "prompts/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libpas", choices=["libpas", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--prompts", type=int, default=None, help="override N")
    ap.add_argument("--cache", type=int, default=None, help="override M")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dispatcher", action="store_true",
                    help="route-and-batch through the f3 stateful dispatcher (queues carried across steps)")
    ap.add_argument("--forecast", type=int, default=0, metavar="W",
                    help="the f1 forecast-driven mode: an Optimal-K Predictor window of W prompts, the plan "
                         "rebuilt every batch, i.i.d. Philox K' (0: the exact per-batch plan)")
    ap.add_argument("--force-collective", action="store_true",
                    help="use the NCCL all-gather path even with one rank (transport self-test)")
    ap.add_argument("--graph", action="store_true",
                    help="replay each batch as a captured CUDA graph (pas_set_graph; stage times then total only)")
    ap.add_argument("--collectives", default="folded", choices=["folded", "explicit"],
                    help="G > 1: folded (N1 all-gather, every rank merges all N) or explicit (N1 + slice merge + "
                         "N2 all-reduce of H_K + N3 all-gather), pas_set_collectives")
    return ap.parse_args()


# ----------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms; only the samples taken between
    begin() and stop() count (nvidia-smi takes ~1 s to start, longer than a short timed region)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None
        self.first = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def begin(self):
        """Wait (<= 5 s) until nvidia-smi is producing samples, then open the counted window."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < 5.0:
            time.sleep(0.02)
        self.first = len(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        last = len(self.rows)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.rows = self.rows[self.first:last]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[2]))
            except ValueError:
                pass
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w": statistics.median(pw) if pw else None, "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


def select_peak(peaks: dict, clk: dict | None):
    """Which measured peak bounds K2 (MEASURED_PEAKS.json): the sustained figure (cuBLAS 8192^3 back to
    back under the 1 kW cap) when this run ran power- or thermally-limited -- the long steps (C4, C5)
    -- else the burst figure (short steps at full clock, e.g. C2; also the conservative choice without
    clock samples).  Returns (TFLOP/s, description)."""
    reasons = set((clk or {}).get("reasons") or [])
    capped = bool(reasons & {"sw_power_cap", "hw_power_brake_slowdown", "hw_slowdown", "sw_thermal_slowdown",
                             "hw_thermal_slowdown"})
    if not capped and clk and clk.get("sm_mhz") and clk.get("sm_max_mhz"):
        capped = clk["sm_mhz"] < 0.97 * clk["sm_max_mhz"]
    sustained = peaks.get("bf16_tflops_sustained")
    if capped and sustained:
        return float(sustained), "bf16 sustained (power-capped run)"
    return float(peaks["bf16_tflops"]), "bf16 burst (full-clock run)"


def profiled_traffic(config: str, G: int):
    """dram read+write bytes per K2 launch from the committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "k2_traffic.json")) as fh:
            t = json.load(fh)
        return t.get(f"{config}_G{G}")
    except Exception:
        return None


# ----------------------------------------------------------------------------------------------
ORACLE_PROMPTS = 32          # the one oracle sampling definition of both legs (cpu_baseline and --impl reference)
ORACLE_ROWS = 1 << 20


class OracleSample:
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload: ORACLE_PROMPTS
    prompts (a different slice each step) against the first ORACLE_ROWS cache rows -- Tier-A fp64
    similarity, full-sort top-k, optimal-K (O1..O3) -- plus the downstream O4..O10 on all N prompts.
    The similarity seconds are scaled to the full cache (linear in M) and per prompt; the downstream is
    per prompt of the whole batch.  Used unchanged by the cpu_baseline leg and the reference arm, so the
    two report the same quantity."""

    def __init__(self, cfg, w, N, M, P_host):
        import numpy as np

        from synth import BLOCK
        self.cfg, self.N, self.M, self.P = cfg, N, M, P_host
        self.n_rows = min(ORACLE_ROWS, M)
        self.n_p = min(ORACLE_PROMPTS, N)
        self.chunks = []
        b = 0
        while b * BLOCK < self.n_rows:
            self.chunks.append((b * BLOCK, w.cache_block(b)[: self.n_rows - b * BLOCK].cpu().numpy()))
            b += 1
        self.levels = np.random.default_rng(0).integers(0, len(cfg.grid), N)
        self.i = 0

    def step(self):
        """One bounded sample; returns (seconds per prompt, similarity s, downstream s)."""
        import numpy as np

        from oracle import route as O
        cfg = self.cfg
        idx = (np.arange(self.n_p) + self.i * self.n_p) % self.N
        self.i += 1
        t0 = time.perf_counter()
        ids, sc, valid = O.topk_streaming(self.P[idx], iter(self.chunks), cfg.topk)
        lev = O.optimal_k_level(sc[:, 0], cfg.thresholds, valid)
        t_sim = time.perf_counter() - t0
        levels = self.levels.copy()
        levels[idx] = lev
        setup = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=cfg.F, instance_level=cfg.instance_level,
                        bstar=cfg.bstar, mode=cfg.mode, topk=cfg.topk, seed=cfg.route_seed)
        t1 = time.perf_counter()
        O.downstream(levels, setup)
        t_down = time.perf_counter() - t1
        return t_sim / self.n_p * (self.M / self.n_rows) + t_down / self.N, t_sim, t_down

    def describe(self, t_sim, t_down):
        return (f"per step: {self.n_p} prompts x first {self.n_rows:,} of {self.M:,} cache rows (fp64 Tier-A "
                f"similarity, full-sort top-{self.cfg.topk}, optimal-K; {t_sim:.1f} s, scaled x{self.M / self.n_rows:.2f} "
                f"to the full cache) + O4..O10 on all {self.N:,} prompts ({t_down:.1f} s)")


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return len(os.sched_getaffinity(0))


def cpu_baseline(cfg, w, N, M, P_host, steps: int = 2):
    """The cpu_baseline leg: OracleSample, `steps` samples on rank 0, reported as prompts/s."""
    smp = OracleSample(cfg, w, N, M, P_host)
    per = [smp.step() for _ in range(steps)]
    per_prompt = sum(p[0] for p in per) / len(per)
    return {"value": 1.0 / per_prompt, "unit": UNIT, "cores": _threads(), "kind": "oracle",
            "sample": smp.describe(per[-1][1], per[-1][2]) + f"; mean of {steps} steps",
            "seconds": {"similarity": round(sum(p[1] for p in per) / len(per), 3),
                        "downstream": round(sum(p[2] for p in per) / len(per), 3)},
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ----------------------------------------------------------------------------------------------
def main():
    args = parse()
    import torch

    from synth import BLOCK, CONFIGS, Workload

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    N = args.prompts or cfg.N
    M = args.cache or cfg.M

    if args.impl == "reference":
        return reference_arm(args, cfg, N, M, rank, world)

    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1 or args.force_collective:
        os.environ.setdefault("NCCL_DEBUG", "INFO")           # the communicator's init log (nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    from paper_2502_06798_b200 import dist as pdist
    from paper_2502_06798_b200 import pas

    nccl_id = pdist.bootstrap_nccl_id(rank) if (world > 1 or args.force_collective) else None
    G = world
    M_local = max(1, pdist.shard_rows(M, G, rank))
    router = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=M_local, device=local,
                        rank=rank, world=G, nccl_id=nccl_id, seed=cfg.route_seed)
    router.set_bands(cfg.grid, cfg.thresholds)
    router.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    if nccl_id is not None:
        pas.pas_set_collectives(router.ctx, pas.PAS_COLL_EXPLICIT if args.collectives == "explicit"
                                else pas.PAS_COLL_FOLDED)
    gap_us = 0
    if args.graph:
        pas.pas_set_graph(router.ctx, True)
    if args.forecast:
        router.set_forecast(args.forecast, 1)
    if args.dispatcher:
        # SPEC S:75 service model per instance at b*: (T - K) x 100 ms x (1 + 0.3 (b* - 1)); batches
        # arrive at 90 % of the instances' capacity, so queues stay short but non-empty
        svc = [int(round((50 - cfg.grid[lv]) * 100_000 * (1 + 0.3 * (cfg.bstar - 1)))) for lv in cfg.instance_level]
        router.set_dispatcher(svc, 250_000)
        cap = sum(cfg.bstar / (s_ * 1e-6) for s_ in svc)
        gap_us = int(N / (0.9 * cap) * 1e6)
    clock = [0]

    def route_step():
        if args.dispatcher:
            clock[0] += gap_us
            router.set_clock(clock[0])
        router.route(P, out)

    w = Workload(cfg, device=dev, M=M)
    t_load = time.perf_counter()
    for b in range(w.n_blocks()):
        router.load_cache(w.cache_block(b).contiguous())
    torch.cuda.synchronize()
    t_load = time.perf_counter() - t_load
    P = w.prompts(N)
    out = router.alloc_out(N)
    stream = torch.cuda.current_stream()
    cache_bytes = M_local * cfg.d * 2
    l2_note = ("inputs larger than L2: the %.1f GB cache shard is streamed every step" % (cache_bytes / 1e9)
               if cache_bytes > 200e6 else "L2 flushed between steps (256 MB write)")
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if cache_bytes <= 200e6 else None

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        route_step()
    barrier()

    # per-step events on the routing stream and the library's stage-timing ring: nothing in the timed
    # loop waits on the device (no stats() / host sync between steps)
    ring = min(args.steps, 4096)                 # PAS_MAX_RING: stage times of the last <= 4,096 steps
    pas.pas_stage_ring(router.ctx, ring)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.begin()
    launches = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    s0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    s1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    ev0.record(stream)
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)
        s0[i].record(stream)
        route_step()
        s1[i].record(stream)
        launches += pas.pas_last_launch_count(router.ctx)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(s0, s1)]
    stages = pas.pas_stage_ring_read(router.ctx, ring)
    pas.pas_stage_ring(router.ctx, 0)
    stage_sum = [sum(r[i] for r in stages) for i in range(7)]
    n_st = max(1, len(stages))        # 0 in graph mode: a replayed batch is timed as a whole
    total_ms = sum(step_ms) if flush is not None else ev0.elapsed_time(ev1)
    total_ms = max_over_ranks(total_ms, dist, dev, torch)
    k2_ms = max_over_ranks(stage_sum[1] / n_st, dist, dev, torch) if stages else None
    value = N * args.steps / (total_ms / 1e3)
    q = statistics.quantiles(step_ms, n=10) if len(step_ms) >= 2 else [step_ms[0]] * 9
    step_stats = {"median": statistics.median(step_ms), "p10": q[0], "p90": q[-1], "min": min(step_ms),
                  "max": max(step_ms), "note": "device time per pas_route_batch (CUDA events, this rank)"}

    # ---- e2e through the host-buffer entry point (H2D of the prompts, D2H of every output)
    e2e = None
    if not args.no_e2e:
        Ph = P.cpu().pin_memory()
        host_out = router.alloc_out(N, device="cpu")
        for k_, v in host_out.items():
            host_out[k_] = v.pin_memory()
        bi = Ph.numel() * Ph.element_size()
        bo = sum(v.numel() * v.element_size() for k_, v in host_out.items() if k_ != "bucket_offsets") \
            + (router.W + 1) * 4
        pas.pas_route_batch_host(router.ctx, Ph, host_out)
        barrier()
        # (1) the synchronous call: every step copies in, routes, copies out and waits
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            pas.pas_route_batch_host(router.ctx, Ph, host_out)
        e1.record(stream)
        barrier()
        e_sync_ms = max_over_ranks(e0.elapsed_time(e1), dist, dev, torch)
        # (2) the pipelined call (a serving loop): the same copies every step, each batch's copies
        # overlapping its neighbours' routing; two input / output buffer pairs alternate so a step
        # never overwrites host memory a batch in flight still uses
        Ph2 = [Ph, P.cpu().pin_memory()]
        outs = [host_out, {k_: v.clone().pin_memory() for k_, v in host_out.items()}]
        barrier()
        e0.record(stream)
        pas.pas_route_host_begin(router.ctx, stream)
        for i in range(args.steps):
            pas.pas_route_batch_host_async(router.ctx, Ph2[i & 1], outs[i & 1], stream)
        pas.pas_route_host_end(router.ctx, stream)
        e1.record(stream)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1), dist, dev, torch)
        e2e = {"value": N * args.steps / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo,
               "api": "pas_route_batch_host_async (pinned host buffers, two batches in flight; every step's "
                      "H2D and D2H inside the timed region)",
               "value_sync": N * args.steps / (e_sync_ms / 1e3),
               "api_sync": "pas_route_batch_host (copy in, route, copy out, wait: one batch at a time)"}

    peaks, peak_src = measured_peaks()
    flops = 2.0 * N * M_local * cfg.d
    achieved = flops / (k2_ms / 1e3) / 1e12 if k2_ms else None
    peak, peak_kind = select_peak(peaks, clk)
    traffic = profiled_traffic(args.config, G)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (synth-v1: clustered CLIP-shaped embeddings, d=768, seeded)",
        "config": {"workload": f"{args.config}: {N:,} prompts vs {M:,}-entry cache ({cfg.note})", "N": N, "M": M,
                   "G": G, "M_per_gpu": M_local, "d": cfg.d, "topk": cfg.topk, "levels": len(cfg.grid),
                   "instances": len(cfg.instance_level), "mode": "uniform" if cfg.mode else "greedy",
                   "bstar": cfg.bstar, "dispatcher": "stateful (f3)" if args.dispatcher else "stateless (R13)",
                   "plan": f"forecast (f1, window {args.forecast})" if args.forecast else "exact per batch",
                   "launch": "CUDA graph replay" if args.graph else "eager",
                   "parallelism": f"cache row-sharded x{G}" + ((" + NCCL all-gather" if args.collectives == "folded" else
                                                                   " + NCCL all-gather / all-reduce H_K / all-gather (explicit N2)")
                                                                  if G > 1 else ""),
                   "l2": l2_note},
        "roofline": {"kernel": "k_simtopk (K2: tcgen05 similarity GEMM + fused top-k)", "bound": "tensor",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if achieved else None,
                     "traffic": traffic, "peak_source": f"{peak_kind}, {peak_src}",
                     "algorithmic": f"2*N*M_per_gpu*d = {flops:.4g} flop per launch / mean K2 event time "
                                    + (f"{k2_ms:.3f} ms" if k2_ms else "n/a (graph replay: no per-stage events)")},
        "step_ms": step_stats,
        "value_median": N / (step_stats["median"] / 1e3),
        "stages_ms": {n: round(stage_sum[i] / n_st, 4) for i, n in enumerate(
            ["normalise", "similarity_topk", "merge_collective_optimalK", "plan", "redirect", "route_and_batch",
             "total"])},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "setup": {"cache_load_s": round(t_load, 2)},
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, w, N, M, P.cpu().numpy())
    if rank == 0:
        print(json.dumps(line), flush=True)
    router.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def max_over_ranks(x, dist, dev, torch):
    from paper_2502_06798_b200 import dist as pdist
    return pdist.max_over_ranks(x, dev) if dist else x


def reference_arm(args, cfg, N, M, rank, world):
    """The CPU oracle as it stands, timed on this host's cores: each step is one OracleSample (the same
    bounded sample definition as the cpu_baseline leg), W warm-up steps, then K timed steps."""
    if rank != 0:
        return
    import torch

    from synth import Workload

    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    w = Workload(cfg, device=dev, M=M)
    smp = OracleSample(cfg, w, N, M, w.prompts(N).cpu().numpy())
    for _ in range(args.warmup):
        smp.step()
    per = [smp.step() for _ in range(args.steps)]
    per_prompt = sum(p[0] for p in per) / len(per)
    value = 1.0 / per_prompt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_prompt * N * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth-v1)",
            "config": {"workload": f"{args.config}: {N:,} prompts vs {M:,}-entry cache ({cfg.note})", "N": N,
                       "M": M},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": _threads(), "kind": "oracle",
                             "sample": smp.describe(per[-1][1], per[-1][2]) + f"; mean of {args.steps} steps",
                             "seconds": {"similarity": round(sum(p[1] for p in per) / len(per), 3),
                                         "downstream": round(sum(p[2] for p in per) / len(per), 3)},
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
