"""NVTX range per stage (tracing row; VERDICT r1 missing #7): every routed batch marks the
enqueue of its six stages K1..K7 as NVTX ranges, in order, each closed.  Checked with a test-only
NVTX injection library (tests/native/nvtx_probe.c, loaded via NVTX_INJECTION64_PATH as nsys would be)
that logs the ranges libpas starts and ends, on the latency path (N <= 1024) and the full chain."""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGES = ["pas K1 normalise", "pas K2 similarity + top-k", "pas K3/K4 merge + optimal-K", "pas K5 plan",
          "pas K6 redirect", "pas K7 route-and-batch"]

SCRIPT = textwrap.dedent("""
    import sys, torch
    sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
    from paper_2502_06798_b200 import pas
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C1"]
    dev = torch.device("cuda", 0)
    for N in (64, 3000):
        w = Workload(cfg, device=dev, M=2000)
        r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=2000, device=0, seed=cfg.route_seed)
        r.set_bands(cfg.grid, cfg.thresholds)
        r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
        r.load_cache(w.cache_rows(0, 2000).contiguous())
        out = r.alloc_out(N)
        for b in range(2):
            r.route(w.prompts(N, batch=b).contiguous(), out)
        torch.cuda.synchronize()
        r.close()
""")


def test_stage_ranges(tmp_path):
    from paper_2502_06798_b200 import build
    build.build()
    probe = str(tmp_path / "nvtx_probe.so")
    subprocess.run(["gcc", "-shared", "-fPIC", "-O2", "-o", probe, os.path.join(ROOT, "tests", "native", "nvtx_probe.c")],
                   check=True)
    log = tmp_path / "nvtx.log"
    env = dict(os.environ, NVTX_INJECTION64_PATH=probe, PAS_NVTX_LOG=str(log))
    script = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    starts, ends, order = {}, set(), []
    for line in log.read_text().splitlines():
        kind, rid, *name = line.split(" ", 2)
        if kind == "S":
            starts[rid] = name[0] if name else ""
            order.append(starts[rid])
        else:
            ends.add(rid)
    ours = [n for n in order if n.startswith("pas K")]
    assert ours == STAGES * 4, ours                      # 2 sizes x 2 batches, six stages each in order
    assert {rid for rid, n in starts.items() if n.startswith("pas K")} <= ends   # every range closed
