"""Seeded synthetic workloads ("synth-v1") shared by the tests, bench.py and the oracle legs.

This module generates INPUTS only and holds none of the method's arithmetic (no
similarity, top-k, thresholds, planning, sampling or batching).  The same arrays
are handed to the CUDA path (via the C-ABI) and to the CPU oracle (by D2H copy).

Recipe (after SURVEY.md 8(d)):
* d = 768 (CLIP ViT-L/14 text width).  Anisotropy: a unit vector mu with weight
  a = 0.5 (a^2 = 0.25) so unrelated prompts have cosine ~0.25.
* C = clamp(M / 1000, 16, 50000) clusters.  centroid_j = unit(a mu + sqrt(1-a^2) unit(g_j)),
  spread tau_j ~ U[0.25, 0.90], popularity w_j ~ (j+1)^-1.1 (Zipf).
* cache row: j ~ w; row = unit(centroid_j + tau_j n / sqrt(d)) * scale, scale ~ U[0.5, 2]
  (embeddings arrive un-normalised; the method normalises them itself).
* prompt mix (novel, dup, cluster), default (0.15, 0.15, 0.70):
    novel   -- a fresh centroid never in the cache, tau = 0.5  (s1 ~ 0.3, K = 0)
    dup     -- unit(row_g + 0.12 n / sqrt(d)), g ~ U[0, M)  (planted near-duplicate, s1 ~ 0.99)
    cluster -- j ~ w, drawn like a cache row.
* Cache rows are produced in blocks of BLOCK rows; block b is seeded by (seed, b), so a
  chunk's contents do not depend on how the caller chunks the load.

Configurations C1..C5 follow BASELINE.json ``configs``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

D_MODEL = 768
BLOCK = 1 << 16
ANISO_A = 0.5
GRID6 = [0, 5, 10, 15, 20, 25]
BANDS6 = [0.65, 0.72, 0.79, 0.86, 0.93]
GRID10 = [0, 5, 10, 15, 20, 25, 30, 35, 40, 45]
BANDS10 = [0.65 + 0.035 * (m - 1) for m in range(1, 10)]     # DESIGN.md R8
ROUTE_SEED = 0x5EED2502


@dataclass
class Config:
    name: str
    N: int
    M: int
    grid: list
    thresholds: list
    instance_level: list           # level index of each serving instance
    F: list
    bstar: int = 4
    mode: int = 0                  # 0 greedy, 1 uniform
    topk: int = 8
    mix: tuple = (0.15, 0.15, 0.70)
    gen_seed: int = 1000
    route_seed: int = ROUTE_SEED
    world: int = 1
    d: int = D_MODEL
    note: str = ""


def _dirichlet_F(n: int, seed: int) -> list:
    rng = np.random.default_rng(seed)
    v = rng.dirichlet(np.ones(n))
    v = np.round(v, 6)
    v[-1] = 1.0 - float(np.sum(v[:-1]))
    return [float(x) for x in v]


CONFIGS = {
    "C1": Config("C1", N=64, M=1000, grid=GRID6, thresholds=BANDS6,
                 instance_level=[0, 2, 4, 5], F=[0.25, 0.0, 0.25, 0.0, 0.25, 0.25],
                 bstar=4, mode=0, gen_seed=1001,
                 note="64 prompts vs 1,000-entry cache, 4 instances"),
    "C2": Config("C2", N=4096, M=100_000, grid=GRID6, thresholds=BANDS6,
                 instance_level=[0, 1, 2, 3, 4, 5, 5, 5], F=[0.05, 0.05, 0.10, 0.10, 0.20, 0.50],
                 bstar=4, mix=(0.60, 0.05, 0.35), gen_seed=1002,
                 note="skewed H_K vs F_K (heavy redirection)"),
    "C3": Config("C3", N=16384, M=1_000_000, grid=GRID10, thresholds=BANDS10,
                 instance_level=list(range(10)), F=_dirichlet_F(10, 1003),
                 bstar=4, gen_seed=1003, note="10 K levels, top-k 8"),
    "C4": Config("C4", N=65536, M=10_000_000, grid=GRID6, thresholds=BANDS6,
                 instance_level=[0, 0, 1, 2, 3, 4, 5, 5], F=[0.10, 0.10, 0.15, 0.15, 0.20, 0.30],
                 bstar=4, gen_seed=1004, note="10M cache, sharded over G router GPUs"),
    "C5": Config("C5", N=131072, M=50_000_000, grid=GRID6, thresholds=BANDS6,
                 instance_level=[0, 0, 1, 2, 3, 4, 5, 5], F=[1.0 / 6] * 5 + [1.0 - 5.0 / 6],
                 bstar=4, gen_seed=1005, note="load sweep 256..131072, F recomputed per batch"),
}


def c5_fractions(prev_h, prev_N: int, N: int) -> list:
    """The C5 controller input for a batch of N prompts ("only faster
    K = 25 variants running at peak loads"): F_b = (1 - l_b) h_{b-1} / N_{b-1} + l_b e_{K=25},
    l_b = log2(N_b / 256) / 9, renormalised; uniform before the first batch.  A workload recipe
    (what the controller hands the path), not method arithmetic."""
    if prev_h is None:
        n = len(CONFIGS["C5"].grid)
        return [1.0 / n] * n
    ell = math.log2(N / 256) / 9
    F = [(1 - ell) * h / prev_N for h in prev_h]
    F[-1] += ell
    s = sum(F)
    return [f / s for f in F]


def n_clusters(M: int) -> int:
    return int(min(max(M // 1000, 16), 50000))


def _unit(x: torch.Tensor) -> torch.Tensor:
    return x / torch.linalg.vector_norm(x, dim=-1, keepdim=True)


class Workload:
    """Deterministic generator for one configuration's cache and prompt batch."""

    def __init__(self, cfg: Config, device="cpu", M: int | None = None, d: int | None = None):
        self.cfg = cfg
        self.device = torch.device(device)
        self.M = cfg.M if M is None else M
        self.d = cfg.d if d is None else d
        g = torch.Generator(device="cpu").manual_seed(cfg.gen_seed)
        d_ = self.d
        self.C = n_clusters(self.M)
        mu = _unit(torch.randn(d_, generator=g, dtype=torch.float64))
        base = _unit(torch.randn(self.C, d_, generator=g, dtype=torch.float64))
        cent = _unit(ANISO_A * mu + math.sqrt(1 - ANISO_A ** 2) * base)
        self.mu = mu
        self.centroids = cent.to(torch.float32)
        self.tau = (0.25 + 0.65 * torch.rand(self.C, generator=g, dtype=torch.float64)).to(torch.float32)
        w = (torch.arange(self.C, dtype=torch.float64) + 1.0) ** -1.1
        self.weights = (w / w.sum()).to(torch.float32)
        self._cent_dev = self.centroids.to(self.device)
        self._tau_dev = self.tau.to(self.device)
        # cluster draws of cache rows by inverse CDF on a CPU fp64 cumulative sum: regenerating a block
        # (rows_at) must reproduce it bit for bit, which torch.multinomial on CUDA does not guarantee
        # (its device cumsum is a decoupled look-back scan whose float summation order varies)
        cdf = torch.cumsum(w, 0)
        self._cdf_dev = (cdf / cdf[-1]).to(self.device)

    # ---- cache ---------------------------------------------------------------------
    def _gen(self, *key) -> torch.Generator:
        s = self.cfg.gen_seed
        for k in key:
            s = (s * 1_000_003 + int(k) + 0x9E3779B1) % (1 << 62)
        return torch.Generator(device=self.device).manual_seed(s)

    def cache_block(self, b: int) -> torch.Tensor:
        """Rows [b*BLOCK, min((b+1)*BLOCK, M)) as fp32 [rows, d] on self.device."""
        lo = b * BLOCK
        rows = min(BLOCK, self.M - lo)
        if rows <= 0:
            return torch.empty(0, self.d, device=self.device)
        g = self._gen(1, b)
        u = torch.rand(rows, generator=g, device=self.device, dtype=torch.float64)
        j = torch.searchsorted(self._cdf_dev, u, right=True).clamp_(max=self.C - 1)
        noise = torch.randn(rows, self.d, generator=g, device=self.device)
        scale = 0.5 + 1.5 * torch.rand(rows, 1, generator=g, device=self.device)
        row = _unit(self._cent_dev[j] + self._tau_dev[j, None] * noise / math.sqrt(self.d))
        return row * scale

    def cache_rows(self, lo: int, hi: int) -> torch.Tensor:
        """Rows [lo, hi) (any alignment) as fp32."""
        out = []
        b = lo // BLOCK
        while b * BLOCK < hi:
            blk = self.cache_block(b)
            a = max(lo, b * BLOCK) - b * BLOCK
            z = min(hi, (b + 1) * BLOCK) - b * BLOCK
            out.append(blk[a:z])
            b += 1
        if not out:
            return torch.empty(0, self.d, device=self.device)
        return torch.cat(out, 0)

    def n_blocks(self) -> int:
        return (self.M + BLOCK - 1) // BLOCK

    # ---- prompts -------------------------------------------------------------------
    def prompt_plan(self, N: int, batch: int = 0):
        """Kinds (0 novel, 1 dup, 2 cluster), dup source gids and cluster ids for a batch."""
        g = torch.Generator(device="cpu").manual_seed(self.cfg.gen_seed * 7919 + batch)
        mix = torch.tensor(self.cfg.mix, dtype=torch.float64)
        kind = torch.multinomial(mix, N, replacement=True, generator=g)
        if self.M == 0:
            kind = torch.where(kind == 1, torch.full_like(kind, 2), kind)
        src = torch.randint(0, max(self.M, 1), (N,), generator=g)
        cl = torch.multinomial(self.weights.double(), N, replacement=True, generator=g)
        return kind, src, cl

    def prompts(self, N: int, batch: int = 0, dup_rows: torch.Tensor | None = None) -> torch.Tensor:
        """fp32 [N, d].  ``dup_rows`` ([N, d], rows of the cache at the dup gids) may be passed
        by a caller streaming the cache; otherwise the needed cache rows are regenerated."""
        kind, src, cl = self.prompt_plan(N, batch)
        dev = self.device
        g = self._gen(2, batch)
        d_ = self.d
        noise = torch.randn(N, d_, generator=g, device=dev)
        scale = 0.5 + 1.5 * torch.rand(N, 1, generator=g, device=dev)
        fresh = _unit(ANISO_A * self.mu.to(dev, torch.float32)
                      + math.sqrt(1 - ANISO_A ** 2)
                      * _unit(torch.randn(N, d_, generator=g, device=dev)))
        out = torch.empty(N, d_, device=dev)
        kind_d = kind.to(dev)
        # novel
        nov = _unit(fresh + 0.5 * noise / math.sqrt(d_))
        # cluster
        cl_d = cl.to(dev)
        clu = _unit(self._cent_dev[cl_d] + self._tau_dev[cl_d, None] * noise / math.sqrt(d_))
        out = torch.where((kind_d == 0)[:, None], nov, clu)
        if bool((kind == 1).any()):
            if dup_rows is None:
                dup_rows = self.rows_at(src[kind == 1])
                full = torch.zeros(N, d_, device=dev)
                full[(kind == 1).to(dev)] = dup_rows
                dup_rows = full
            dup = _unit(_unit(dup_rows) + 0.12 * noise / math.sqrt(d_))
            out = torch.where((kind_d == 1)[:, None], dup, out)
        return (out * scale).contiguous()

    def rows_at(self, gids: torch.Tensor) -> torch.Tensor:
        """Cache rows at arbitrary gids (regenerates the covering blocks)."""
        gids = gids.to(torch.int64)
        out = torch.empty(len(gids), self.d, device=self.device)
        blocks = torch.unique(gids // BLOCK)
        for b in blocks.tolist():
            sel = (gids // BLOCK) == b
            blk = self.cache_block(b)
            out[sel.to(self.device)] = blk[(gids[sel] - b * BLOCK).to(self.device)]
        return out
