"""K1 (a1 / a2) bit for bit: the bf16 rows the CUDA path writes -- the prompt-side Q_hat and the cache
store -- equal the oracle's quantisation (R11, oracle.quantize: bf16_RNE(fp32_RN(v / |v|_64))) on
adversarial rows (tests/k1_adversarial.py: quotients a few fp64 ulp from fp32 midpoints next to bf16
ties, exact fp32-subnormal midpoints, scales 2^+-100 ~ 1e+-30), on ordinary synth-v1 rows, and on bf16
input.  Until round 2 this was a claim; the subnormal rows caught a real
divergence (K1's fast path rounded subnormal quotients from the fp64 product)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import route as O
from synth import CONFIGS, Workload

from .k1_adversarial import near_midpoint_rows, scaled, subnormal_rows

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _oracle_bits(rows: np.ndarray) -> np.ndarray:
    q, valid = O.quantize(rows)
    bits = (q.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    bits[~valid] = 0
    return bits


def _rows() -> np.ndarray:
    mid, straddle = near_midpoint_rows(64)
    sub = subnormal_rows(16)
    syn = Workload(CONFIGS["C2"], device="cpu").prompts(2048).double().numpy()
    bad = np.zeros((3, 768))
    bad[1, 5] = np.nan
    bad[2, 7] = np.inf
    rows = np.concatenate([mid, scaled(mid, 100), scaled(mid, -100), sub, scaled(sub, 80), syn, bad])
    assert straddle.sum() == 64
    return rows.astype(np.float32)


def _gpu_bits(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _router(pas, N, M, world=1, rank=0):
    cfg = CONFIGS["C2"]
    r = pas.Router(d=768, topk=8, max_batch=N, max_rows_per_rank=M, device=0, rank=rank, world=world)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(cfg.F, cfg.instance_level, cfg.bstar, cfg.mode)
    return r


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_prompt_qhat_bit_exact(pas, dtype):
    rows = _rows()
    if dtype == "bf16":   # bf16 input: the oracle quantises the same (bf16-valued) rows
        rows = torch.from_numpy(rows).to(torch.bfloat16).float().numpy()
    N = len(rows)
    r = _router(pas, N, 256)
    r.load_cache(torch.from_numpy(_rows()[-200:-3]).to(DEV).contiguous())
    emb = torch.from_numpy(rows).to(DEV)
    if dtype == "bf16":
        emb = emb.to(torch.bfloat16)
    out = r.route(emb.contiguous())
    q = torch.empty(N, 768, dtype=torch.bfloat16, device=DEV)
    pas.pas_debug_qhat(r.ctx, q)
    torch.cuda.synchronize()
    got, want = _gpu_bits(q), _oracle_bits(rows)
    diff = np.argwhere(got != want)
    assert diff.size == 0, f"{len(diff)} bf16 values differ, first (row, col) {tuple(diff[0])}: gpu {got[tuple(diff[0])]:#06x} oracle {want[tuple(diff[0])]:#06x}"
    fl = out["flags"].cpu().numpy()
    assert np.all(fl[-2:] & 1) and np.all(fl[-3] & 1) and not np.any(fl[:-3] & 1)
    r.close()


def test_store_rows_bit_exact_on_both_shards(pas):
    """Cache insert (a2) through the round-robin shard filter: each rank's store rows are the oracle's
    quantisation of exactly its gids (g % 2 == rank, local row g // 2)."""
    rows = _rows()[:-3]                      # cache rows must be valid
    M = len(rows)
    want = _oracle_bits(rows)
    for rank in (0, 1):
        r = _router(pas, 8, (M + 1) // 2, world=2, rank=rank)
        r.load_cache(torch.from_numpy(rows[:777]).to(DEV).contiguous())
        r.load_cache(torch.from_numpy(rows[777:]).to(DEV).contiguous())
        n_local = pas.pas_cache_size(r.ctx)[1]
        q = torch.empty(n_local, 768, dtype=torch.bfloat16, device=DEV)
        pas.pas_debug_store_rows(r.ctx, 0, q)
        torch.cuda.synchronize()
        got = _gpu_bits(q)
        assert np.array_equal(got, want[rank::2]), (rank, int((got != want[rank::2]).sum()))
        r.close()
