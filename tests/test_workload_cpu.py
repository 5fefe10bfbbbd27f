"""Test plumbing and workload recipes (CPU): the synthetic generator reproduces rows bit for bit, the
C5 controller recipe, and the parallel streaming top-k used for the 50M-row parity test equals the
oracle's sequential streaming top-k."""
import numpy as np
import pytest
import torch

from oracle import route as O
from synth import BLOCK, CONFIGS, Workload, c5_fractions

from .parity import oracle_topk_parallel, oracle_topk_streaming


def test_rows_at_reproduces_loaded_blocks():
    """rows_at regenerates exactly the rows cache_block produced (the cluster draw is an
    inverse CDF on a CPU fp64 cumsum, so repeated generation is bit-identical)."""
    w = Workload(CONFIGS["C2"], M=3 * BLOCK + 17)
    gids = torch.tensor([0, 5, BLOCK - 1, BLOCK, 2 * BLOCK + 3, 3 * BLOCK + 16], dtype=torch.int64)
    got = w.rows_at(gids)
    for i, g in enumerate(gids.tolist()):
        blk = w.cache_block(g // BLOCK)
        assert torch.equal(got[i], blk[g % BLOCK])
    assert torch.equal(w.cache_block(1), w.cache_block(1))


def test_c5_fractions_recipe():
    grid = CONFIGS["C5"].grid
    F0 = c5_fractions(None, None, 256)
    assert F0 == [1.0 / len(grid)] * len(grid)
    h = [10, 20, 30, 40, 50, 106]
    F = c5_fractions(h, 256, 256)                      # l = 0: the previous batch's H_K / N
    assert np.allclose(F, np.array(h) / 256)
    F = c5_fractions(h, 256, 131072)                   # l = 1: everything at K = 25
    assert F[-1] == pytest.approx(1.0) and sum(F[:-1]) == pytest.approx(0.0)
    for N in (512, 4096, 65536):
        F = c5_fractions(h, 256, N)
        assert sum(F) == pytest.approx(1.0) and all(f >= 0 for f in F)


def test_parallel_streaming_topk_equals_sequential():
    w = Workload(CONFIGS["C1"], M=2500)
    rows = w.cache_rows(0, 2500).numpy()
    P = w.prompts(7).numpy()
    P[3] = 0.0                                          # an invalid prompt: sentinels
    chunks = [(a, rows[a:a + 300]) for a in range(0, 2500, 300)]
    a = oracle_topk_parallel(P, iter(chunks), 8, workers=3)
    b = oracle_topk_streaming(P, iter(chunks), 8)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert (a[0][3] == O.SENTINEL_GID).all()
