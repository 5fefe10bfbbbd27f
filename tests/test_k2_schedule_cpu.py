"""K2's work-schedule choice (host logic in libpas, no device): the dynamic chunked schedule and the
static ranges satisfy the invariants the kernels rely on (DESIGN.md 8 "K2 schedule")."""
import math

import pytest

WORKERS = 148          # persistent single-CTA workers (one per SM)


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


CASES = [(N, M) for N in (1, 64, 256, 512, 513, 2048, 2200, 4096, 4097, 16384, 65536, 131072)
         for M in (1, 255, 1000, 100_000, 1_000_000, 10_000_000, 50_000_000, 110_000_000)]


@pytest.mark.parametrize("N,M", CASES)
def test_schedule_invariants(pas, N, M):
    s = pas.pas_debug_k2_schedule(N, M)
    MT, NT, R, T, CS = s["MT"], s["NT"], s["R"], s["T"], s["CS"]
    small = N <= 128 and MT % 2 == 1 and math.ceil(M / 128) <= 128          # the 128-row cache tile
    assert s["tile_rows"] == (128 if small else 256)
    assert MT == math.ceil(N / 128) and NT == math.ceil(M / s["tile_rows"])
    if small:
        assert T == 0 and R == max(1, min(NT, s["cand_cap"] // max(N, 1)))   # one cache tile per CTA
    assert 1 <= R <= min(128, max(NT, 1)) and R * N <= s["cand_cap"]      # S-way merge, candidate buffer
    assert s["pair"] == (MT <= 4 and MT % 2 == 0)                          # CTA pair: whole tile pairs, N <= 512
    if T:
        L = math.ceil(NT / R)                                              # tiles of the longest range
        assert not s["pair"] and 4 <= T <= 128
        assert CS == math.ceil(L / T) and CS >= 2                          # every tile in some chunk
        assert T <= max(4, math.ceil(L / 6))                               # short ranges: >= ~6 steps
        assert R * s["MTg"] >= WORKERS                                     # >= one unit per SM per step
        assert 1 <= s["MTg"] <= MT
        assert CS * R * MT < 2 ** 31                                       # unit ids are int32
        # L2: the chunks in flight, (ceil(148 / MTg) + 1) T tiles of 256 x 768 bf16, fit the budget
        assert (math.ceil(WORKERS / s["MTg"]) + 1) * T * 256 * 768 * 2 <= 100 << 20 or T == 4
    else:
        assert CS == 0


def test_bench_configs(pas):
    c4 = pas.pas_debug_k2_schedule(65536, 10_000_000)
    assert (c4["R"], c4["T"], c4["MTg"]) == (1, 128, 512)                 # C4: one range, 128-tile chunks
    c3 = pas.pas_debug_k2_schedule(16384, 1_000_000)
    assert c3["R"] == 3 and c3["T"] > 0                                    # 128 prompt tiles < 148 SMs
    c2 = pas.pas_debug_k2_schedule(4096, 100_000)                          # C2: 40-tile ranges, 6 chunks
    assert (c2["R"], c2["T"], c2["CS"]) == (10, 7, 6)
    c1 = pas.pas_debug_k2_schedule(64, 1000)
    assert c1["pair"] == 0 and c1["T"] == 0                                # one 128-row tile: a single CTA
    assert c1["tile_rows"] == 128 and c1["R"] == 8                         # 8 CTAs of 128 cache rows
    assert pas.pas_debug_k2_schedule(256, 50_000_000)["pair"] == 1         # C5 at N = 256: the pair


def test_static_override(pas, monkeypatch):
    monkeypatch.setenv("PAS_K2_SCHED", "static")
    s = pas.pas_debug_k2_schedule(65536, 10_000_000)
    assert s["T"] == 0 and s["R"] >= 1


def test_bad_arguments(pas):
    with pytest.raises(pas.PasError):
        pas.pas_debug_k2_schedule(10, 100, 768, max_batch=5)
