"""GPU parity of the stateful dispatcher (R28-R32) vs oracle/dispatch.py.

Batch after batch, teacher-forced on the GPU's optimal-K levels (their own parity is covered by
test_gpu_parity.py): the exact plan's K' (oracle O4-O8 on those levels) and then the oracle's
discrete-event Dispatcher, fed the same clock, must agree bit for bit with the CUDA path on K',
instance, slot (queue position), the batch lists, and the queue state after every batch
(queue lengths, busy-until, fired prompts and batches).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import dispatch as OD
from oracle import route as O
from synth import CONFIGS, Workload

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def pas():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas as p
    return p


def _run(pas, name, N, M, schedule, service, timeout, instance_level=None, F=None, bstar=4,
         mode=OD.GREEDY, loads=None, forecast=0):
    """schedule: list of (gap_us, n_prompts); loads: {batch: (lambda_rps, bstar_high)}."""
    cfg = CONFIGS[name]
    il = list(cfg.instance_level if instance_level is None else instance_level)
    F = list(cfg.F if F is None else F)
    w = Workload(cfg, device=DEV, M=max(M, 1000))
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=N, max_rows_per_rank=max(M, 1), device=0,
                   seed=cfg.route_seed)
    r.set_bands(cfg.grid, cfg.thresholds)
    r.set_fractions(F, il, bstar, mode)
    r.load_cache(w.cache_rows(0, M).contiguous())
    r.set_dispatcher(service, timeout)
    if forecast:
        r.set_forecast(forecast, 1)
    s = O.Setup(grid=cfg.grid, thresholds=cfg.thresholds, F=F, instance_level=il, bstar=bstar, mode=mode,
                topk=cfg.topk, seed=cfg.route_seed)
    disp = OD.Dispatcher(il, service, timeout)
    omode = mode
    now = 0
    P_all = w.prompts(N * len(schedule))
    W = len(il)
    stats = []
    for b, (gap, n) in enumerate(schedule):
        now += gap
        if loads and b in loads:
            lam, bh = loads[b]
            gm = r.set_load(lam, bh)
            omode = OD.load_mode(omode, lam, service, bh)
            assert gm == omode
            s.mode, s.bstar = omode, (bh if omode == OD.GREEDY else 1)
        r.set_clock(now)
        out = r.route(P_all[b * N:b * N + n].contiguous(), out=r.alloc_out(n))
        torch.cuda.synchronize()
        st = r.stats()
        g = {k: v.cpu().numpy() for k, v in out.items()}
        level = np.searchsorted(np.asarray(cfg.grid), g["K"])
        kp = np.searchsorted(np.asarray(cfg.grid), g["K_prime"])
        if not forecast:   # exact mode: K' from the oracle's plan on the same levels
            s.batch_seq = b
            ref = O.downstream(level, s)
            assert np.array_equal(kp, ref["level_prime"]), "K' differs"
        inst, slot = disp.dispatch(kp, s.mode, s.bstar, cfg.route_seed, b, now)
        assert np.array_equal(g["instance"], inst), f"batch {b}: instance differs"
        assert np.array_equal(g["slot"], slot), f"batch {b}: slot differs"
        # batch lists: this batch's prompts per instance in slot order
        counts = np.bincount(np.asarray(inst, dtype=np.int64), minlength=W)
        offs = np.concatenate([[0], np.cumsum(counts)])
        assert np.array_equal(g["bucket_offsets"][:W + 1], offs)
        for wi in range(W):
            mine = [p for p in range(n) if inst[p] == wi]
            assert g["bucket_prompts"][offs[wi]:offs[wi + 1]].tolist() == mine
        ost = disp.state()
        busy = [OD_NEVER if v is None else v for v in ost["busy_until"]]
        assert st["dispatcher"] == 1 and st["now_us"] == now
        assert st["queue_len"] == ost["queue"], (b, st["queue_len"], ost["queue"])
        assert st["busy_until_us"] == busy, (b, st["busy_until_us"], busy)
        assert st["fired_prompts"] == ost["fired_prompts"] and st["fired_batches"] == ost["fired_batches"]
        assert st["bucket_count"] == counts.tolist()
        stats.append(st)
    r.close()
    return stats


OD_NEVER = -(1 << 62)


def test_greedy_sequence_c2(pas):
    """C2's 8 instances (three at K=25), b* = 4: queues build up, drain between batches, time out."""
    rng = np.random.default_rng(11)
    sched = [(int(rng.integers(0, 400_000)), int(rng.integers(1, 1025))) for _ in range(10)]
    sched[3] = (0, 1024)                     # same instant as the previous batch
    sched[6] = (5_000_000, 7)                # long gap: everything drains, partial queues time out
    svc = [900_000, 1_100_000, 700_000, 1_300_000, 500_000, 400_000, 450_000, 400_000]
    _run(pas, "C2", 1024, 20_000, sched, svc, 250_000)


def test_greedy_overload_phase2_many_instances(pas):
    """Many instances on few levels, long service times: almost every pick is phase 2 (R29)."""
    il = [0] * 3 + [2] * 5 + [5] * 20
    F = [0.2, 0.0, 0.3, 0.0, 0.0, 0.5]
    rng = np.random.default_rng(5)
    svc = rng.integers(2_000_000, 9_000_000, len(il)).tolist()
    sched = [(int(rng.integers(0, 300_000)), 4096) for _ in range(6)]
    st = _run(pas, "C2", 4096, 20_000, sched, svc, 100_000, instance_level=il, F=F, bstar=3)
    assert max(st[-1]["queue_len"]) > 50       # really overloaded


def test_uniform_sequence_and_zero_timeout(pas):
    rng = np.random.default_rng(3)
    sched = [(int(rng.integers(0, 50_000)), int(rng.integers(1, 513))) for _ in range(8)]
    svc = rng.integers(10_000, 200_000, 8).tolist()
    _run(pas, "C2", 512, 20_000, sched, svc, 0, bstar=1, mode=OD.UNIFORM)


def test_load_mode_switches(pas):
    """pas_set_load flips uniform <-> greedy with hysteresis (R32) mid-sequence; queues carry over."""
    svc = [200_000] * 8                 # capacity at b* = 4: 8 x 4 / 0.2 s = 160 prompts/s
    sched = [(100_000, 256)] * 7
    loads = {0: (10.0, 4), 2: (150.0, 4), 3: (120.0, 4), 5: (100.0, 4), 6: (20.0, 4)}
    st = _run(pas, "C2", 256, 20_000, sched, svc, 250_000, bstar=1, mode=OD.UNIFORM, loads=loads)
    assert len(st) == 7


def test_small_c1_with_forecast_mode(pas):
    """The dispatcher composes with the f1 forecast mode (K' drawn i.i.d.; dispatch downstream)."""
    sched = [(30_000, 64)] * 12
    svc = [80_000, 120_000, 60_000, 90_000]
    _run(pas, "C1", 64, 1000, sched, svc, 40_000, forecast=200)


def test_dispatcher_api_errors(pas):
    cfg = CONFIGS["C1"]
    r = pas.Router(d=cfg.d, topk=cfg.topk, max_batch=64, max_rows_per_rank=1000, device=0)
    r.set_bands(cfg.grid, cfg.thresholds)
    with pytest.raises(pas.PasError):
        r.set_dispatcher([1000] * 4)                     # fractions first
    r.set_fractions(cfg.F, cfg.instance_level, 4, 0)
    with pytest.raises(pas.PasError):
        r.set_dispatcher([1000] * 3)                     # W mismatch
    with pytest.raises(pas.PasError):
        r.set_dispatcher([0] * 4)                        # service time >= 1 us
    with pytest.raises(pas.PasError):
        r.set_clock(5)                                   # dispatcher off
    r.set_dispatcher([1000] * 4, 10)
    r.set_clock(100)
    with pytest.raises(pas.PasError):
        r.set_fractions(cfg.F, cfg.instance_level, 65, 0)   # b* <= 64 while on
    st = r.dispatcher_state()
    assert st["queue"] == [0] * 4 and st["busy_until"] == [OD_NEVER] * 4
    r.set_dispatcher(None)                               # off again
    r.close()


def test_greedy_full_c4_batch(pas):
    """C4's batch size (65,536 prompts, 8 instances) through the dispatcher: three batches, the
    second at the same instant (all queues >= b*: phase 2 for most prompts)."""
    svc = [1_500_000, 1_400_000, 900_000, 1_000_000, 800_000, 700_000, 600_000, 650_000]
    _run(pas, "C4", 65536, 20_000, [(0, 65536), (0, 65536), (2_000_000, 65536)], svc, 250_000)
