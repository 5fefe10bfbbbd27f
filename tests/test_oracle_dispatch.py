"""Pins for the f3 stateful dispatcher oracle (oracle/dispatch.py, R28-R32).

What pins it (none of these retypes the oracle's own rule):
  * SPEC's worked examples of pick_worker and form_batch (tests/golden/spec_dispatch.json);
  * the reduction to the stateless closed form of R13 (O9, itself pinned to W1) when every
    instance starts empty and idle with one service time;
  * "fired soonest" by what-if simulation: with Delta = 0, every greedy pick made while
    all queues hold >= b* goes to an instance where the prompt's batch actually STARTS no later
    than at any other instance of its level, measured by draining a copy of the system;
  * conservation, FIFO per instance, the form_batch invariant after every batch (no idle
    instance holds a ready batch), the b* = 1 low-load rule, S:312 statistics;
  * the load-mode switch examples of S:245-246 and its hysteresis.
"""
import copy
import json
import os
from collections import deque

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import dispatch as D
from oracle import route as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_dispatch.json")))
FAR = 10**12


def _preset(queues, busy_until, level=None, service=None, timeout=250_000):
    W = len(queues)
    d = D.Dispatcher(level or [0] * W, service or [1000] * W, timeout)
    for w, q in enumerate(queues):
        d.queue[w] = deque([0] * q)
        d.tags[w] = deque([("pre", i) for i in range(q)])
        d.busy_until[w] = busy_until[w]
    d.clock = 0
    return d


def test_spec_pick_worker_high_longest_below_bstar():
    g = GOLD["pick_worker_high_longest_below_bstar"]
    d = _preset(g["queues"], [FAR] * 3)
    assert d.pick(0, D.GREEDY, g["bstar"], 0, now=10) == g["expect_worker"]


def test_spec_pick_worker_tie_lowest_id():
    g = GOLD["pick_worker_high_tie_lowest_id"]
    d = _preset(g["queues"], [FAR, FAR])
    assert d.pick(0, D.GREEDY, g["bstar"], 0, now=10) == g["expect_worker"]


def test_spec_pick_worker_uniform_statistics():
    g = GOLD["pick_worker_uniform"]
    d = D.Dispatcher([0] * g["workers"], [10**9] * g["workers"], 0)
    inst, _ = d.dispatch(np.zeros(g["picks"], int), D.UNIFORM, 1, seed=7, batch_seq=0, now=0)
    counts = np.bincount(inst, minlength=g["workers"])
    assert np.all(np.abs(counts - g["expect_each"]) <= g["tol"])


def test_spec_form_batch_full():
    g = GOLD["form_batch_full"]
    d = _preset([g["queue"]], [None])
    d.advance(0, g["bstar"])
    assert d.fired_prompts == [g["expect_fired"]] and len(d.queue[0]) == g["queue"] - g["expect_fired"]
    assert d.log[0][2] == [("pre", i) for i in range(g["expect_fired"])]   # the FIRST b* (FIFO)


def test_spec_form_batch_timeout():
    g = GOLD["form_batch_timeout"]
    d = _preset([g["queue"]], [None], timeout=g["timeout_us"])
    d.advance(g["timeout_us"] - 1, g["bstar"])   # the oldest has not yet waited Delta: nothing
    assert d.fired_prompts == [0]
    d.advance(g["waited_us"], g["bstar"])
    assert d.fired_prompts == [g["expect_fired"]]
    assert d.log[0][0] == g["timeout_us"]            # fired when the oldest had waited Delta
    assert d.busy_until[0] == g["timeout_us"] + 1000


def test_spec_form_batch_low_load_immediate():
    g = GOLD["form_batch_low_load"]
    d = D.Dispatcher([0], [5000], 250_000)
    d.dispatch(np.zeros(g["queue"], int), D.UNIFORM, g["bstar"], seed=1, batch_seq=0, now=100)
    assert d.fired_prompts == [g["expect_fired"]] and d.log[0][0] == 100


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 400), st.integers(1, 5), st.integers(2, 5), st.integers(0, 2**31))
def test_reduces_to_stateless_packing(N, bstar, nK, seed):
    rng = np.random.default_rng(seed)
    inst_level = list(range(nK)) + rng.integers(0, nK, int(rng.integers(0, 6))).tolist()
    kp = rng.integers(0, nK, N)
    d = D.Dispatcher(inst_level, [4000] * len(inst_level), 10**9)
    inst, slot = d.dispatch(kp, D.GREEDY, bstar, seed=seed, batch_seq=0, now=0)
    i0, s0 = O.route_and_batch(kp, inst_level, bstar, O.GREEDY, seed, 0)
    assert inst == i0.tolist() and slot == s0.tolist()


def _drain_start(d: D.Dispatcher, tag, bstar):
    """Time at which the batch holding `tag` starts when nothing else arrives."""
    d.advance(FAR * 10, bstar)
    for t, w, tags in d.log:
        if tag in tags:
            return t
    raise AssertionError("never fired")


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 2**31))
def test_greedy_pick_fires_soonest(seed):
    """Phase-2 picks (all queues >= b*) minimise the real start time of the prompt's batch."""
    rng = np.random.default_rng(seed)
    W = int(rng.integers(2, 6))
    bstar = int(rng.integers(1, 5))
    service = rng.integers(100, 3000, W).tolist()
    queues = rng.integers(bstar, 4 * bstar + 3, W).tolist()
    busy = [int(b) if b > 0 else None for b in rng.integers(-500, 5000, W)]
    d = _preset(queues, busy, service=service, timeout=0)
    # busy-until in the past with a full queue would have fired already: make the state consistent
    d.advance(0, bstar)
    if any(len(q) < bstar for q in d.queue):
        return
    w = d.pick(0, D.GREEDY, bstar, 0, now=0)
    starts = []
    for cand in range(W):
        e = copy.deepcopy(d)
        e.queue[cand].append(0)
        e.tags[cand].append(("new", 0))
        starts.append(_drain_start(e, ("new", 0), bstar))
    assert starts[w] == min(starts)
    assert w == min(c for c in range(W) if starts[c] == min(starts))   # ties: lowest id


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 2**31), st.sampled_from([D.GREEDY, D.UNIFORM]))
def test_multibatch_invariants(seed, mode):
    rng = np.random.default_rng(seed)
    nK = int(rng.integers(1, 4))
    inst_level = list(range(nK)) + rng.integers(0, nK, int(rng.integers(0, 4))).tolist()
    W = len(inst_level)
    bstar = 1 if mode == D.UNIFORM else int(rng.integers(1, 6))
    d = D.Dispatcher(inst_level, rng.integers(500, 20_000, W).tolist(), int(rng.integers(0, 30_000)))
    now, total = 0, 0
    enq = {w: [] for w in range(W)}
    for b in range(int(rng.integers(1, 8))):
        now += int(rng.integers(0, 15_000))
        kp = rng.integers(0, nK, int(rng.integers(0, 60)))
        q_before = None
        d.advance(now, d.bstar)            # what dispatch will see first (idempotent: same events)
        q_before = [len(q) for q in d.queue]
        inst, slot = d.dispatch(kp, mode, bstar, seed, b, now)
        total += len(kp)
        for w in range(W):   # slots of one instance: consecutive from its queue length (R31)
            mine = [slot[p] for p in range(len(kp)) if inst[p] == w]
            assert mine == list(range(q_before[w], q_before[w] + len(mine)))
            enq[w] += [(b, p) for p in range(len(kp)) if inst[p] == w]
        for p in range(len(kp)):
            assert inst_level[inst[p]] == kp[p]
        assert sum(d.fired_prompts) + sum(len(q) for q in d.queue) == total     # conservation
        for w in range(W):   # after the batch no idle instance holds a ready batch (form_batch)
            t = d._ready_time(w, bstar)
            assert t is None or t > now
    fired = {w: [tag for _, ww, tags in d.log if ww == w for tag in tags] for w in range(W)}
    for w in range(W):   # FIFO per instance: fired, then waiting, in enqueue order
        assert fired[w] + list(d.tags[w]) == enq[w]
        assert all(len(tags) <= bstar for _, ww, tags in d.log if ww == w)
    if mode == D.UNIFORM:
        assert all(len(tags) == 1 for _, _, tags in d.log)   # S:334 low load never batches


def test_clock_must_not_go_back():
    d = D.Dispatcher([0], [100], 0)
    d.dispatch([0], D.GREEDY, 2, 0, 0, now=50)
    with pytest.raises(ValueError):
        d.dispatch([0], D.GREEDY, 2, 0, 1, now=49)


def test_load_mode_spec_examples():
    service = [200_000] * 4                      # 0.2 s per batch
    cap = D.capacity_rps(service, 4)             # 4 instances x 4 prompts / 0.2 s = 80 rps
    assert cap == pytest.approx(80.0)
    # S:245 stationary low load stays low; S:246 a step above 0.8 capacity flips to high
    assert D.load_mode(D.UNIFORM, 10.0, service, 4) == D.UNIFORM
    assert D.load_mode(D.UNIFORM, 0.81 * cap, service, 4) == D.GREEDY
    # hysteresis 0.1: between 0.7 and 0.8 the mode holds; below 0.7 back to low
    assert D.load_mode(D.GREEDY, 0.75 * cap, service, 4) == D.GREEDY
    assert D.load_mode(D.UNIFORM, 0.75 * cap, service, 4) == D.UNIFORM
    assert D.load_mode(D.GREEDY, 0.69 * cap, service, 4) == D.UNIFORM
