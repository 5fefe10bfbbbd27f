"""NEXT f3: the stateful load-aware Query Dispatcher.

Test infrastructure only (see oracle/__init__.py).  A plain discrete-event restatement, prompt by
prompt and event by event, of SPEC's pick_worker / form_batch rules; nothing here is closed-form
or tuned.

Passages followed
-----------------
P:104  "employs uniform routing with a batch size of 1" at low load, "distributing prompts randomly
       to workers"; at high load it "assigns prompts to GPU workers with the longest queues ...
       likely to be fired soonest at optimal batch size"; the dispatcher alternates between the two
       "based on load".
SPEC S:286-295 WorkerQueue / BatchPolicy (FIFO queue, busy-until, oldest-enqueue timestamp; b*,
       batch timeout Delta), S:305-313 pick_worker, S:314-322 form_batch, S:242 / S:268 the load-
       mode switch (0.8 utilisation, hysteresis 0.1), S:336-338 FIFO and timeout invariants.

Readings (R28-R32)
----------------------------
R28  Time is an integer number of microseconds.  Every routed batch arrives at one instant `now`
     (non-decreasing across batches, given by the caller); its prompts are dispatched one by one in
     prompt order at that instant, and no batch fires between two prompts of the same routed batch
     (the routed batch is dispatched atomically).  Events between two routed batches follow the
     policy (b*) in force when the earlier one was dispatched.
R29  pick_worker, greedy (high load): among the instances at K', those whose queue is shorter than
     b*: the longest, ties to the lowest id.  If every queue holds >= b*: the instance whose
     next batch would START soonest, busy-until + (queued full batches) x service =
     max(B_w, now) + floor(Q_w / b*) s_w, ties to the lowest id.  SPEC's "busy-until + queued work"
     is read as the start time of the batch the prompt would join ("fired soonest"): the prompt
     joins a partially filled last batch at no extra delay.  From empty, idle instances with equal
     service times this reduces exactly to the stateless packing of R13 (pinned).
     Uniform (low load): I_j[(u n_j) >> 32] with the Philox stream-2 word u (R14), b* = 1.
R30  form_batch: an instance fires when it is idle (busy-until <= t) and its queue holds >= b*
     prompts (ready when the b*-th oldest arrived) or its oldest prompt has waited >= Delta (ready
     at oldest + Delta); it fires min(Q, b*) prompts in FIFO order and is busy for s_w
     (one service time per batch, whatever its size <= b*).  Events are processed in time order
     (ties: lowest instance id) up to and including `now`, before and again after the routed
     batch is dispatched.
R31  Outputs: slot = the prompt's position in its instance's queue when it was appended (the
     prompts still waiting from earlier batches come first); the batch lists hold this batch's
     prompts per instance in slot order.  State after the batch: per-instance queue length,
     busy-until, cumulative fired prompts and batches.
R32  Load mode: utilisation u = lambda / capacity, capacity = sum_w b*_high / s_w
     (prompts per second at the optimal batch size); low -> high when u > 0.8, high -> low when
     u < 0.7; high uses b*_high, low uses b* = 1.

Pins (tests/test_oracle_dispatch.py): SPEC worked examples (queues [2,3,1], b* = 4 -> the queue of
3; queues [4,4], equal busy-until -> instance 0; form_batch b* = 4 with 5 queued -> 4; 2 queued
after 0.3 s > Delta = 0.25 s -> 2; b* = 1 -> immediate), the reduction to the stateless closed form
R13 (tests/test_oracle_routing.py pins it to W1), conservation, FIFO, the timeout bound, the
"fired soonest" optimality of every phase-2 pick checked by brute force over the instances, and
the S:312 uniform statistics.  Parity unpinned vs the paper's own numbers (it prints no queue
trace).
"""
from __future__ import annotations

from collections import deque

from . import philox

GREEDY = 0
UNIFORM = 1
HIGH_UTIL = 0.8          # S:242 "utilisation > 0.8"
HYSTERESIS = 0.1         # S:242 "hysteresis 0.1"


class Dispatcher:
    """Per-instance FIFO queues with busy-until times (SPEC S:286-295 WorkerQueue)."""

    def __init__(self, instance_level, service_us, timeout_us: int):
        if len(service_us) != len(instance_level):
            raise ValueError("one service time per instance")
        if any(int(s) <= 0 for s in service_us) or int(timeout_us) < 0:
            raise ValueError("service times must be > 0 and the timeout >= 0")
        self.level = [int(v) for v in instance_level]
        self.service = [int(s) for s in service_us]
        self.timeout = int(timeout_us)
        self.W = len(self.level)
        self.queue = [deque() for _ in range(self.W)]     # arrival times of the waiting prompts
        self.tags = [deque() for _ in range(self.W)]      # (batch_seq, p) of the waiting prompts
        self.log = []                                      # fired batches: (time, w, [tags])
        self.busy_until = [None] * self.W                  # None: never busy
        self.fired_prompts = [0] * self.W
        self.fired_batches = [0] * self.W
        self.clock = None
        self.bstar = 1                                     # policy in force since the last batch

    # ---- form_batch (R30) ---------------------------------------------------------------------
    def _ready_time(self, w: int, bstar: int):
        q = self.queue[w]
        if not q:
            return None
        if len(q) >= bstar:
            ready = q[bstar - 1]              # the batch filled up when its b*-th prompt arrived
        else:
            ready = q[0] + self.timeout       # the oldest prompt has waited Delta
        b = self.busy_until[w]
        return ready if b is None else max(b, ready)

    def advance(self, now: int, bstar: int):
        """Fire every batch whose time is <= now, in time order (ties: lowest id)."""
        while True:
            events = []
            for w in range(self.W):
                t = self._ready_time(w, bstar)
                if t is not None and t <= now:
                    events.append((t, w))
            if not events:
                return
            t, w = min(events)
            n = min(len(self.queue[w]), bstar)
            for _ in range(n):
                self.queue[w].popleft()
            self.log.append((t, w, [self.tags[w].popleft() for _ in range(n)]))
            self.busy_until[w] = t + self.service[w]
            self.fired_prompts[w] += n
            self.fired_batches[w] += 1

    # ---- pick_worker (R29) --------------------------------------------------------------------
    def start_time(self, w: int, now: int, bstar: int) -> int:
        """When the batch a new prompt would join at instance w starts (R29)."""
        b = self.busy_until[w]
        free = now if b is None else max(b, now)
        return free + (len(self.queue[w]) // bstar) * self.service[w]

    def pick(self, j: int, mode: int, bstar: int, u: int, now: int) -> int:
        I = [w for w in range(self.W) if self.level[w] == j]
        if not I:
            raise ValueError(f"no instance at level {j} (S:309)")
        if mode == UNIFORM:
            return I[(int(u) * len(I)) >> 32]
        below = [w for w in I if len(self.queue[w]) < bstar]
        if below:   # the longest queue still below b*, lowest id on ties
            return min(below, key=lambda w: (-len(self.queue[w]), w))
        return min(I, key=lambda w: (self.start_time(w, now, bstar), w))

    # ---- one routed batch ---------------------------------------------------------------------
    def dispatch(self, kp, mode: int, bstar: int, seed: int, batch_seq: int, now: int):
        """Route-and-batch one batch of K' level indices arriving at `now` (R28).

        Returns (instance, slot) per prompt; the state moves to after the batch."""
        if bstar < 1 or (mode == UNIFORM and bstar != 1):
            raise ValueError("b* >= 1, and uniform routing uses b* = 1 (P:104)")
        if self.clock is not None and now < self.clock:
            raise ValueError("the clock must not go backwards")
        self.advance(now, self.bstar)           # events since the last batch, old policy
        self.clock = now
        self.bstar = bstar
        n = len(kp)
        u = philox.uniform_words(n, seed, batch_seq) if mode == UNIFORM else [0] * n
        inst = [0] * n
        slot = [0] * n
        for p in range(n):
            w = self.pick(int(kp[p]), mode, bstar, int(u[p]), now)
            inst[p] = w
            slot[p] = len(self.queue[w])
            self.queue[w].append(now)
            self.tags[w].append((batch_seq, p))
        self.advance(now, bstar)                # idle instances fire at once (form_batch at now)
        return inst, slot

    def state(self):
        return dict(queue=[len(q) for q in self.queue],
                    busy_until=list(self.busy_until),
                    fired_prompts=list(self.fired_prompts),
                    fired_batches=list(self.fired_batches))


def capacity_rps(service_us, bstar_high: int) -> float:
    """Prompts per second the instances serve at the optimal batch size (R32)."""
    return sum(bstar_high / (s * 1e-6) for s in service_us)


def load_mode(prev_mode: int, lam_rps: float, service_us, bstar_high: int) -> int:
    """S:242 / S:268: high iff utilisation > 0.8, with hysteresis 0.1 (R32)."""
    u = lam_rps / capacity_rps(service_us, bstar_high)
    if prev_mode == UNIFORM:
        return GREEDY if u > HIGH_UTIL else UNIFORM
    return UNIFORM if u < HIGH_UTIL - HYSTERESIS else GREEDY
