"""NEXT f1: the forecast-driven streaming mode of the dispatcher.

Test infrastructure only (see oracle/__init__.py).  Plain restatement, no tuning.

Passages followed
-----------------
P:88   "the Optimal-K Predictor forecasts the optimal-K distribution (H_K) for the incoming
       prompt queries"; the Controller "runs periodically using query logs".
P:89   the K-to-K' Route Planner finds "redirection probabilities" (the Route-Plan), which the
       Query Dispatcher uses "as Redirection Logic": for an incoming prompt with an optimal-K the
       plan "determines the appropriate alternate value of K (K')".
P:96   Eq. 1, D_Q = sum_{i,j: K'_j > K_i} P(K'_j|K_i) H_K(K_i) D(K'_j, K_i).
P:218, P:225  H_K is predicted from a window of past K's; "for the chosen value of 1000, it
       saturated at low error at around 0.01" (L2 prediction error).
SPEC S:202-213 HkPredictor / predict_hk, S:296-304 route_prompt, S:323-330 record_optimal_k,
S:533-540 l2_hist_error give the interface and worked examples.

Readings (R21-R24)
----------------------------
R21  The predictor is a ring buffer of the last W optimal-K level indices, fed after every batch
     with that batch's K's in prompt order; the forecast is its normalised histogram, uniform over
     the grid when empty.
R22  The Route-Plan for fractional (H, F) is the Eq. 1 optimum for convex D: the monotone
     (north-west-corner) coupling x_ij = |[Hc_{i-1}, Hc_i) n [Fc_{j-1}, Fc_j)|, P(K'_j|K_i) =
     x_ij / H_i.  Cumulative masses are held in 32-bit fixed point (units of 2^-32) so that plan and
     sampling are integer arithmetic:
       Hc_i = floor(2^32 * cnt_{<=i} / n)           (exact integer division; uniform if n = 0)
       Fc_j = floor(2^32 * fl(F_0 + ... + F_j))      (fp64, summed left to right), and 2^32 from
                                                     the last level with F_j > 0 on.
R23  K' is sampled i.i.d. per prompt by inverse CDF on the coupling: u = w0 of the
     Philox stream 3 word of prompt p, pos = Hc_{i-1} + ((u * (Hc_i - Hc_{i-1})) >> 32), and
     K'_p = grid[j] for the j with Fc_{j-1} <= pos < Fc_j; so P(K' = j | K = i) = x_ij / H_i up to
     2^-32.  A class the forecast gives no mass (Hc_i = Hc_{i-1}) maps to pos = min(Hc_{i-1},
     2^32 - 1), the level the monotone coupling assigns at that cumulative mass ("unforecast").
R24  The plan is rebuilt from the window every `replan_every`-th batch ("runs periodically")
     and whenever F changes; between rebuilds the held plan routes.  Reported per batch: the
     plan's expected D_Q (Eq. 1 on the fixed-point plan), the realised D_Q = sum_p D(K'_p, K_p) / N,
     the realised move counts x_ij, and the L2 error between the forecast the plan was built from
     and the batch's realised H_K.

Pins (tests/test_oracle_forecast.py): SPEC worked examples (predict_hk, record_optimal_k,
route_prompt, l2_hist_error, the three plan_routes examples in fractional form), the HiGHS LP on
fractional (H, F) for random convex instances, exact integer marginals of the coupling, the
closed-form count of Philox words per (i, j), sampling statistics, and the stationary-stretch
invariant (L1 < 0.03 over 10k prompts).  No number printed by the paper applies: "parity unpinned
vs the paper's own numbers" (the figure's 0.01 error depends on the trace, which is not published).
"""
from __future__ import annotations

import math
from collections import deque

import numpy as np

from . import philox

ONE = 1 << 32                 # fixed-point unit of cumulative mass (R22)
STREAM_FORECAST = 3           # Philox stream of the i.i.d. K' draw (R23)


# --------------------------------------------------------------------------------------
# R21 the Optimal-K Predictor (ring buffer of past K's)
# --------------------------------------------------------------------------------------

class Predictor:
    """record_optimal_k / predict_hk on level indices."""

    def __init__(self, nK: int, window: int):
        if window < 1:
            raise ValueError("window must be >= 1")
        self.nK = nK
        self.W = window
        self.buf = deque(maxlen=window)

    def record(self, levels) -> None:
        """Append the batch's optimal-K levels in prompt order, evicting the oldest beyond W."""
        for lv in levels:
            self.buf.append(int(lv))

    def counts(self):
        """(cnt[nK], n): occurrences of each level in the window and the window length."""
        cnt = np.zeros(self.nK, dtype=np.int64)
        for lv in self.buf:
            cnt[lv] += 1
        return cnt, len(self.buf)

    def predict(self) -> np.ndarray:
        """Normalised histogram; uniform over the grid when the window is empty."""
        cnt, n = self.counts()
        if n == 0:
            return np.full(self.nK, 1.0 / self.nK)
        return cnt / n


def l2_hist_error(predicted, realized) -> float:
    """sqrt(sum_K (p_hat - p)^2) ("L2 prediction error")."""
    p = np.asarray(predicted, dtype=np.float64)
    q = np.asarray(realized, dtype=np.float64)
    if p.shape != q.shape:
        raise ValueError("grid mismatch")
    acc = 0.0
    for a, b in zip(p, q):
        acc += (a - b) * (a - b)
    return math.sqrt(acc)


# --------------------------------------------------------------------------------------
# R22 the fixed-point Route-Plan
# --------------------------------------------------------------------------------------

def cumulative_H(cnt, n: int, nK: int):
    """Hc[0..nK]: Hc[0] = 0, Hc[i+1] = floor(2^32 cnt_{<=i} / n); uniform 1/nK if n = 0."""
    Hc = [0] * (nK + 1)
    run = 0
    for i in range(nK):
        if n == 0:
            Hc[i + 1] = ((i + 1) * ONE) // nK
        else:
            run += int(cnt[i])
            Hc[i + 1] = (run * ONE) // n
    return Hc


def cumulative_F(F):
    """Fc[0..nK]: Fc[0] = 0, Fc[j+1] = floor(2^32 fl(F_0 + .. + F_j)) (left to right), and 2^32
    from the last level with F_j > 0 on (so no mass reaches a level without serving instances)."""
    nK = len(F)
    jlast = max(j for j in range(nK) if float(F[j]) > 0.0)
    Fc = [0] * (nK + 1)
    s = 0.0
    for j in range(nK):
        s = s + float(F[j])
        Fc[j + 1] = ONE if j >= jlast else min(max(math.floor(s * ONE), 0), ONE)
    return Fc


def coupling(Hc, Fc):
    """x_ij = |[Hc_i, Hc_{i+1}) n [Fc_j, Fc_{j+1})| in units of 2^-32 (the monotone coupling)."""
    nK = len(Hc) - 1
    x = np.zeros((nK, nK), dtype=np.int64)
    for i in range(nK):
        for j in range(nK):
            lo = max(Hc[i], Fc[j])
            hi = min(Hc[i + 1], Fc[j + 1])
            x[i, j] = max(0, hi - lo)
    return x


def plan_rows(Hc, Fc):
    """P(K'_j | K_i) = x_ij / H_i as floats (rows with no forecast mass are None)."""
    x = coupling(Hc, Fc)
    rows = []
    for i in range(len(Hc) - 1):
        w = Hc[i + 1] - Hc[i]
        rows.append(None if w == 0 else x[i] / w)
    return rows


def dq_plan(Hc, Fc, grid, c) -> float:
    """Eq. 1 on the fixed-point plan: sum_{j>i} (x_ij / 2^32) c(K_j - K_i), summed i-major."""
    x = coupling(Hc, Fc)
    nK = len(grid)
    acc = 0.0
    for i in range(nK):
        for j in range(nK):
            if j > i and x[i, j]:
                acc += (x[i, j] / ONE) * float(c[grid[j] - grid[i]])
    return acc


# --------------------------------------------------------------------------------------
# R23 i.i.d. sampling from the plan
# --------------------------------------------------------------------------------------

def sample(levels, Hc, Fc, seed: int, batch_seq: int):
    """K' level index per prompt and the 'unforecast' mask (R23)."""
    n = len(levels)
    nK = len(Hc) - 1
    w0, _, _, _ = philox.stream_words(n, seed, batch_seq, STREAM_FORECAST)
    kp = np.empty(n, dtype=np.int64)
    unf = np.zeros(n, dtype=bool)
    for p in range(n):
        i = int(levels[p])
        width = Hc[i + 1] - Hc[i]
        unf[p] = width == 0
        pos = min(Hc[i] + ((int(w0[p]) * width) >> 32), ONE - 1)
        j = 0
        while j < nK - 1 and Fc[j + 1] <= pos:
            j += 1
        kp[p] = j
    return kp, unf


def words_per_level(Hc, Fc, i: int):
    """Closed form: how many of the 2^32 words u send class i to each level j.

    floor(u w / 2^32) < m  <=>  u < ceil(m 2^32 / w), so the words landing in offsets [a, b) of
    the class interval number ceil(b 2^32 / w) - ceil(a 2^32 / w).  Independent of sample()."""
    nK = len(Hc) - 1
    w = Hc[i + 1] - Hc[i]
    out = np.zeros(nK, dtype=np.int64)
    if w == 0:
        return out
    for j in range(nK):
        a = max(Hc[i], Fc[j]) - Hc[i]
        b = min(Hc[i + 1], Fc[j + 1]) - Hc[i]
        if b > a:
            out[j] = -((-b * ONE) // w) - (-((-a * ONE) // w))
    return out


def dq_realized(levels, kp, grid, c) -> float:
    """sum over prompts of D(K'_p, K_p) / N, from the move counts (i-major, j-minor)."""
    n = len(levels)
    if n == 0:
        return 0.0
    x = moves(levels, kp, len(grid))
    acc = 0.0
    for i in range(len(grid)):
        for j in range(len(grid)):
            if j > i and x[i, j]:
                acc += x[i, j] * float(c[grid[j] - grid[i]])
    return acc / n


def moves(levels, kp, nK: int):
    x = np.zeros((nK, nK), dtype=np.int64)
    for i, j in zip(levels, kp):
        x[int(i), int(j)] += 1
    return x


# --------------------------------------------------------------------------------------
# R24 the streaming dispatcher, batch by batch
# --------------------------------------------------------------------------------------

class ForecastRouter:
    """Batches through the forecast-driven path: plan (held or rebuilt), i.i.d. K', then the
    same route-and-batch as the exact path (oracle.route.route_and_batch / buckets)."""

    def __init__(self, nK: int, window: int, replan_every: int = 1):
        if replan_every < 1:
            raise ValueError("replan_every must be >= 1")
        self.pred = Predictor(nK, window)
        self.T = replan_every
        self.tick = 0
        self.Hc = None
        self.plan_cnt = None
        self.plan_n = 0
        self.F_planned = None

    def batch(self, level, s, route_mod):
        """One batch: level = the batch's optimal-K level indices (from O3), s = route.Setup."""
        nK = len(s.grid)
        F = [float(v) for v in s.F]
        replanned = self.Hc is None or self.tick % self.T == 0 or F != self.F_planned
        if replanned:
            cnt, n = self.pred.counts()
            self.Hc = cumulative_H(cnt, n, nK)
            self.plan_cnt, self.plan_n = cnt.copy(), n
            self.F_planned = F
        Fc = cumulative_F(F)
        self.tick += 1
        N = len(level)
        h = np.array([int(np.sum(level == i)) for i in range(nK)], dtype=np.int64)
        predicted = (np.full(nK, 1.0 / nK) if self.plan_n == 0 else self.plan_cnt / self.plan_n)
        l2 = l2_hist_error(predicted, h / N) if N else 0.0
        kp, unf = sample(level, self.Hc, Fc, s.seed, s.batch_seq)
        inst, slot = route_mod.route_and_batch(kp, s.instance_level, s.bstar, s.mode, s.seed, s.batch_seq)
        offsets, bp = route_mod.buckets(inst, slot, len(s.instance_level))
        x = moves(level, kp, nK)
        out = dict(h=h, x=x, f=x.sum(axis=0), level_prime=kp, instance=inst, slot=slot, offsets=offsets,
                   bucket_prompts=bp, D_Q=dq_realized(level, kp, s.grid, s.c),
                   D_Q_plan=dq_plan(self.Hc, Fc, s.grid, s.c), l2=l2, n_unforecast=int(unf.sum()),
                   replanned=replanned, Hc=list(self.Hc), Fc=Fc, plan_counts=self.plan_cnt.copy(),
                   plan_n=self.plan_n)
        self.pred.record(level)
        return out
