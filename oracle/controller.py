"""NEXT f4: the Resource Controller's Model Cache Assigner + Query Fraction Solver.

Test infrastructure only (see oracle/__init__.py).  Exhaustive enumeration of every assignment of
the serving instances to K levels, each scored by the definition below; nothing is pruned or
reordered.

Passages followed
-----------------
P:88   "the Model Cache Assigner determines the optimal distribution of models across different
       values of K ... and the Query Fraction Solver calculates the proportion of prompts to be
       redirected to model at K ... denoted by F(K)" (via the Proteus MILP, not given in the paper).
P:207  "all K=0 models running at low loads, a mix of models running at moderate loads, and all
       K=25 models running at peak loads".
P:223  "For a cluster with tens of GPUs, the solver time is within 100 ms".
SPEC S:221-229 solve_assignment (lexicographic: served fraction, then expected quality)
LatencyProfile / QualityProfile, S:74-75 quality and service-time models.

Readings (R33-R36)
----------------------------
R33  Inputs: W serving instances, arrival rate lambda (prompts/s, >= 0), forecast H over the levels,
     per-level batch service time s_K (us) at the optimal batch size b*, and the degradation table
     c of Eq. 1 (D(K', K) = c(K' - K) for K' > K).  rate_K = (b* 1e6) / s_K prompts/s (SPEC:
     rate(K) = max_batch / service(K, max_batch)).  Prompt-agnostic quality of serving the forecast
     mix at K: a_K = 1 - sum_{i : K_i < K} H_i c(K - K_i)  (S:74 quality = 1 - D), summed over i
     ascending.
R34  For an assignment n (n_K instances at level K, sum n = W): cap_K = (n_K rate_K) / lambda,
     served S = min(1, sum_K cap_K) (levels ascending; lambda = 0: S = 1, cap unbounded where
     n_K > 0); F fills S in order of a_K descending (ties: lower level), F_K = min(cap_K, S - filled);
     quality q = sum F_K a_K in fill order.  This greedy fill is the exact optimum of the Query
     Fraction Solver's LP for that n (pinned against HiGHS).  All fp64, round-to-nearest, no fused
     multiply-add.
R35  The optimum: lexicographically max S, then max q, then the lexicographically LARGEST
     (n_0, n_1, ...) -- instances stay at the slower, higher-quality levels unless the load needs
     otherwise.  S and q are compared after rounding to integer multiples of 2^-40.
R36  Outputs: n, F (sums to S), F_route = F / S (what pas_set_fractions takes: the dispatcher never
     drops prompts), the instance levels (instances 0..W-1 level by level, ascending), S, q.

Pins (tests/test_oracle_controller.py): SPEC S:226-228 examples; exact-rational brute force
(fractions.Fraction, itertools) on 200 random small instances; HiGHS MILP (scipy.optimize.milp,
the paper's own formulation class) on random W <= 64 instances for (S*, q*); HiGHS LP for the
greedy fill; capacity and sum invariants.  Parity unpinned vs the paper's own numbers (Fig.
scale_solver gives solver times, not assignments).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

QUANT = float(2 ** 40)


def rates(service_us, bstar: int):
    """rate_K = (b* 1e6) / s_K prompts per second (R33)."""
    return [(float(bstar) * 1e6) / float(s) for s in service_us]


def agnostic_quality(H, grid, c):
    """a_K = 1 - sum_{i: K_i < K} H_i c(K - K_i), i ascending (R33)."""
    a = []
    for j, K in enumerate(grid):
        deg = 0.0
        for i in range(len(grid)):
            if grid[i] < K:
                deg = deg + float(H[i]) * float(c[K - grid[i]])
        a.append(1.0 - deg)
    return a


def fill_order(a):
    """Levels by a_K descending, ties to the lower level (R34)."""
    return sorted(range(len(a)), key=lambda k: (-a[k], k))


def evaluate(n, r, a, lam: float):
    """(S, q, F) of one assignment n (R34), scalar fp64."""
    nK = len(n)
    if lam == 0.0:
        cap = [math.inf if n[k] > 0 else 0.0 for k in range(nK)]
        S = 1.0
    else:
        cap = [(float(n[k]) * r[k]) / lam for k in range(nK)]
        tot = 0.0
        for k in range(nK):
            tot = tot + cap[k]
        S = min(1.0, tot)
    F = [0.0] * nK
    filled, q = 0.0, 0.0
    for k in fill_order(a):
        take = min(cap[k], S - filled)
        F[k] = take
        filled = filled + take
        q = q + take * a[k]
    return S, q, F


def quant(v: float) -> int:
    return int(np.rint(v * QUANT))


def compositions(W: int, nK: int):
    """Every n with n_K >= 0 and sum n = W."""
    for bars in itertools.combinations(range(W + nK - 1), nK - 1):
        prev, n = -1, []
        for b in bars:
            n.append(b - prev - 1)
            prev = b
        n.append(W + nK - 2 - prev)
        yield tuple(n)


def n_compositions(W: int, nK: int) -> int:
    return math.comb(W + nK - 1, nK - 1)


def _best(cands):
    """max over (quant S, quant q, n) (R35)."""
    return max(cands, key=lambda t: (t[0], t[1], t[2]))


def solve(W: int, lam: float, H, service_us, bstar: int, grid, c):
    """Exhaustive enumeration (plain loops; small W / nK).  Returns a dict of R36 outputs."""
    r = rates(service_us, bstar)
    a = agnostic_quality(H, grid, c)
    best = None
    for n in compositions(W, len(grid)):
        S, q, F = evaluate(n, r, a, lam)
        key = (quant(S), quant(q), n)
        if best is None or key > best[0]:
            best = (key, S, q, F)
    return _result(best[0][2], best[1], best[2], best[3], grid)


def _result(n, S, q, F, grid):
    inst = [k for k in range(len(grid)) for _ in range(n[k])]
    return dict(n=list(n), S=S, q=q, F=list(F), F_route=[f / S for f in F], instance_level=inst)


def solve_vectorized(W: int, lam: float, H, service_us, bstar: int, grid, c):
    """The same enumeration as solve(), evaluated with NumPy arrays (elementwise IEEE fp64 in the
    same operation order), for W up to 64 with 6 levels (11M assignments)."""
    nK = len(grid)
    r = rates(service_us, bstar)
    a = agnostic_quality(H, grid, c)
    # all compositions, built level by level (n_0 outermost)
    n = np.zeros((1, 0), dtype=np.int64)
    rem = np.array([W], dtype=np.int64)
    for k in range(nK - 1):
        reps = rem + 1
        idx = np.repeat(np.arange(len(rem)), reps)
        v = np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps)   # 0..rem per row
        n = np.concatenate([n[idx], v[:, None]], axis=1)
        rem = rem[idx] - v
    n = np.concatenate([n, rem[:, None]], axis=1)
    nf = n.astype(np.float64)
    if lam == 0.0:
        cap = np.where(n > 0, np.inf, 0.0)
        S = np.ones(len(n))
    else:
        cap = (nf * np.array(r)[None, :]) / lam
        tot = np.zeros(len(n))
        for k in range(nK):
            tot = tot + cap[:, k]
        S = np.minimum(1.0, tot)
    filled = np.zeros(len(n))
    q = np.zeros(len(n))
    for k in fill_order(a):
        take = np.minimum(cap[:, k], S - filled)
        filled = filled + take
        q = q + take * a[k]
    qS = np.rint(S * QUANT).astype(np.int64)
    qq = np.rint(q * QUANT).astype(np.int64)
    # lexicographic max of (qS, qq, n_0, n_1, ...): np.lexsort sorts by the LAST key first
    keys = [n[:, k] for k in range(nK - 1, -1, -1)] + [qq, qS]
    order = np.lexsort(keys)
    bi = int(order[-1])
    nb = tuple(int(x) for x in n[bi])
    S_b, q_b, F_b = evaluate(nb, r, a, lam)
    return _result(nb, S_b, q_b, F_b, grid)


def solve_exact(W: int, lam, H, service_us, bstar: int, grid, c):
    """Exact-rational brute force (fractions.Fraction of the fp64 inputs): the lexicographic
    optimum of (S, q, n) with no rounding at all (pin for tiny instances)."""
    from fractions import Fraction as Fr
    r = [Fr(bstar) * Fr(10**6) / Fr(int(s)) for s in service_us]
    a = []
    for j, K in enumerate(grid):
        a.append(Fr(1) - sum((Fr(H[i]) * Fr(c[K - grid[i]]) for i in range(len(grid)) if grid[i] < K), Fr(0)))
    order = sorted(range(len(grid)), key=lambda k: (-a[k], k))
    lamF = Fr(lam)
    best = None
    for n in compositions(W, len(grid)):
        if lamF == 0:
            S = Fr(1)
            cap = [None if n[k] > 0 else Fr(0) for k in range(len(grid))]
        else:
            cap = [Fr(n[k]) * r[k] / lamF for k in range(len(grid))]
            S = min(Fr(1), sum(cap, Fr(0)))
        filled, q = Fr(0), Fr(0)
        for k in order:
            take = S - filled if cap[k] is None else min(cap[k], S - filled)
            filled += take
            q += take * a[k]
        key = (S, q, n)
        if best is None or key > best:
            best = key
    return dict(n=list(best[2]), S=best[0], q=best[1])
