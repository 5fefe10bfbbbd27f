"""O1..O10: plain CPU restatement of one batch of the paper's prompt routing.

Test infrastructure only (see oracle/__init__.py).  Nothing here is tuned; every
function follows the definition or the algorithm it cites, in the paper's order.
Readings of silent / garbled passages are DESIGN.md R1..R20.

Passages followed
-----------------
P:75   optimal-K = the least number of steps giving optimal quality; K = steps skipped.
P:88   Controller: F(K) per-K load fractions; H_K the optimal-K distribution.
P:89   Route Planner: redirect to K' < K (slower/better) or the closest K' > K
       (faster/worse, with degradation D), minimising D_Q.
P:96   Eq. 1: D_Q = sum_{i,j: K'_j > K_i} P(K'_j|K_i) H_K(K_i) D(K'_j, K_i).
P:102  Optimal-K Selector "first retrieves the nearest cache and determines the
       optimal K"; K-to-K' Router "selects the final approximate model at K'".
P:104  route-and-batch: uniform (random worker, batch 1) at low load, greedy
       (longest queue, optimal batch size) at high load.
SPEC S:149 (bands), S:160-171 (nearest / select examples), S:231-238 (plan_routes),
S:296-322 (route_prompt / pick_worker / form_batch) give the interface and examples.

Parity pins (tests/test_oracle_*.py): SPEC worked examples, Random123 KATs, brute
force on tiny inputs, HiGHS LP, the linear-D closed form, the worked example W1,
invariants and statistics.  The paper prints no routing output, so every pin is
definitional: "parity unpinned vs the paper's own numbers" applies to the whole
module ("Oracle pins").
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import philox

T_TOTAL = 50            # SPEC S:27 default total denoising steps ("50 to 100")
NEG_INF = float("-inf")
SENTINEL_GID = -1
NEAR_MARGIN = 2e-2      # north_star: near-tie margin reported, not failed

FLAG_INVALID = 1
FLAG_COLD = 2
FLAG_NEAR_TOP1 = 4
FLAG_NEAR_THRESHOLD = 8


# --------------------------------------------------------------------------------------
# O1 / O1'  similarity
# --------------------------------------------------------------------------------------

def row_valid(x: np.ndarray) -> np.ndarray:
    """A row is valid iff every element is finite and its L2 norm is non-zero (R16)."""
    x64 = np.asarray(x, dtype=np.float64)
    finite = np.all(np.isfinite(x64), axis=1)
    sq = np.where(finite[:, None], x64, 0.0)
    return finite & (np.sqrt(np.sum(sq * sq, axis=1)) > 0.0)


def similarity_A(P: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Tier A cosine similarity s(p,g) = <x_p, c_g> / (|x_p| |c_g|) in float64 ("closeness").

    From the caller's original (fp32) arrays; rows must be valid.
    """
    P64 = np.asarray(P, dtype=np.float64)
    C64 = np.asarray(C, dtype=np.float64)
    dots = P64 @ C64.T
    return dots / np.outer(np.linalg.norm(P64, axis=1), np.linalg.norm(C64, axis=1))


def bf16_rne_bits(y32: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit pattern (uint16) by round-to-nearest-even on the bits."""
    b = np.ascontiguousarray(y32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))
    return ((b + rounding) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def quantize(x: np.ndarray):
    """Tier B quantisation (R11): v_hat = bf16_RNE(fp32_RN(v / sqrt(sum v^2)_64)).

    Returns (bf16 values as float64 [n,d], valid[n]).  Invalid rows are all zero.
    """
    x64 = np.asarray(x, dtype=np.float64)
    valid = row_valid(x64)
    out = np.zeros_like(x64)
    if valid.any():
        xv = x64[valid]
        norm = np.sqrt(np.sum(xv * xv, axis=1))
        y32 = (xv / norm[:, None]).astype(np.float32)          # fp32 round-to-nearest
        out[valid] = bf16_bits_to_f64(bf16_rne_bits(y32))
    return out, valid


def similarity_B(Pq: np.ndarray, Cq: np.ndarray) -> np.ndarray:
    """Tier B: s_hat(p,g) = sum_i q_hat_pi c_hat_gi in float64 over the quantised vectors."""
    return np.asarray(Pq, dtype=np.float64) @ np.asarray(Cq, dtype=np.float64).T


# --------------------------------------------------------------------------------------
# O2  top-k
# --------------------------------------------------------------------------------------

def topk_sorted(scores: np.ndarray, gids: np.ndarray, k: int):
    """Full sort of every row by (score desc, gid asc) and keep k (R10); pad (-inf, -1) (R16)."""
    n, m = scores.shape
    ids = np.full((n, k), SENTINEL_GID, dtype=np.int64)
    sc = np.full((n, k), NEG_INF, dtype=np.float64)
    for p in range(n):
        order = np.lexsort((gids, -scores[p]))
        take = order[:k]
        ids[p, :len(take)] = gids[take]
        sc[p, :len(take)] = scores[p, take]
    return ids, sc


def topk_prefiltered(scores: np.ndarray, gids: np.ndarray, k: int):
    """Same result as ``topk_sorted``: rows are first cut to the elements whose score is at
    least the k-th largest value (no member of the top-k can be below it), then sorted."""
    n, m = scores.shape
    if m <= k:
        return topk_sorted(scores, gids, k)
    kth = -np.partition(-scores, k - 1, axis=1)[:, k - 1]
    ids = np.empty((n, k), dtype=np.int64)
    sc = np.empty((n, k), dtype=np.float64)
    for p in range(n):
        keep = np.nonzero(scores[p] >= kth[p])[0]
        sub_i, sub_s = topk_sorted(scores[p:p + 1, keep], gids[keep], k)
        ids[p], sc[p] = sub_i[0], sub_s[0]
    return ids, sc


def merge_topk(a_ids, a_sc, b_ids, b_sc, k: int):
    """Top-k of the union of two candidate sets (the top-k of a union is the top-k of the
    union of the parts' top-k) -- used to stream a cache too large to hold in fp64."""
    ids = np.concatenate([a_ids, b_ids], axis=1)
    sc = np.concatenate([a_sc, b_sc], axis=1)
    out_i = np.empty((ids.shape[0], k), dtype=np.int64)
    out_s = np.empty((ids.shape[0], k), dtype=np.float64)
    for p in range(ids.shape[0]):
        # sentinels (-inf, -1) sort last because real scores are finite
        order = np.lexsort((np.where(ids[p] < 0, np.iinfo(np.int64).max, ids[p]), -sc[p]))
        out_i[p] = ids[p, order[:k]]
        out_s[p] = sc[p, order[:k]]
    return out_i, out_s


def topk_streaming(P: np.ndarray, cache_chunks, k: int):
    """Tier-A top-k of prompts P [n, d] over an iterable of (first_gid, fp32 rows [m, d]) chunks
    (a cache too large to hold in fp64), merged with ``merge_topk``.  Invalid prompts get sentinels.
    Returns (ids [n, k], scores [n, k], valid [n])."""
    n = P.shape[0]
    ids = np.full((n, k), SENTINEL_GID, dtype=np.int64)
    sc = np.full((n, k), NEG_INF)
    valid = row_valid(P)
    Pv = np.where(valid[:, None], P, 1.0)
    for first, rows in cache_chunks:
        S = similarity_A(Pv, rows)
        gids = np.arange(first, first + rows.shape[0], dtype=np.int64)
        ci, cs = topk_prefiltered(S, gids, k)
        ids, sc = merge_topk(ids, sc, ci, cs, k)
    ids[~valid] = SENTINEL_GID
    sc[~valid] = NEG_INF
    return ids, sc, valid


# --------------------------------------------------------------------------------------
# O3 / O4  optimal-K and H_K
# --------------------------------------------------------------------------------------

def optimal_k_level(s1: np.ndarray, thresholds_f32, usable: np.ndarray) -> np.ndarray:
    """K_p = grid[#{m : s1_p >= t_m}] (R8, R9): the level index, 0 for cold / invalid (R16).

    S:163-171 select_optimal_k: bands closed below; none -> K = 0 (vanilla).
    """
    t = np.asarray(thresholds_f32, dtype=np.float32).astype(np.float64)
    lvl = np.zeros(len(s1), dtype=np.int64)
    for p in range(len(s1)):
        if usable[p]:
            lvl[p] = int(np.sum(s1[p] >= t))
    return lvl


def histogram(levels: np.ndarray, nK: int) -> np.ndarray:
    """h_i = #{p : K_p = grid[i]} (P:88 H_K, counts form, R4)."""
    return np.array([int(np.sum(levels == i)) for i in range(nK)], dtype=np.int64)


# --------------------------------------------------------------------------------------
# O5  targets: largest-remainder apportionment of N*F (R3)
# --------------------------------------------------------------------------------------

def apportion(F, N: int) -> np.ndarray:
    """f_j = floor(N F_j) plus one unit to each of the R = N - sum floor largest
    fractional parts, ties to the lower level index."""
    q = [float(N) * float(Fj) for Fj in F]
    f = [int(math.floor(v)) for v in q]
    frac = [q[j] - f[j] for j in range(len(q))]
    R = N - sum(f)
    order = sorted(range(len(q)), key=lambda j: (-frac[j], j))
    for j in order[:R]:
        f[j] += 1
    return np.array(f, dtype=np.int64)


# --------------------------------------------------------------------------------------
# O6 / O7  Eq. 1 route plan on integer counts
# --------------------------------------------------------------------------------------

def default_degradation(per_step: float = 0.006, length: int = T_TOTAL) -> np.ndarray:
    """c(dK) = 0.006 * dK (R6)."""
    return np.array([per_step * t for t in range(length)], dtype=np.float64)


def degradation_matrix(grid, c) -> np.ndarray:
    """D[i][j] = D(K'_j, K_i) = c(K_j - K_i) if K_j > K_i else 0 (Eq. 1 sums K'_j > K_i; R5)."""
    nK = len(grid)
    D = np.zeros((nK, nK), dtype=np.float64)
    for i in range(nK):
        for j in range(nK):
            if grid[j] > grid[i]:
                D[i, j] = c[grid[j] - grid[i]]
    return D


def d_q(x, grid, c, N: int) -> float:
    """Eq. 1 with H_K(K_i) = h_i/N and P(K'_j|K_i) = x_ij/h_i:  D_Q = sum_{K_j>K_i} x_ij D_ij / N."""
    if N == 0:
        return 0.0
    nK = len(grid)
    tot = 0.0
    for i in range(nK):
        for j in range(nK):
            if grid[j] > grid[i]:
                tot += float(x[i][j]) * float(c[grid[j] - grid[i]])
    return tot / N


def _plans(h, f):
    """Every non-negative integer matrix with row sums h and column sums f."""
    nK = len(h)

    def rows(i, colrem):
        if i == nK:
            if all(v == 0 for v in colrem):
                yield []
            return
        for row in _compositions(h[i], colrem):
            rest = [colrem[j] - row[j] for j in range(nK)]
            for tail in rows(i + 1, rest):
                yield [row] + tail

    yield from rows(0, list(f))


def _compositions(total, caps):
    if len(caps) == 1:
        if total <= caps[0]:
            yield [total]
        return
    for v in range(min(total, caps[0]) + 1):
        for rest in _compositions(total - v, caps[1:]):
            yield [v] + rest


D_TIE_REL = 1e-9   # D totals closer than this (relative) are equal: c is a real-valued
                   # loss given as doubles, so 0.006*1 + 0.006*3 vs 0.006*4 must tie (R7)


def plan_bruteforce(h, f, grid, c):
    """Exhaustive search (tiny N, nK <= 4): lexicographic min of (D, sum x dK^2) (R2, R7).

    D totals are summed exactly in rationals of the given doubles and compared with the
    relative tolerance D_TIE_REL; sum x dK^2 is an exact integer.
    Returns (x, number of plans sharing the optimal key).
    """
    nK = len(grid)
    Dfr = [[Fraction(0) if grid[j] <= grid[i] else Fraction(float(c[grid[j] - grid[i]]))
            for j in range(nK)] for i in range(nK)]
    plans = []
    for x in _plans([int(v) for v in h], [int(v) for v in f]):
        D = sum(x[i][j] * Dfr[i][j] for i in range(nK) for j in range(nK))
        Q = sum(x[i][j] * (grid[j] - grid[i]) ** 2 for i in range(nK) for j in range(nK))
        plans.append((D, Q, x))
    dmin = min(p[0] for p in plans)
    tol = Fraction(D_TIE_REL) * max(Fraction(1), dmin)
    near = [p for p in plans if p[0] - dmin <= tol]
    qmin = min(p[1] for p in near)
    best = [p for p in near if p[1] == qmin]
    return np.array(best[0][2], dtype=np.int64), len(best)


def plan_lp(h, f, grid, c):
    """Two-phase HiGHS LP on the transportation polytope (R2, R7):
    phase 1 min sum x_ij D_ij; phase 2 min sum x_ij (K_j-K_i)^2 s.t. sum x_ij D_ij <= D*.
    The constraint matrix is totally unimodular, so the optimal vertex is integral."""
    from scipy.optimize import linprog

    nK = len(grid)
    h = [int(v) for v in h]
    f = [int(v) for v in f]
    A_eq, b_eq = [], []
    for i in range(nK):
        row = np.zeros(nK * nK)
        row[i * nK:(i + 1) * nK] = 1
        A_eq.append(row)
        b_eq.append(h[i])
    for j in range(nK):
        col = np.zeros(nK * nK)
        col[j::nK] = 1
        A_eq.append(col)
        b_eq.append(f[j])
    A_eq = np.array(A_eq)
    b_eq = np.array(b_eq, dtype=np.float64)
    D = degradation_matrix(grid, c).reshape(-1)
    Q = np.array([(grid[j] - grid[i]) ** 2 for i in range(nK) for j in range(nK)], dtype=np.float64)
    r1 = linprog(D, A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    if r1.status != 0:
        raise RuntimeError(f"phase-1 LP failed: {r1.message}")
    dstar = float(r1.fun)
    r2 = linprog(Q, A_ub=D[None, :], b_ub=[dstar + D_TIE_REL * max(1.0, abs(dstar))],
                 A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    if r2.status != 0:
        raise RuntimeError(f"phase-2 LP failed: {r2.message}")
    x = np.rint(r2.x).astype(np.int64).reshape(nK, nK)
    if np.max(np.abs(r2.x - x.reshape(-1))) > 1e-6:
        raise RuntimeError("LP vertex not integral")
    if not (np.array_equal(x.sum(axis=1), h) and np.array_equal(x.sum(axis=0), f)):
        raise RuntimeError("LP plan violates the marginals")
    return x


# ----------------------------------------------------------------------------------------------
# O6' Eq. 1 for an arbitrary (non-convex) degradation table (R37; NEXT f4)
# ----------------------------------------------------------------------------------------------
DEG_SHIFT = 24   # R37: non-convex c is held as integers cI = round-half-even(c * 2^24)


def is_convex(c) -> bool:
    """R6: second differences >= -1e-12 (1 + |c_t|) -- the tables the NW-corner plan is exact for."""
    c = [float(v) for v in c]
    return all(c[t + 1] - 2 * c[t] + c[t - 1] >= -1e-12 * (1.0 + abs(c[t])) for t in range(1, len(c) - 1))


def degradation_int(c) -> np.ndarray:
    """cI = round-half-even(c * 2^24) (exact: scaling a double by 2^24 is exact, np.rint ties to even)."""
    return np.rint(np.ldexp(np.asarray(c, dtype=np.float64), DEG_SHIFT)).astype(np.int64)


def _cost_pairs(grid, cI):
    nK = len(grid)
    D = [[int(cI[grid[j] - grid[i]]) if grid[j] > grid[i] else 0 for j in range(nK)] for i in range(nK)]
    Q = [[(grid[j] - grid[i]) ** 2 for j in range(nK)] for i in range(nK)]
    return D, Q


def plan_int_bruteforce(h, f, grid, cI):
    """R37 by exhaustive search (tiny N, nK <= 4): min over all integer plans of the exact integer pair
    (sum x cI, sum x dK^2), then the lexicographically greatest x in row-major order.
    Returns (x, number of plans sharing the optimal pair)."""
    nK = len(grid)
    D, Q = _cost_pairs(grid, cI)
    best, best_key, ties = None, None, 0
    for x in _plans([int(v) for v in h], [int(v) for v in f]):
        d = sum(x[i][j] * D[i][j] for i in range(nK) for j in range(nK))
        q = sum(x[i][j] * Q[i][j] for i in range(nK) for j in range(nK))
        flat = [v for row in x for v in row]
        key = (d, q)
        if best is None or key < best_key:
            best, best_key, ties = flat, key, 1
        elif key == best_key:
            ties += 1
            if flat > best:
                best = flat
    return np.array(best, dtype=np.int64).reshape(nK, nK), ties


def plan_int_lp(h, f, grid, cI):
    """R37 by phased HiGHS LPs on the transportation polytope (integral vertices: total unimodularity).
    Phase 1 min sum x cI; phase 2 min sum x dK^2 over the phase-1 optimal face; phase 3 raises
    x_00, x_01, ... in row-major order, each to its maximum on the face with the earlier cells fixed.
    The optimal face of a phase is {x feasible : x_ij = 0 where the phase's reduced cost is > 0}
    (complementary slackness with an optimal dual; with integer data the reduced costs are integers,
    so > 0.5 decides).  Every objective coefficient is a small integer: no big-M, no D <= D* row."""
    from scipy.optimize import linprog

    nK = len(grid)
    h = [int(v) for v in h]
    f = [int(v) for v in f]
    A_eq = np.zeros((2 * nK, nK * nK))
    for i in range(nK):
        A_eq[i, i * nK:(i + 1) * nK] = 1
    for j in range(nK):
        A_eq[nK + j, j::nK] = 1
    b_eq = np.array(h + f, dtype=np.float64)
    D, Q = _cost_pairs(grid, cI)
    ub = [None] * (nK * nK)

    def solve(cost):
        r = linprog(np.asarray(cost, dtype=np.float64), A_eq=A_eq, b_eq=b_eq,
                    bounds=[(0, u) for u in ub], method="highs")
        if r.status != 0:
            raise RuntimeError(f"LP failed: {r.message}")
        return r

    for cost in ([v for row in D for v in row], [v for row in Q for v in row]):
        r = solve(cost)
        rc = r.lower.marginals           # reduced costs of x >= 0
        for e in range(nK * nK):
            if rc[e] > 0.5:
                ub[e] = 0.0
    lo = [0.0] * (nK * nK)
    for e in range(nK * nK):
        if ub[e] == 0.0:
            continue
        obj = np.zeros(nK * nK)
        obj[e] = -1.0
        r = linprog(obj, A_eq=A_eq, b_eq=b_eq, bounds=list(zip(lo, ub)), method="highs")
        if r.status != 0:
            raise RuntimeError(f"phase-3 LP failed: {r.message}")
        v = float(np.rint(-r.fun))
        if abs(-r.fun - v) > 1e-6:
            raise RuntimeError("phase-3 optimum not integral")
        lo[e] = v
        ub[e] = v
    x = np.array([int(v) for v in lo], dtype=np.int64).reshape(nK, nK)
    if not (np.array_equal(x.sum(axis=1), h) and np.array_equal(x.sum(axis=0), f)):
        raise RuntimeError("plan violates the marginals")
    return x


def plan_for(h, f, grid, c, solver: str = "lp"):
    """The plan the hot path must produce for table c: R7 (convex c) or R37 (any other table)."""
    if is_convex(c):
        return plan_bruteforce(h, f, grid, c)[0] if solver == "brute" else plan_lp(h, f, grid, c)
    cI = degradation_int(c)
    return plan_int_bruteforce(h, f, grid, cI)[0] if solver == "brute" else plan_int_lp(h, f, grid, cI)


def dq_linear_closed_form(h, f, grid, alpha: float, N: int) -> float:
    """For D = alpha * dK (linear), D*/N = alpha * sum_t (K_{t+1}-K_t) max(0, CDF_h(t) - CDF_f(t)) / N:
    every prompt whose level is <= t but is served above t crosses the gap (K_t, K_{t+1})."""
    cum_h = np.cumsum(h)
    cum_f = np.cumsum(f)
    tot = 0.0
    for t in range(len(grid) - 1):
        tot += (grid[t + 1] - grid[t]) * max(0, int(cum_h[t]) - int(cum_f[t]))
    return alpha * tot / N if N else 0.0


def dq_continuous(Hfrac, F, grid, c) -> float:
    """D_Q_LP: Eq. 1 optimum on the unrounded masses (H = h/N, F) via the LP (context only)."""
    from scipy.optimize import linprog

    nK = len(grid)
    A_eq, b_eq = [], []
    for i in range(nK):
        row = np.zeros(nK * nK)
        row[i * nK:(i + 1) * nK] = 1
        A_eq.append(row)
        b_eq.append(Hfrac[i])
    for j in range(nK):
        col = np.zeros(nK * nK)
        col[j::nK] = 1
        A_eq.append(col)
        b_eq.append(F[j])
    D = degradation_matrix(grid, c).reshape(-1)
    r = linprog(D, A_eq=np.array(A_eq), b_eq=np.array(b_eq), bounds=(0, None), method="highs")
    return float(r.fun)


# --------------------------------------------------------------------------------------
# O8  redirection by rank within optimal-K class
# --------------------------------------------------------------------------------------

def redirect(levels: np.ndarray, x: np.ndarray, seed: int, batch_seq: int):
    """K'_p from the Route-Plan (R3, R18).

    key_p = (class_p << 60) | kappa_p; all prompts ordered by (key_p, p); rank_p is the
    position minus the number of prompts in lower classes; K'_p = grid[j] with
    X_i[j-1] <= rank_p < X_i[j], X_i the prefix sums of row i of x.
    Returns (K' level index per prompt, rank within class).
    """
    n = len(levels)
    nK = x.shape[0]
    kappa = philox.redirect_keys(n, seed, batch_seq)
    key = (levels.astype(np.uint64) << np.uint64(60)) | kappa
    order = np.lexsort((np.arange(n), key))       # by key, then prompt index
    position = np.empty(n, dtype=np.int64)
    position[order] = np.arange(n)
    h = np.array([int(np.sum(levels == i)) for i in range(nK)])
    class_start = np.concatenate([[0], np.cumsum(h)[:-1]])
    rank = position - class_start[levels]
    kp = np.empty(n, dtype=np.int64)
    for p in range(n):
        i = levels[p]
        X = np.cumsum(x[i])
        kp[p] = int(np.searchsorted(X, rank[p], side="right"))
    return kp, rank


# --------------------------------------------------------------------------------------
# O9 / O10  route-and-batch and buckets
# --------------------------------------------------------------------------------------

GREEDY = 0
UNIFORM = 1


def instance_lists(instance_level, nK: int):
    """I_j: ascending ids of the serving instances at level j (P:74 'GPU workers' at K; R12)."""
    return [[w for w, lv in enumerate(instance_level) if lv == j] for j in range(nK)]


def route_and_batch(kp: np.ndarray, instance_level, bstar: int, mode: int,
                    seed: int, batch_seq: int):
    """Instance and slot per prompt (R13, R14).

    Greedy: t_p = #{p' < p : K'_p' = K'_p}; instance = I_j[(t div b*) mod n_j];
            slot = (t div (b* n_j)) b* + t mod b*.
    Uniform: u = w0 of Philox stream 2; instance = I_j[(u n_j) >> 32];
             slot = #{p' < p : instance_p' = instance_p}.
    """
    n = len(kp)
    nK = int(max(kp.max() + 1 if n else 0, max(instance_level) + 1))
    I = instance_lists(instance_level, nK)
    inst = np.empty(n, dtype=np.int64)
    slot = np.empty(n, dtype=np.int64)
    if mode == GREEDY:
        seen = {}
        for p in range(n):
            j = int(kp[p])
            t = seen.get(j, 0)
            seen[j] = t + 1
            nj = len(I[j])
            inst[p] = I[j][(t // bstar) % nj]
            slot[p] = (t // (bstar * nj)) * bstar + t % bstar
    else:
        u = philox.uniform_words(n, seed, batch_seq)
        seen = {}
        for p in range(n):
            j = int(kp[p])
            nj = len(I[j])
            w = I[j][(int(u[p]) * nj) >> 32]
            inst[p] = w
            slot[p] = seen.get(w, 0)
            seen[w] = slot[p] + 1
    return inst, slot


def buckets(inst: np.ndarray, slot: np.ndarray, W: int):
    """Per-instance FIFO lists: offsets = exclusive scan of counts; prompts in slot order."""
    counts = np.array([int(np.sum(inst == w)) for w in range(W)], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    prompts = np.full(len(inst), -1, dtype=np.int64)
    for p in range(len(inst)):
        prompts[offsets[inst[p]] + slot[p]] = p
    return offsets, prompts


# --------------------------------------------------------------------------------------
# composite
# --------------------------------------------------------------------------------------

@dataclass
class Setup:
    """Controller inputs for one batch (the hot path takes them as given)."""
    grid: list                      # K values, strictly increasing, grid[0] == 0
    thresholds: list                # nK-1 fp32 similarity thresholds, increasing
    F: list                         # per-level load fractions, sum 1
    instance_level: list            # level index of each serving instance
    bstar: int = 4
    mode: int = GREEDY
    c: np.ndarray = field(default_factory=default_degradation)
    topk: int = 8
    seed: int = 0x5EED2502
    batch_seq: int = 0


@dataclass
class Result:
    topk_id: np.ndarray
    topk_score: np.ndarray
    level: np.ndarray
    K: np.ndarray
    h: np.ndarray
    f: np.ndarray
    x: np.ndarray
    D_Q: float
    level_prime: np.ndarray
    K_prime: np.ndarray
    rank: np.ndarray
    instance: np.ndarray
    slot: np.ndarray
    offsets: np.ndarray
    bucket_prompts: np.ndarray
    valid: np.ndarray
    flags: np.ndarray


def downstream(level: np.ndarray, s: Setup, solver: str = "lp"):
    """O4..O10 from a vector of optimal-K level indices (used directly, or teacher-forced on
    the GPU's K vector when a flagged near-tie flips a K)."""
    N = len(level)
    nK = len(s.grid)
    h = histogram(level, nK)
    f = apportion(s.F, N)
    if N == 0:
        x = np.zeros((nK, nK), dtype=np.int64)
    else:
        x = plan_for(h, f, s.grid, s.c, solver)
    DQ = d_q(x, s.grid, s.c, N)
    kp, rank = redirect(level, x, s.seed, s.batch_seq) if N else (np.zeros(0, np.int64),) * 2
    inst, slot = route_and_batch(kp, s.instance_level, s.bstar, s.mode, s.seed, s.batch_seq)
    offsets, bp = buckets(inst, slot, len(s.instance_level))
    return dict(h=h, f=f, x=x, D_Q=DQ, level_prime=kp, rank=rank, instance=inst, slot=slot,
                offsets=offsets, bucket_prompts=bp)


def tier_a_flags(sc: np.ndarray, s1_next: np.ndarray, thresholds, valid, cold: bool):
    """Oracle-side near-tie flags on Tier A scores (north_star: margins below 2e-2 are
    reported, not failed): 4 = top-1 vs top-2 margin < 2e-2; 8 = s1 within 2e-2 of a threshold."""
    n = sc.shape[0]
    flags = np.zeros(n, dtype=np.int64)
    t = np.asarray(thresholds, dtype=np.float32).astype(np.float64)
    for p in range(n):
        if not valid[p]:
            flags[p] |= FLAG_INVALID
            continue
        if cold:
            flags[p] |= FLAG_COLD
            continue
        s1 = sc[p, 0]
        s2 = sc[p, 1] if sc.shape[1] > 1 else s1_next[p]
        if np.isfinite(s2) and s1 - s2 < NEAR_MARGIN:
            flags[p] |= FLAG_NEAR_TOP1
        if len(t) and np.min(np.abs(s1 - t)) < NEAR_MARGIN:
            flags[p] |= FLAG_NEAR_THRESHOLD
    return flags


def route(P: np.ndarray, C: np.ndarray, s: Setup, solver: str = "lp") -> Result:
    """The whole batch on Tier A similarity (O1..O10), small inputs (full score matrix)."""
    N = P.shape[0]
    M = C.shape[0]
    valid = row_valid(P)
    k = s.topk
    if M == 0:
        ids = np.full((N, k), SENTINEL_GID, dtype=np.int64)
        sc = np.full((N, k), NEG_INF)
        nxt = np.full(N, NEG_INF)
    else:
        if not np.all(row_valid(C)):
            raise ValueError("cache rows must be valid")
        S = similarity_A(np.where(valid[:, None], P, 1.0), C)
        gids = np.arange(M, dtype=np.int64)
        ids, sc = topk_sorted(S, gids, k)
        ids2, sc2 = topk_sorted(S, gids, k + 1)
        nxt = sc2[:, k]
        ids[~valid] = SENTINEL_GID
        sc[~valid] = NEG_INF
    usable = valid & (M > 0)
    level = optimal_k_level(sc[:, 0], s.thresholds, usable)
    flags = tier_a_flags(sc, nxt, s.thresholds, valid, M == 0)
    d = downstream(level, s, solver)
    grid = np.asarray(s.grid)
    return Result(topk_id=ids, topk_score=sc, level=level, K=grid[level],
                  h=d["h"], f=d["f"], x=d["x"], D_Q=d["D_Q"],
                  level_prime=d["level_prime"], K_prime=grid[d["level_prime"]], rank=d["rank"],
                  instance=d["instance"], slot=d["slot"], offsets=d["offsets"],
                  bucket_prompts=d["bucket_prompts"], valid=valid, flags=flags)
