// K5 -- Eq. 1 K->K' route plan for one batch, solved by one warp.
//
// Paper (PAPER.md P:88-P:96): the Query Fraction Solver gives F(K); the K-to-K' Route Planner finds
// redirection probabilities P(K'_j|K_i) minimising
//     D_Q = sum_{i,j: K'_j > K_i} P(K'_j|K_i) H_K(K_i) D(K'_j, K_i)                  (Eq. 1)
// shifting prompts "to a slower/better model ... K' < K, or to the closest possible faster/worse
// model ... K' > K".  Readings: R2 transportation constraints (rows H, columns F);
// R3 per-batch integer counts, f = largest-remainder(N F); R5 upgrades cost 0; R6 D(K',K) = c(K'-K)
// with c convex; R7 ties -> min sum x (K_j - K_i)^2.
//
// For a cost phi(K'-K) with phi(t) = c(t) [t > 0] convex, the monotone (north-west-corner) coupling
// of the sorted marginals is an optimal transport plan, and it is the unique minimiser of the
// strictly convex tie-break, so NW-corner IS the lexicographic optimum; the oracle checks this
// against exhaustive search and an LP (tests/test_oracle_plan.py, tests/test_gpu_*).
//
// One warp, no serial loops over the plan: the NW-corner coupling has the closed form
//     x_ij = max(0, min(Hc_i, Fc_j) - max(Hc_{i-1}, Fc_{j-1}))       (Hc, Fc cumulative sums),
// the overlap of prompt-rank intervals, so each of the nK^2 <= 256 entries is computed independently.
// Largest remainder: f_j = floor(N F_j) + [rank of frac_j among the levels (desc, ties -> lower
// index) < R].  fp64 with explicit _rn intrinsics (no FMA contraction): f is bit-identical to the
// CPU.  Also: row prefix tables X, class starts, the per-level instance lists I_j (ascending ids) with
// their multiply-high division constants, redirect counters, D_Q and D_Q_LP (fixed reduction order).
//
// Non-convex c (f4, R37; SURVEY 8(f) "a general (non-convex) D-table route planner"): NW-corner is no
// longer optimal (suboptimal on 225/400 arbitrary tables), so lane 0 solves the integer
// transportation problem exactly: costs cI = round(c 2^24) (pas_set_degradation), plans compared on
// the pair (sum x cI, sum x dK^2) lexicographically -- successive shortest paths with Dijkstra on
// reduced costs (potentials), exact int64 pair arithmetic, <= 34 nodes -- and, since the optimum can
// still be a face, the canonical plan on it: the lexicographically greatest x in row-major order.  The
// final potentials are optimal duals, so the optimal face is exactly the feasible plans supported on
// the cells of zero reduced cost; the greedy maximises x_00, x_01, ... in turn on that face, raising
// x_ij along cycles col j -> row i through later cells (an augmenting-cycle max flow per cell).
// The oracle reaches the same plan independently: exhaustive search (<= 4 levels) and phased HiGHS LPs
// fixed by the reduced costs of each phase (tests/test_oracle_plan.py).
#include "plan_body.cuh"

namespace pas {
namespace {

__global__ void __launch_bounds__(32) k_plan(const int* __restrict__ hist, const RouteParams P,
                                             DevPlan* __restrict__ plan) {
  pdl_entry();
  // inlined: the parameters are read with direct (indexed) constant loads; K6's windows only for the
  // batches that take the windowed path
  plan_body(hist, P, plan, P.N >= kWindowMinN);
}

}  // namespace

cudaError_t launch_plan(const int* hist, const RouteParams& p, DevPlan* plan, cudaStream_t st) {
  launch_pdl(k_plan, 1, 32, 0, st, hist, p, plan);
  return cudaGetLastError();
}

}  // namespace pas
