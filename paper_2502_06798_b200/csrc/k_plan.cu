// K5 -- Eq. 1 K->K' route plan for one batch, solved in one CTA.
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
// nK <= 16: one thread does the arithmetic (fp64 with explicit _rn intrinsics, no FMA contraction,
// so f is bit-identical to the CPU).  Also builds the row prefix tables X, the class starts, the
// per-level instance lists I_j (ascending ids) and the redirect counters.
#include "pas_internal.cuh"

namespace pas {
namespace {

__global__ void k_plan(const int* __restrict__ hist, const RouteParams P, DevPlan* __restrict__ plan) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int nK = P.nK;
  const int N = (int)P.N;
  int h[kMaxLevels], f[kMaxLevels];
  for (int i = 0; i < nK; ++i) h[i] = hist[i];
  // ---- O5 largest remainder apportionment of N*F
  double frac[kMaxLevels];
  int sumf = 0;
  for (int j = 0; j < nK; ++j) {
    const double q = __dmul_rn((double)N, P.F[j]);
    const double fl = floor(q);
    f[j] = (int)fl;
    frac[j] = __dsub_rn(q, fl);
    sumf += f[j];
  }
  int R = N - sumf;
  bool used[kMaxLevels];
  for (int j = 0; j < nK; ++j) used[j] = false;
  for (int r = 0; r < R; ++r) {
    int best = -1;
    for (int j = 0; j < nK; ++j)
      if (!used[j] && (best < 0 || frac[j] > frac[best])) best = j;   // ties -> lower index
    used[best] = true;
    f[best] += 1;
  }
  // ---- O6 north-west-corner integer transport (monotone coupling)
  int x[kMaxLevels][kMaxLevels];
  for (int i = 0; i < nK; ++i)
    for (int j = 0; j < nK; ++j) x[i][j] = 0;
  {
    int rem_r[kMaxLevels], rem_c[kMaxLevels];
    for (int i = 0; i < nK; ++i) { rem_r[i] = h[i]; rem_c[i] = f[i]; }
    int i = 0, j = 0;
    while (i < nK && j < nK) {
      if (rem_r[i] == 0) { ++i; continue; }
      if (rem_c[j] == 0) { ++j; continue; }
      const int t = rem_r[i] < rem_c[j] ? rem_r[i] : rem_c[j];
      x[i][j] += t;
      rem_r[i] -= t;
      rem_c[j] -= t;
    }
  }
  // ---- O7 D_Q (Eq. 1 on counts), in (i, j) order
  double dq = 0.0;
  int n_red = 0, n_up = 0, n_down = 0;
  for (int i = 0; i < nK; ++i)
    for (int j = 0; j < nK; ++j) {
      if (j != i) n_red += x[i][j];
      if (j < i) n_up += x[i][j];
      if (j > i) {
        n_down += x[i][j];
        dq = __dadd_rn(dq, __dmul_rn((double)x[i][j], P.c[P.grid[j] - P.grid[i]]));
      }
    }
  plan->D_Q = N > 0 ? __ddiv_rn(dq, (double)N) : 0.0;
  // ---- D_Q_LP: same monotone coupling on the unrounded masses (h/N, F), context only
  {
    double rr[kMaxLevels], rc[kMaxLevels];
    for (int i = 0; i < nK; ++i) { rr[i] = N > 0 ? __ddiv_rn((double)h[i], (double)N) : 0.0; rc[i] = P.F[i]; }
    int i = 0, j = 0;
    double lp = 0.0;
    while (i < nK && j < nK) {
      if (rr[i] <= 1e-15) { ++i; continue; }
      if (rc[j] <= 1e-15) { ++j; continue; }
      const double t = rr[i] < rc[j] ? rr[i] : rc[j];
      if (j > i) lp = __dadd_rn(lp, __dmul_rn(t, P.c[P.grid[j] - P.grid[i]]));
      rr[i] = __dsub_rn(rr[i], t);
      rc[j] = __dsub_rn(rc[j], t);
    }
    plan->D_Q_LP = lp;
  }
  int cs = 0;
  for (int i = 0; i < nK; ++i) {
    plan->h[i] = h[i];
    plan->f[i] = f[i];
    plan->class_start[i] = cs;
    cs += h[i];
    int acc = 0;
    for (int j = 0; j < nK; ++j) {
      plan->x[i][j] = x[i][j];
      acc += x[i][j];
      plan->X[i][j] = acc;
    }
  }
  plan->class_start[nK] = cs;
  plan->n_redirected = n_red;
  plan->n_upgraded = n_up;
  plan->n_downgraded = n_down;
  // ---- I_j: ascending instance ids per level
  for (int j = 0; j < nK; ++j) plan->n_inst[j] = 0;
  for (int w = 0; w < P.W; ++w) {
    const int j = P.inst_level[w];
    plan->inst_list[j][plan->n_inst[j]++] = w;
  }
  for (int j = 0; j < nK; ++j) {
    const uint64_t d = plan->n_inst[j] > 0 ? (uint64_t)plan->n_inst[j] : 1;
    plan->n_inst_magic[j] = ((1ull << 32) + d - 1) / d;
  }
}

}  // namespace

cudaError_t launch_plan(const int* hist, const RouteParams& p, DevPlan* plan, cudaStream_t st) {
  k_plan<<<1, 32, 0, st>>>(hist, p, plan);
  return cudaGetLastError();
}

}  // namespace pas
