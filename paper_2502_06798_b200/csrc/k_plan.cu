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
#include "pas_internal.cuh"

namespace pas {
namespace {

__device__ __forceinline__ double warp_sum_fixed(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(32) k_plan(const int* __restrict__ hist, const RouteParams P,
                                             DevPlan* __restrict__ plan) {
  pdl_entry();
  __shared__ int h_s[kMaxLevels], f_s[kMaxLevels], hc[kMaxLevels + 1], fc[kMaxLevels + 1];
  __shared__ double frac_s[kMaxLevels];
  const int lane = threadIdx.x;
  const int nK = P.nK;
  const int N = (int)P.N;
  // ---- O5 largest remainder apportionment of N*F
  int fl = 0;
  double frac = -1.0;
  if (lane < nK) {
    h_s[lane] = hist[lane];
    const double q = __dmul_rn((double)N, P.F[lane]);
    const double f0 = floor(q);
    fl = (int)f0;
    frac = __dsub_rn(q, f0);
    frac_s[lane] = frac;
  }
  const int R = N - warp_sum(lane < nK ? fl : 0);
  __syncwarp();
  if (lane < nK) {
    int rank = 0;
    for (int j = 0; j < nK; ++j) rank += (frac_s[j] > frac || (frac_s[j] == frac && j < lane)) ? 1 : 0;
    f_s[lane] = fl + (rank < R ? 1 : 0);
  }
  __syncwarp();
  if (lane == 0) {   // cumulative sums (<= 16 terms)
    hc[0] = 0;
    fc[0] = 0;
    for (int i = 0; i < nK; ++i) {
      hc[i + 1] = hc[i] + h_s[i];
      fc[i + 1] = fc[i] + f_s[i];
    }
  }
  __syncwarp();
  // ---- O6 NW-corner coupling in closed form, O7 D_Q and counters
  double dq = 0.0, lp = 0.0;
  int n_red = 0, n_up = 0, n_down = 0;
  const double invN = N > 0 ? __ddiv_rn(1.0, (double)N) : 0.0;
  for (int e = lane; e < nK * nK; e += 32) {
    const int i = e / nK, j = e % nK;
    const int lo = max(hc[i], fc[j]), hi = min(hc[i + 1], fc[j + 1]);
    const int x = hi > lo ? hi - lo : 0;
    plan->x[i][j] = x;
    if (j != i) n_red += x;
    if (j < i) n_up += x;
    if (j > i) {
      n_down += x;
      dq = __dadd_rn(dq, __dmul_rn((double)x, P.c[P.grid[j] - P.grid[i]]));
    }
    // D_Q_LP: the same monotone coupling on the unrounded masses (h/N, F), context only
    double hlo = __dmul_rn((double)hc[i], invN), hhi = __dmul_rn((double)hc[i + 1], invN);
    double flo = 0.0, fhi = 0.0;
    for (int jj = 0; jj < j; ++jj) flo = __dadd_rn(flo, P.F[jj]);
    fhi = __dadd_rn(flo, P.F[j]);
    const double ov = fmin(hhi, fhi) - fmax(hlo, flo);
    if (j > i && ov > 0) lp = __dadd_rn(lp, __dmul_rn(ov, P.c[P.grid[j] - P.grid[i]]));
  }
  dq = warp_sum_fixed(dq);
  lp = warp_sum_fixed(lp);
  n_red = warp_sum(n_red);
  n_up = warp_sum(n_up);
  n_down = warp_sum(n_down);
  __syncwarp();
  if (lane < nK) {   // row prefix tables and class starts
    const int i = lane;
    plan->h[i] = h_s[i];
    plan->f[i] = f_s[i];
    plan->class_start[i] = hc[i];
    int acc = 0;
    for (int j = 0; j < nK; ++j) {
      const int lo = max(hc[i], fc[j]), hi = min(hc[i + 1], fc[j + 1]);
      acc += hi > lo ? hi - lo : 0;
      plan->X[i][j] = acc;
    }
    // I_j: ascending instance ids at level j, and the multiply-high constant for div n_j
    int n = 0;
    for (int w = 0; w < P.W; ++w)
      if (P.inst_level[w] == i) plan->inst_list[i][n++] = w;
    plan->n_inst[i] = n;
    const uint64_t d = n > 0 ? (uint64_t)n : 1;
    plan->n_inst_magic[i] = ((1ull << 32) + d - 1) / d;
  }
  if (lane == 0) {
    plan->class_start[nK] = hc[nK];
    plan->D_Q = N > 0 ? __ddiv_rn(dq, (double)N) : 0.0;
    plan->D_Q_LP = lp;
    plan->n_redirected = n_red;
    plan->n_upgraded = n_up;
    plan->n_downgraded = n_down;
  }
}

}  // namespace

cudaError_t launch_plan(const int* hist, const RouteParams& p, DevPlan* plan, cudaStream_t st) {
  launch_pdl(k_plan, 1, 32, 0, st, hist, p, plan);
  return cudaGetLastError();
}

}  // namespace pas
