// plan_body.cuh -- K5's Eq. 1 route plan for one batch, executed by one warp: largest-remainder
// targets f, the plan x (NW-corner closed form for convex c; the exact min-cost solver of R37
// otherwise), D_Q, D_Q_LP, counters, prefix tables and instance lists into a DevPlan.  Shared by the
// K5 kernel (k_plan.cu) and the fused small-batch kernel (k_small.cu).  Readings and the algorithm's
// description: the head of k_plan.cu.
#pragma once
#include "pas_internal.cuh"

namespace pas {
namespace {

// (D, Q) cost pair, compared lexicographically
struct Cost2 {
  long long d, q;
};
__device__ __forceinline__ bool lt(const Cost2& a, const Cost2& b) { return a.d < b.d || (a.d == b.d && a.q < b.q); }
__device__ __forceinline__ Cost2 add(const Cost2& a, const Cost2& b) { return {a.d + b.d, a.q + b.q}; }
__device__ __forceinline__ Cost2 sub(const Cost2& a, const Cost2& b) { return {a.d - b.d, a.q - b.q}; }
__device__ __forceinline__ bool is_zero(const Cost2& a) { return a.d == 0 && a.q == 0; }

constexpr long long kInfD = (long long)1 << 62;

// Exact lexicographic min-cost transportation plan (R37) for rows h, columns f (sum h == sum f),
// unit cost of cell (i, j) = (cI[K_j - K_i] if K_j > K_i else 0, (K_j - K_i)^2); then the
// lexicographically greatest optimal x in row-major order.  One thread; x in shared memory.  Returns
// the number of augmentations, or -1 if the iteration cap was hit (x is then feasible, not canonical).
__device__ __forceinline__ int mcf_plan(const int* h, const int* f, const RouteParams& P, int (*x)[kMaxLevels]) {
  const int nK = P.nK;
  const int V = 2 * nK + 2, S = 0, T = 2 * nK + 1;   // S, rows 1..nK, cols nK+1..2nK, T
  // working arrays in shared memory (one thread runs the solver; no per-thread stack frame)
  __shared__ Cost2 C[kMaxLevels][kMaxLevels];
#pragma unroll 1
  for (int i = 0; i < nK; ++i)
#pragma unroll 1
    for (int j = 0; j < nK; ++j) {
      const int dk = P.grid[j] - P.grid[i];
      C[i][j] = {dk > 0 ? P.cI[dk] : 0, (long long)dk * dk};
      x[i][j] = 0;
    }
  __shared__ int rs[kMaxLevels], rd[kMaxLevels];
#pragma unroll 1
  for (int i = 0; i < nK; ++i) {
    rs[i] = h[i];
    rd[i] = f[i];
  }
  __shared__ Cost2 pot[2 * kMaxLevels + 2], dist[2 * kMaxLevels + 2];
  __shared__ int prev[2 * kMaxLevels + 2];
  __shared__ bool done[2 * kMaxLevels + 2];
#pragma unroll 1
  for (int v = 0; v < V; ++v) pot[v] = {0, 0};
  int iters = 0;
  const int cap = 64 * nK * nK + 64;
  int left = 0;
#pragma unroll 1
  for (int i = 0; i < nK; ++i) left += rs[i];
  // residual capacity of edge u -> v (0 = absent); cost of u -> v
  auto rcap = [&](int u, int v) -> long long {
    if (u == S && v >= 1 && v <= nK) return rs[v - 1];
    if (v == S && u >= 1 && u <= nK) return h[u - 1] - rs[u - 1];
    if (u >= 1 && u <= nK && v > nK && v < T) return kInfD;
    if (u > nK && u < T && v >= 1 && v <= nK) return x[v - 1][u - nK - 1];
    if (u > nK && u < T && v == T) return rd[u - nK - 1];
    if (u == T && v > nK && v < T) return f[v - nK - 1] - rd[v - nK - 1];
    return 0;
  };
  auto cost = [&](int u, int v) -> Cost2 {
    if (u >= 1 && u <= nK && v > nK && v < T) return C[u - 1][v - nK - 1];
    if (u > nK && u < T && v >= 1 && v <= nK) return Cost2{-C[v - 1][u - nK - 1].d, -C[v - 1][u - nK - 1].q};
    return Cost2{0, 0};
  };
  while (left > 0) {
    if (++iters > cap) return -1;
#pragma unroll 1
    for (int v = 0; v < V; ++v) {
      dist[v] = {kInfD, 0};
      done[v] = false;
      prev[v] = -1;
    }
    dist[S] = {0, 0};
#pragma unroll 1
    for (int it = 0; it < V; ++it) {   // dense Dijkstra on reduced costs (all >= 0)
      int u = -1;
#pragma unroll 1
      for (int v = 0; v < V; ++v)
        if (!done[v] && dist[v].d < kInfD && (u < 0 || lt(dist[v], dist[u]))) u = v;
      if (u < 0) break;
      done[u] = true;
#pragma unroll 1
      for (int v = 0; v < V; ++v) {
        if (done[v] || rcap(u, v) <= 0) continue;
        const Cost2 nd = add(dist[u], sub(add(cost(u, v), pot[u]), pot[v]));
        if (dist[v].d >= kInfD || lt(nd, dist[v])) {
          dist[v] = nd;
          prev[v] = u;
        }
      }
    }
    if (dist[T].d >= kInfD) return -1;   // cannot happen: every cell is open
#pragma unroll 1
    for (int v = 0; v < V; ++v) pot[v] = add(pot[v], (dist[v].d < kInfD && lt(dist[v], dist[T])) ? dist[v] : dist[T]);
    long long b = kInfD;
#pragma unroll 1
    for (int v = T; v != S; v = prev[v]) {
      const long long c = rcap(prev[v], v);
      b = c < b ? c : b;
    }
#pragma unroll 1
    for (int v = T; v != S; v = prev[v]) {
      const int u = prev[v];
      if (u == S) rs[v - 1] -= (int)b;
      else if (v == T) rd[u - nK - 1] -= (int)b;
      else if (u <= nK) x[u - 1][v - nK - 1] += (int)b;   // row -> col: more on the cell
      else x[v - 1][u - nK - 1] -= (int)b;                // col -> row: less on the cell
    }
    left -= (int)b;
  }
  // optimal face: cells with zero reduced cost under the final potentials (optimal duals)
  __shared__ bool tight[kMaxLevels][kMaxLevels];
#pragma unroll 1
  for (int i = 0; i < nK; ++i)
#pragma unroll 1
    for (int j = 0; j < nK; ++j) tight[i][j] = is_zero(sub(add(C[i][j], pot[1 + i]), pot[1 + nK + j]));
  // lexicographically greatest x in row-major order on the face: raise x_ij along cycles
  // row i -> col j -> row r (lower a later cell (r, j)) -> col c (raise a later tight (r, c)) -> ... -> row i
  __shared__ int q[2 * kMaxLevels], from[2 * kMaxLevels];
#pragma unroll 1
  for (int e = 0; e < nK * nK; ++e) {
    const int i = e / nK, j = e % nK;
    if (!tight[i][j]) continue;
#pragma unroll 1
    for (;;) {
      if (++iters > cap) return -1;
      // BFS over nodes: rows 0..nK-1, cols nK..2nK-1; start at col j, target row i
#pragma unroll 1
      for (int v = 0; v < 2 * nK; ++v) from[v] = -2;
      int qh = 0, qt = 0;
      q[qt++] = nK + j;
      from[nK + j] = -1;
      bool found = false;
      while (qh < qt && !found) {
        const int u = q[qh++];
        if (u >= nK) {   // col c: lower a later cell (r, c) with x > 0
          const int c = u - nK;
#pragma unroll 1
          for (int r = 0; r < nK; ++r)
            if (from[r] == -2 && r * nK + c > e && x[r][c] > 0) {
              from[r] = u;
              q[qt++] = r;
              if (r == i) {
                found = true;
                break;
              }
            }
        } else {         // row r: raise a later tight cell (r, c)
          const int r = u;
#pragma unroll 1
          for (int c = 0; c < nK; ++c)
            if (from[nK + c] == -2 && r * nK + c > e && tight[r][c]) {
              from[nK + c] = u;
              q[qt++] = nK + c;
            }
        }
      }
      if (!found) break;
      long long b = kInfD;
#pragma unroll 1
      for (int v = i; from[v] != -1; v = from[v]) {
        const int u = from[v];
        if (u >= nK) {   // col u -> row v: lowered cell (v, u - nK)
          const long long c = x[v][u - nK];
          b = c < b ? c : b;
        }
      }
#pragma unroll 1
      for (int v = i; from[v] != -1; v = from[v]) {
        const int u = from[v];
        if (u >= nK) x[v][u - nK] -= (int)b;   // lowered
        else x[u][v - nK] += (int)b;           // raised (row u -> col v)
      }
      x[i][j] += (int)b;
    }
  }
  return iters;
}

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


// K6's windows (DevPlan comment in pas_internal.cuh): per class the distinct split ranks 0 < X < h_i of
// the prefix row X_i (K' level of class rank r = #{j : X_i[j] <= r}), the window of the X-th smallest
// of h_i uniform kappas (Beta(X + 1, h - X): mean +- 8 sd, +- 2 / h slack) in units of 2^-60, merged
// into zones; list capacities (2x the expected entries + 1024, within N) and bases.  One thread.
__device__ __forceinline__ void k6_zones(const int* h_s, const int (*x)[kMaxLevels], const RouteParams& P,
                                      DevPlan* __restrict__ plan) {
  const int nK = P.nK;
  const double two60 = 1152921504606846976.0;   // 2^60
  int nz = 0, ns = 0, slot = 0;
  int64_t used = 0;
  bool fallback = false;
#pragma unroll 1
  for (int i = 0; i < nK; ++i) {
    const int h = h_s[i];
    plan->cls_zone0[i] = nz;
    plan->cls_slot0[i] = slot;
    int jb = 0, X = 0, lastX = -1, zc = -1;
#pragma unroll 1
    for (int j = 0; j + 1 < nK; ++j) {
      X += x[i][j];
      if (X <= 0) {        // every class prompt has rank >= 0
        ++jb;
        continue;
      }
      if (X >= h) continue;  // no prompt of the class reaches it
      if (X == lastX) {      // the same split rank again (x_ij == 0): one more level boundary there
        ++plan->s_mult[ns - 1];
        continue;
      }
      if (ns == kMaxZones) {
        fallback = true;
        continue;
      }
      const double mu = ((double)X + 1.0) / ((double)h + 1.0);
      const double sd = sqrt(mu * (1.0 - mu) / ((double)h + 2.0));
      const double lo = mu - 8.0 * sd - 2.0 / h, hi = mu + 8.0 * sd + 2.0 / h;
      const uint64_t lo_k = lo <= 0.0 ? 0ull : (uint64_t)(lo * two60);
      const uint64_t hi_k = hi >= 1.0 ? (1ull << 60) : (uint64_t)(hi * two60) + 1ull;
      if (zc >= 0 && lo_k <= plan->z_hi[zc]) {   // overlaps the previous window of the class: merge
        plan->z_hi[zc] = hi_k > plan->z_hi[zc] ? hi_k : plan->z_hi[zc];
        ++plan->z_nsplit[zc];
      } else {
        zc = nz++;
        plan->z_cls[zc] = i;
        plan->z_lo[zc] = lo_k;
        plan->z_hi[zc] = hi_k;
        plan->z_first[zc] = ns;
        plan->z_nsplit[zc] = 1;
      }
      plan->s_X[ns] = X;
      plan->s_mult[ns] = 1;
      ++ns;
      lastX = X;
    }
    // K' level below each zone of the class (rank below all its splits) and above all of them
    int j = jb;
#pragma unroll 1
    for (int z = plan->cls_zone0[i]; z < nz; ++z) {
      plan->z_jbelow[z] = j;
#pragma unroll 1
      for (int t = 0; t < plan->z_nsplit[z]; ++t) j += plan->s_mult[plan->z_first[z] + t];
      const double E = (double)(plan->z_hi[z] - plan->z_lo[z]) / two60 * h;
      int64_t cap = (int64_t)(2.0 * E) + 1024;
      if (cap > h) cap = h;
      if (used + cap > P.N) cap = P.N - used;
      plan->z_cap[z] = (int)cap;
      plan->z_base[z] = (int)used;
      used += cap;
    }
    plan->cls_jtot[i] = j;
    plan->cls_nzone[i] = nz - plan->cls_zone0[i];
    slot += plan->cls_nzone[i] + 1;   // gaps 0 .. nzone of the class
  }
  plan->k6_nz = nz;
  if (fallback || P.k6_force_fallback) plan->k6_fallback = 1;
}

// One warp (lanes threadIdx.x & 31 of the calling warp); hist may point to shared or global memory.
// Inlined (with mcf_plan and k6_zones) so that P, a kernel parameter, is read with direct indexed
// constant loads: a reference escaping into a called function would make the compiler copy the whole
// parameter block to local memory per thread.
__device__ __forceinline__ void plan_body(const int* hist, const RouteParams& P, DevPlan* __restrict__ plan,
                                       bool k6_windows = true) {
  __shared__ int h_s[kMaxLevels], f_s[kMaxLevels], hc[kMaxLevels + 1], fc[kMaxLevels + 1];
  __shared__ double frac_s[kMaxLevels];
  __shared__ int x_s[kMaxLevels][kMaxLevels];
  __shared__ int iters_s;
  const int lane = threadIdx.x & 31;
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
#pragma unroll 1
    for (int j = 0; j < nK; ++j) rank += (frac_s[j] > frac || (frac_s[j] == frac && j < lane)) ? 1 : 0;
    f_s[lane] = fl + (rank < R ? 1 : 0);
  }
  __syncwarp();
  if (lane == 0) {   // cumulative sums (<= 16 terms)
    hc[0] = 0;
    fc[0] = 0;
#pragma unroll 1
    for (int i = 0; i < nK; ++i) {
      hc[i + 1] = hc[i] + h_s[i];
      fc[i + 1] = fc[i] + f_s[i];
    }
  }
  __syncwarp();
  // ---- O6 plan: NW-corner coupling in closed form (convex c), else the exact min-cost solver (R37)
  if (P.convex) {
#pragma unroll 1
    for (int e = lane; e < nK * nK; e += 32) {
      const int i = e / nK, j = e % nK;
      const int lo = max(hc[i], fc[j]), hi = min(hc[i + 1], fc[j + 1]);
      x_s[i][j] = hi > lo ? hi - lo : 0;
    }
    if (lane == 0) iters_s = 0;
  } else if (lane == 0) {
    iters_s = mcf_plan(h_s, f_s, P, x_s);
  }
  __syncwarp();
  // ---- O7 D_Q and counters
  double dq = 0.0, lp = 0.0;
  int n_red = 0, n_up = 0, n_down = 0;
  const double invN = N > 0 ? __ddiv_rn(1.0, (double)N) : 0.0;
#pragma unroll 1
  for (int e = lane; e < nK * nK; e += 32) {
    const int i = e / nK, j = e % nK;
    const int x = x_s[i][j];
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
#pragma unroll 1
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
#pragma unroll 1
    for (int j = 0; j < nK; ++j) {
      acc += x_s[i][j];
      plan->X[i][j] = acc;
    }
    // I_j: ascending instance ids at level j, and the multiply-high constant for div n_j
    int n = 0, nb = 0;
#pragma unroll 1
    for (int w = 0; w < P.W; ++w) {
      nb += P.inst_level[w] < i ? 1 : 0;
      if (P.inst_level[w] == i) {
        plan->inst_pos[w] = n;
        plan->inst_list[i][n++] = w;
      }
    }
    plan->inst_base[i] = nb;
    plan->n_inst[i] = n;
    plan->n_inst_recip[i] = n > 1 ? 0xFFFFFFFFu / (uint32_t)n + 1u : 0u;   // = ceil(2^32 / n)
  }
  if (lane == 0) {
    plan->class_start[nK] = hc[nK];
    plan->D_Q = N > 0 ? __ddiv_rn(dq, (double)N) : 0.0;
    plan->D_Q_LP = P.convex ? lp : __longlong_as_double(0x7FF8000000000000LL);
    plan->solver_iters = iters_s;
    plan->n_redirected = n_red;
    plan->n_upgraded = n_up;
    plan->n_downgraded = n_down;
  }
  __syncwarp();
  if (lane == 0 && k6_windows) k6_zones(h_s, x_s, P, plan);
  if (lane == 0 && !k6_windows && P.k6_force_fallback) plan->k6_fallback = 1;   // (reported as forced)
}

}  // namespace
}  // namespace pas
