// dispatch.cuh -- f3 stateful dispatcher: integer-time helpers shared by the prep kernel
// (k_dispatch.cu) and the per-prompt pick in K7 (k_batch.cu).  DESIGN.md R28-R32.
//
// Phase 2 of a greedy pick (every queue of the level holds >= b*): the prompt goes to the
// instance whose next batch starts soonest, key_w(Q) = B'_w + floor(Q / b*) s_w (R29), ties to the
// lowest id, and the queue grows by one.  Each key sequence is non-decreasing in Q, so the
// sequential picks of a level are the merge of the instances' key sequences ordered by
// (key, id, queue position).  The r-th phase-2 prompt of a level is therefore found without
// replaying the r-1 before it: the number of merged entries with key <= T is
//   count(T) = sum_w cnt_w(T),  cnt_w(T) = max(0, (floor((T - B'_w) / s_w) + 1) b* - Q1_w)  (T >= B'_w)
// so T* = min{T : count(T) > r} by binary search, then the entries with key T* are walked in
// instance order.  All arithmetic is exact int64.
#pragma once

#include "pas_internal.cuh"

namespace pas {

constexpr int64_t kQSat = (int64_t)1 << 44;   // saturate floor((T - B') / s) (never reached at T*-1)

// floor(a / s) for 0 <= a, 1 <= s, from an fp64 estimate corrected by exact products
__device__ __forceinline__ int64_t disp_fdiv(int64_t a, int64_t s, double inv) {
  int64_t q = (int64_t)((double)a * inv);
  while (q > 0 && q * s > a) --q;
  while ((q + 1) * s <= a) ++q;
  return q;
}

// merged entries of instance w with key <= T (R29 key, phase 2)
__device__ __forceinline__ int64_t disp_cnt(const DispPlan* __restrict__ dp, int w, int64_t T, int64_t b) {
  const int64_t Bp = dp->Bp[w];
  if (T < Bp) return 0;
  int64_t q = disp_fdiv(T - Bp, dp->svc[w], dp->inv_svc[w]);
  if (q > kQSat) q = kQSat;
  const int64_t c = (q + 1) * b - dp->Q1[w];
  return c > 0 ? c : 0;
}

// Phase-2 pick of the r-th prompt (0-based, after phase 1) among the nj instances `ws` (ascending
// ids) of one level: instance and its queue position m past Q1 (the prompt's slot is Q1 + m).
__device__ __forceinline__ void disp_phase2(const DispPlan* __restrict__ dp, const int* ws, int nj, int64_t r,
                                            int64_t b, int& inst, int64_t& m) {
  int64_t lo = INT64_MAX, hi = INT64_MAX;
  for (int i = 0; i < nj; ++i) {
    const int w = ws[i];
    const int64_t k0 = dp->Bp[w] + (dp->Q1[w] / b) * dp->svc[w];        // first key
    const int64_t kr = dp->Bp[w] + ((dp->Q1[w] + r) / b) * dp->svc[w];  // key if w alone took r+1
    lo = k0 < lo ? k0 : lo;
    hi = kr < hi ? kr : hi;
  }
  lo -= 1;                                  // count(lo) = 0 <= r < count(hi)
  while (hi - lo > 1) {
    const int64_t mid = lo + (hi - lo) / 2;
    int64_t c = 0;
    for (int i = 0; i < nj && c <= r; ++i) c += disp_cnt(dp, ws[i], mid, b);
    if (c > r) hi = mid; else lo = mid;
  }
  int64_t before = 0;                       // count(T* - 1)
  for (int i = 0; i < nj; ++i) before += disp_cnt(dp, ws[i], lo, b);
  int64_t rr = r - before;
  inst = ws[nj - 1];
  m = 0;
  for (int i = 0; i < nj; ++i) {            // entries with key T*, instance order
    const int w = ws[i];
    const int64_t c0 = disp_cnt(dp, w, lo, b), e = disp_cnt(dp, w, hi, b) - c0;
    if (rr < e) {
      inst = w;
      m = c0 + rr;
      return;
    }
    rr -= e;
  }
}

// Greedy pick (R29) of the t-th prompt (0-based, prompt order) of level j; slot = queue position (R31).
__device__ __forceinline__ void disp_pick_greedy(const DispPlan* __restrict__ dp, const int* ws, int nj, int j,
                                                 int64_t t, int64_t b, int& inst, int64_t& slot) {
  const int beg = dp->p1_beg[j], end = dp->p1_beg[j + 1];
  if (t < dp->p1_total[j]) {                // phase 1: fill the longest queues below b* first
    int e = beg;
    while (e + 1 < end && dp->p1_cum[e + 1] <= t) ++e;
    inst = dp->p1_w[e];
    slot = dp->Q0[inst] + (t - dp->p1_cum[e]);
    return;
  }
  int64_t m;
  disp_phase2(dp, ws, nj, t - dp->p1_total[j], b, inst, m);
  slot = dp->Q1[inst] + m;
}

}  // namespace pas
