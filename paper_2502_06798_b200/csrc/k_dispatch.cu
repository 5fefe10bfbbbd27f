// f3 -- the stateful load-aware Query Dispatcher (R28-R32).
//
// The queue state of every serving instance (waiting prompts Q, busy-until B, the arrival times of
// the last 64 enqueued prompts) lives on the device across batches.  One routed batch arrives at
// `now` (R28).  k_disp_prep -- one CTA, one thread per instance, launched between K7's class scan and
// its rank pass -- does, in closed form per instance:
//   1. the form_batch events since the last batch (R30) with the b* then in force: full batches
//      fire back to back from B (floor((now - B) / s) + 1 of them, at most Q div b*), then a partial
//      queue fires at max(B, oldest + Delta) if that is <= now;
//   2. the pick tables of the batch: phase 1 (queues below b*, longest first, ties to the lowest id,
//      each topped up to b*) as a prefix table per level, and the phase-2 parameters
//      (B' = max(B, now), Q1 = max(Q, b*), s) the per-prompt search of dispatch.cuh reads;
//   3. this batch's count per instance from the level totals (the batch-list offsets);
//   4. the state after the batch: Q += count, the arrival ring, then form_batch at `now` again
//      (idle instances fire at once).
// The oracle (oracle/dispatch.py) replays the same rules prompt by prompt and event by event; the
// two are compared bit-exactly (tests/test_gpu_dispatch.py).
#include "dispatch.cuh"

namespace pas {
namespace {

// form_batch events of one instance up to and including `now` (R30), closed form.
// base: the time the instance is free (B, or max(B, now) right after a dispatch).  Returns the
// busy-until after the events (base unchanged if nothing fired).
__device__ int64_t disp_advance(int64_t& Q, int64_t base, int64_t& fp, int64_t& fb, const int64_t* arr, int64_t E,
                                int64_t s, double inv, int64_t now, int64_t b, int64_t timeout, bool& fired) {
  int64_t B = base;
  if (Q >= b && B <= now) {   // full batches back to back (B is never earlier than the b*-th arrival)
    int64_t nb = disp_fdiv(now - B, s, inv) + 1;
    if (nb > Q / b) nb = Q / b;
    Q -= nb * b;
    fp += nb * b;
    fb += nb;
    B += nb * s;
    fired = true;
  }
  if (Q > 0 && Q < b) {       // partial queue: the oldest prompt has waited Delta
    const int64_t head = arr[(E - Q) & (kArrRing - 1)];
    const int64_t t = B > head + timeout ? B : head + timeout;
    if (t <= now) {
      fp += Q;
      fb += 1;
      Q = 0;
      B = t + s;
      fired = true;
    }
  }
  return B;
}

__global__ void __launch_bounds__(kMaxInst) k_disp_prep(const __grid_constant__ RouteParams P, int ntiles, int nC,
                                                        const int32_t* __restrict__ scanned) {
  pdl_entry();
  DispState* S = P.dstate;
  DispPlan* D = P.dplan;
  __shared__ int64_t q0_s[kMaxInst];
  __shared__ int32_t lev_s[kMaxInst], below_s[kMaxInst], tot_s[kMaxInst];
  __shared__ int64_t bp_s[kMaxInst], q1_s[kMaxInst];
  const int w = threadIdx.x;
  const bool live = w < P.W;
  const int64_t now = P.now_us, b = P.bstar, s = live ? S->svc[w] : 1;
  const double inv = 1.0 / (double)s;
  int64_t Q = 0, B = kNeverBusy, E = 0, fp = 0, fb = 0;
  const int lev = live ? (P.mode == PAS_UNIFORM ? w : P.inst_level[w]) : -1;   // K7 class of w
  if (live) {
    Q = S->Q[w];
    B = S->B[w];
    E = S->E[w];
    fp = S->fired_prompts[w];
    fb = S->fired_batches[w];
    bool fired = false;
    B = disp_advance(Q, B, fp, fb, S->arr[w], E, s, inv, now, P.bstar_prev, P.timeout_us, fired);   // 1.
    q0_s[w] = Q;
    lev_s[w] = P.inst_level[w];
    below_s[w] = P.mode != PAS_UNIFORM && Q < b;
    bp_s[w] = B > now ? B : now;
    q1_s[w] = Q > b ? Q : b;
    // level total (class c of K7: the K' level in greedy mode, the instance in uniform mode)
    const int64_t start = scanned[(int64_t)lev * ntiles];
    const int64_t end = lev + 1 < nC ? scanned[(int64_t)(lev + 1) * ntiles] : P.N;
    tot_s[w] = (int32_t)(end - start);
  }
  __syncthreads();
  // phase-2 parameters of every instance (the per-prompt search reads them from the plan)
  if (live) {
    D->Q0[w] = q0_s[w];
    D->Q1[w] = q1_s[w];
    D->Bp[w] = bp_s[w];
    D->svc[w] = s;
    D->inv_svc[w] = inv;
  }
  int64_t cnt = 0, c = 0, total1 = 0;
  int ws[kMaxInst];   // the instances of w's level, ascending
  int nj = 0;
  const bool greedy = live && P.mode != PAS_UNIFORM;
  if (live && P.mode == PAS_UNIFORM) cnt = tot_s[w];
  if (greedy) {
    // 2. phase 1: rank of w among the below-b* instances of its level by (Q desc, id asc)
    const int j = lev_s[w];
    int rank = 0, beg = 0, n1 = 0;
    int64_t cum = 0;
    for (int v = 0; v < P.W; ++v) {
      if (lev_s[v] == j) ws[nj++] = v;
      if (!below_s[v]) continue;
      if (lev_s[v] < j) ++beg;
      if (lev_s[v] != j) continue;
      ++n1;
      total1 += b - q0_s[v];
      if (v != w && (q0_s[v] > q0_s[w] || (q0_s[v] == q0_s[w] && v < w))) {
        ++rank;
        cum += b - q0_s[v];
      }
    }
    if (below_s[w]) {
      D->p1_w[beg + rank] = w;
      D->p1_cum[beg + rank] = (int32_t)cum;
    }
    if (ws[0] == w) {   // the lowest instance of the level publishes its table bounds
      D->p1_beg[j] = beg;
      D->p1_beg[j + 1] = beg + n1;   // level j+1's publisher writes the same value
      D->p1_total[j] = (int32_t)total1;
    }
    // 3. this batch's prompts at w: its phase-1 share ...
    c = tot_s[w];
    if (below_s[w]) {
      const int64_t a = c - cum, allot = b - q0_s[w];
      cnt = a < 0 ? 0 : (a > allot ? allot : a);
    }
  }
  __syncthreads();   // the plan's phase-2 parameters are complete
  // ... then its phase-2 merged entries up to the level's last prompt r: every entry with a key
  // below T* (the last prompt's key) and its share of the T* group in instance order
  if (greedy && c > total1) {
    const int64_t r = c - total1 - 1;
    int last;
    int64_t m;
    disp_phase2(D, ws, nj, r, b, last, m);
    const int64_t T = bp_s[last] + ((q1_s[last] + m) / b) * D->svc[last];
    int64_t before = 0, upto = 0;
    for (int i = 0; i < nj; ++i) before += disp_cnt(D, ws[i], T - 1, b);
    int64_t take = r + 1 - before;
    for (int i = 0; i < nj && take > 0; ++i) {
      const int v = ws[i];
      const int64_t e = disp_cnt(D, v, T, b) - disp_cnt(D, v, T - 1, b);
      const int64_t got = take < e ? take : e;
      if (v == w) upto = got;
      take -= got;
    }
    cnt += disp_cnt(D, w, T - 1, b) + upto;
  }
  if (live) {
    D->cnt[w] = (int32_t)cnt;
    // 4. the state after the batch: enqueue at `now`, then form_batch at `now` (R28, R30)
    Q += cnt;
    for (int64_t e = (E + cnt - kArrRing > E ? E + cnt - kArrRing : E); e < E + cnt; ++e)
      S->arr[w][e & (kArrRing - 1)] = now;
    E += cnt;
    bool fired = false;
    const int64_t Bn = disp_advance(Q, bp_s[w], fp, fb, S->arr[w], E, s, inv, now, b, P.timeout_us, fired);
    S->Q[w] = Q;
    S->B[w] = fired ? Bn : B;
    S->E[w] = E;
    S->fired_prompts[w] = fp;
    S->fired_batches[w] = fb;
  }
}

}  // namespace

cudaError_t launch_disp_prep(const RouteParams& p, int ntiles, int nC, const int32_t* scanned, cudaStream_t st) {
  return launch_pdl(k_disp_prep, 1, kMaxInst, 0, st, p, ntiles, nC, scanned);
}

}  // namespace pas
