// f1 -- forecast-driven streaming mode (R21-R24).
//
// Paper: the Optimal-K Predictor "forecasts the optimal-K distribution (H_K) for the incoming
// prompt queries" from a window of past K's ("saturates around 1000", P:218,
// P:225); the K-to-K' Route Planner turns (H_K, F) into redirection probabilities P(K'|K) (P:89,
// Eq. 1 at P:96), which the Query Dispatcher applies prompt by prompt.
//
//   k_fc_plan    one warp: (re)build the plan when due -- Hc from the window counts (exact integer
//                division, 2^-32 units), Fc from F (fp64 left-to-right sum, floor), the Eq. 1 value
//                of the fixed-point monotone coupling (D_Q_plan), the L2 error of the forecast the
//                plan was built from against this batch's realised H_K, the instance lists.
//   k_fc_sample  thread per prompt: u = Philox stream 3, pos = Hc_i + (u (Hc_{i+1} - Hc_i)) >> 32,
//                K' = the level whose Fc interval holds pos (inverse CDF of row i of the plan);
//                realised moves x_ij tallied per block, then one atomic per nonzero (i, j).
//   k_fc_window  one CTA: append the batch's K levels to the ring (the last `window` in prompt
//                order), recount it; then the batch's f, realised D_Q and counters from x.
// All integer except D_Q_plan / l2 / D_Q, which use explicit _rn fp64 ops in the oracle's order.
#include "pas_internal.cuh"
#include "philox.cuh"

namespace pas {
namespace {

constexpr uint64_t kOne = 1ull << 32;

__device__ void fill_instance_lists(const RouteParams& P, DevPlan* plan, int lane) {
  if (lane < P.nK) {
    int n = 0, nb = 0;
    for (int w = 0; w < P.W; ++w) {
      nb += P.inst_level[w] < lane ? 1 : 0;
      if (P.inst_level[w] == lane) {
        plan->inst_pos[w] = n;
        plan->inst_list[lane][n++] = w;
      }
    }
    plan->inst_base[lane] = nb;
    plan->n_inst[lane] = n;
    plan->n_inst_recip[lane] = n > 1 ? 0xFFFFFFFFu / (uint32_t)n + 1u : 0u;   // = ceil(2^32 / n)
  }
}

__global__ void __launch_bounds__(32) k_fc_plan(const int* __restrict__ hist, const __grid_constant__ RouteParams P,
                                                DevPlan* __restrict__ plan, FcState* __restrict__ fcs, int replan) {
  pdl_entry();
  const int lane = threadIdx.x;
  const int nK = P.nK;
  fill_instance_lists(P, plan, lane);
  if (lane < nK) plan->h[lane] = hist[lane];
  if (lane != 0) return;
  // ---- R22: forecast cumulative masses (held between rebuilds)
  if (replan) {
    fcs->plan_n = fcs->n;
    uint64_t run = 0;
    fcs->Hc[0] = 0;
    for (int i = 0; i < nK; ++i) {
      fcs->plan_cnt[i] = fcs->cnt[i];
      if (fcs->n == 0) {
        fcs->Hc[i + 1] = ((uint64_t)(i + 1) * kOne) / (uint64_t)nK;
      } else {
        run += (uint64_t)fcs->cnt[i];
        fcs->Hc[i + 1] = (run * kOne) / (uint64_t)fcs->n;
      }
    }
  }
  fcs->replanned = replan;
  // cumulative F, 2^32 from the last level with F > 0 on
  int jlast = 0;
  for (int j = 0; j < nK; ++j)
    if (P.F[j] > 0.0) jlast = j;
  double s = 0.0;
  fcs->Fc[0] = 0;
  for (int j = 0; j < nK; ++j) {
    s = __dadd_rn(s, P.F[j]);
    uint64_t v = kOne;
    if (j < jlast) {
      const double q = floor(__dmul_rn(s, 4294967296.0));
      v = q <= 0.0 ? 0 : (q >= 4294967296.0 ? kOne : (uint64_t)q);
    }
    fcs->Fc[j + 1] = v;
  }
  // Eq. 1 on the fixed-point coupling, i-major
  double dq = 0.0;
  for (int i = 0; i < nK; ++i)
    for (int j = i + 1; j < nK; ++j) {
      const uint64_t lo = max(fcs->Hc[i], fcs->Fc[j]), hi = min(fcs->Hc[i + 1], fcs->Fc[j + 1]);
      if (hi > lo)
        dq = __dadd_rn(dq, __dmul_rn(__ddiv_rn((double)(hi - lo), 4294967296.0), P.c[P.grid[j] - P.grid[i]]));
    }
  fcs->D_Q_plan = dq;
  // L2 error of the forecast the plan was built from vs the realised H_K of this batch
  double acc = 0.0;
  for (int i = 0; i < nK; ++i) {
    const double pr = fcs->plan_n == 0 ? __ddiv_rn(1.0, (double)nK)
                                       : __ddiv_rn((double)fcs->plan_cnt[i], (double)fcs->plan_n);
    const double re = __ddiv_rn((double)hist[i], (double)P.N);
    const double dlt = __dsub_rn(pr, re);
    acc = __dadd_rn(acc, __dmul_rn(dlt, dlt));
  }
  fcs->l2 = __dsqrt_rn(acc);
  fcs->n_unforecast = 0;
}

__global__ void __launch_bounds__(256) k_fc_sample(const uint8_t* __restrict__ level, const __grid_constant__ RouteParams P,
                                                   DevPlan* __restrict__ plan, FcState* __restrict__ fcs,
                                                   int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7) {
  pdl_entry();
  __shared__ uint64_t Hc[kMaxLevels + 1], Fc[kMaxLevels + 1];
  __shared__ int tally[kMaxLevels * kMaxLevels];
  __shared__ int unf;
  const int nK = P.nK;
  if (threadIdx.x <= nK) {
    Hc[threadIdx.x] = fcs->Hc[threadIdx.x];
    Fc[threadIdx.x] = fcs->Fc[threadIdx.x];
  }
  for (int e = threadIdx.x; e < nK * nK; e += blockDim.x) tally[e] = 0;
  if (threadIdx.x == 0) unf = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int my_unf = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P.N; p += stride) {
    const int i = level[p];
    const uint32_t u = philox_stream(P.seed, batch_seq_of(P), (uint32_t)p, kStreamForecast).x;
    const uint64_t w = Hc[i + 1] - Hc[i];
    my_unf += w == 0;
    uint64_t pos = Hc[i] + (((uint64_t)u * w) >> 32);
    if (pos > kOne - 1) pos = kOne - 1;
    int j = 0;
    while (j < nK - 1 && Fc[j + 1] <= pos) ++j;
    K_prime[p] = P.grid[j];
    if (P.mode == PAS_UNIFORM) {
      const uint4 r = philox_stream(P.seed, batch_seq_of(P), (uint32_t)p, kStreamUniform);
      cls7[p] = plan->inst_list[j][(uint32_t)(((uint64_t)r.x * (uint32_t)plan->n_inst[j]) >> 32)];
    } else {
      cls7[p] = j;
    }
    atomicAdd(&tally[i * nK + j], 1);
  }
  if (my_unf) atomicAdd(&unf, my_unf);
  __syncthreads();
  for (int e = threadIdx.x; e < nK * nK; e += blockDim.x)
    if (tally[e]) atomicAdd(&plan->x[e / nK][e % nK], tally[e]);
  if (threadIdx.x == 0 && unf) atomicAdd(&fcs->n_unforecast, unf);
}

__global__ void __launch_bounds__(1024) k_fc_window(const uint8_t* __restrict__ level, const __grid_constant__ RouteParams P,
                                                    DevPlan* __restrict__ plan, FcState* __restrict__ fcs,
                                                    uint8_t* __restrict__ ring, int window) {
  pdl_entry();
  __shared__ int cnt[kMaxLevels];
  __shared__ int head_s, n_s;
  const int64_t N = P.N;
  if (threadIdx.x < kMaxLevels) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    head_s = fcs->head;
    n_s = fcs->n;
  }
  __syncthreads();
  const int head = head_s, n_old = n_s;
  // R21: append in prompt order, keep the last `window`
  int head_new, n_new;
  if (N >= window) {
    for (int t = threadIdx.x; t < window; t += blockDim.x) ring[t] = level[N - window + t];
    head_new = 0;
    n_new = window;
  } else {
    for (int t = threadIdx.x; t < N; t += blockDim.x) ring[(head + t) % window] = level[t];
    head_new = (int)((head + N) % window);
    n_new = (int)min((int64_t)n_old + N, (int64_t)window);
  }
  __syncthreads();
  // valid entries: all `window` once full, else ring[0, n) (filled from 0 since the last reset)
  for (int t = threadIdx.x; t < n_new; t += blockDim.x) atomicAdd(&cnt[ring[t]], 1);
  __syncthreads();
  if (threadIdx.x < P.nK) fcs->cnt[threadIdx.x] = cnt[threadIdx.x];
  if (threadIdx.x == 0) {
    fcs->head = head_new;
    fcs->n = n_new;
    // realised bookkeeping of the batch: f = K' counts, D_Q = sum_p D(K'_p, K_p) / N (i-major)
    const int nK = P.nK;
    double dq = 0.0;
    int n_red = 0, n_up = 0, n_down = 0;
    for (int i = 0; i < nK; ++i)
      for (int j = 0; j < nK; ++j) {
        const int x = plan->x[i][j];
        if (j != i) n_red += x;
        if (j < i) n_up += x;
        if (j > i) {
          n_down += x;
          if (x) dq = __dadd_rn(dq, __dmul_rn((double)x, P.c[P.grid[j] - P.grid[i]]));
        }
      }
    for (int j = 0; j < nK; ++j) {
      int f = 0;
      for (int i = 0; i < nK; ++i) f += plan->x[i][j];
      plan->f[j] = f;
    }
    plan->D_Q = N > 0 ? __ddiv_rn(dq, (double)N) : 0.0;
    plan->D_Q_LP = fcs->D_Q_plan;
    plan->n_redirected = n_red;
    plan->n_upgraded = n_up;
    plan->n_downgraded = n_down;
  }
}

}  // namespace

cudaError_t launch_fc_plan(const int* hist, const RouteParams& p, DevPlan* plan, FcState* fcs, bool replan,
                           cudaStream_t st) {
  launch_pdl(k_fc_plan, 1, 32, 0, st, hist, p, plan, fcs, replan ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_fc_sample(const uint8_t* level, const RouteParams& p, DevPlan* plan, FcState* fcs,
                             int32_t* K_prime, uint8_t* cls7, cudaStream_t st) {
  int64_t blocks = (p.N + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  if (blocks < 1) blocks = 1;
  launch_pdl(k_fc_sample, (unsigned)blocks, 256, 0, st, level, p, plan, fcs, K_prime, cls7);
  return cudaGetLastError();
}

cudaError_t launch_fc_window(const uint8_t* level, const RouteParams& p, DevPlan* plan, FcState* fcs,
                             uint8_t* ring, int window, cudaStream_t st) {
  launch_pdl(k_fc_window, 1, 1024, 0, st, level, p, plan, fcs, ring, window);
  return cudaGetLastError();
}

}  // namespace pas
