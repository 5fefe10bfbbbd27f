// K6 -- redirection sampling: every prompt gets its K' from the Route-Plan.
//
// Exact-count form (R3): within optimal-K class i, prompts are ranked by a 60-bit Philox
// key kappa_p (ties by prompt index), and rank_p in [X_i[j-1], X_i[j]) is served at K'_j, so exactly
// x_ij prompts of class i go to level j and the ranks are a uniformly random permutation of the class
// (R18: kappa depends only on seed, batch_seq, p -- not on the router GPU count).
//
// Ranking without a full sort: composite key (class << 60 | kappa) -> bucket (class, top kb bits of
// kappa) counting sort (count, scan, scatter), then each prompt counts the keys below it inside its
// own bucket (the choice of kb keeps the mean bucket below 16 prompts).  Global rank = bucket start + in-bucket
// rank, which equals the position in the (key, p) order; rank within class = global - class start.
//
// Kernels: k_keys (Philox + bucket histogram), k_scan (one CTA), k_scatter, k_rank (rank, K', and the
// route-and-batch class: K' level in greedy mode, instance I_j[(u n_j) >> 32] in uniform mode).
#include "pas_internal.cuh"
#include "philox.cuh"

namespace pas {
namespace {

__global__ void k_keys(const uint8_t* __restrict__ level, RouteParams P, uint64_t* __restrict__ key,
                       int32_t* __restrict__ bucket, int32_t* __restrict__ bcount) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.N) return;
  const uint4 w = philox_stream(P.seed, P.batch_seq, (uint32_t)p, kStreamRedirect);
  const uint64_t kappa = (((uint64_t)w.y << 32) | w.x) >> 4;
  const uint32_t lvl = level[p];
  key[p] = ((uint64_t)lvl << 60) | kappa;
  const int32_t b = (int32_t)((lvl << P.kb) | (uint32_t)(P.kb ? (kappa >> (60 - P.kb)) : 0));
  bucket[p] = b;
  atomicAdd(&bcount[b], 1);
}

// Exclusive scan of n ints with one CTA of 1024 threads: coalesced tiles of 4096 (int4 per thread),
// warp-shuffle scans, a running carry across tiles.
__global__ void __launch_bounds__(1024) k_scan(const int32_t* __restrict__ in, int32_t* __restrict__ out, int n) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 4096) {
    const int i0 = base + 4 * t;
    int v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (i0 + j < n) ? in[i0 + j] : 0;
    const int local = v[0] + v[1] + v[2] + v[3];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int x = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      wsum[lane] = x;   // inclusive over warps
    }
    __syncthreads();
    int run = carry_s + (w ? wsum[w - 1] : 0) + incl - local;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j < n) out[i0 + j] = run;
      run += v[j];
    }
    __syncthreads();
    if (t == 0) carry_s += wsum[31];
    __syncthreads();
  }
}

__global__ void k_scatter(const int32_t* __restrict__ bucket, int64_t N, const int32_t* __restrict__ bstart,
                          int32_t* __restrict__ bfill, int32_t* __restrict__ items) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int b = bucket[p];
  items[bstart[b] + atomicAdd(&bfill[b], 1)] = (int32_t)p;
}

__global__ void k_rank(const uint8_t* __restrict__ level, RouteParams P, const DevPlan* __restrict__ plan,
                       const uint64_t* __restrict__ key, const int32_t* __restrict__ bucket,
                       const int32_t* __restrict__ bcount, const int32_t* __restrict__ bstart,
                       const int32_t* __restrict__ items, int32_t* __restrict__ lvl_prime,
                       int32_t* __restrict__ cls7, int32_t* __restrict__ K_prime) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.N) return;
  const int b = bucket[p];
  const uint64_t kp = key[p];
  const int start = bstart[b], n = bcount[b];
  int r = 0;
  for (int i = 0; i < n; ++i) {
    const int q = items[start + i];
    const uint64_t kq = key[q];
    r += (kq < kp || (kq == kp && q < p)) ? 1 : 0;
  }
  const int lvl = level[p];
  const int rank = start + r - plan->class_start[lvl];
  int j = 0;
  while (j < P.nK - 1 && rank >= plan->X[lvl][j]) ++j;
  lvl_prime[p] = j;
  K_prime[p] = P.grid[j];
  if (P.mode == PAS_UNIFORM) {
    const uint4 w = philox_stream(P.seed, P.batch_seq, (uint32_t)p, kStreamUniform);
    const uint32_t nj = (uint32_t)plan->n_inst[j];
    cls7[p] = plan->inst_list[j][(uint32_t)(((uint64_t)w.x * nj) >> 32)];
  } else {
    cls7[p] = j;
  }
}

}  // namespace

cudaError_t launch_redirect(const uint8_t* level, const RouteParams& p, const DevPlan* plan, const RedirectWs& w,
                            int32_t* K_prime, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  const int nb = p.nK << p.kb;
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.bcount, 0, sizeof(int32_t) * nb, st))) return e;
  if ((e = cudaMemsetAsync(w.bfill, 0, sizeof(int32_t) * nb, st))) return e;
  const unsigned blocks = (unsigned)((p.N + 255) / 256);
  k_keys<<<blocks, 256, 0, st>>>(level, p, w.key, w.bucket, w.bcount);
  k_scan<<<1, 1024, 0, st>>>(w.bcount, w.bstart, nb);
  k_scatter<<<blocks, 256, 0, st>>>(w.bucket, p.N, w.bstart, w.bfill, w.items);
  k_rank<<<blocks, 256, 0, st>>>(level, p, plan, w.key, w.bucket, w.bcount, w.bstart, w.items, w.lvl_prime,
                                 w.cls7, K_prime);
  *launches += 4;
  return cudaGetLastError();
}

}  // namespace pas
