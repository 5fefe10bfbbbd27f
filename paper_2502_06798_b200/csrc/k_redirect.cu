// K6 -- redirection sampling: every prompt gets its K' from the Route-Plan.
//
// Exact-count form (R3): within optimal-K class i, prompts are ordered by a 60-bit Philox
// key kappa_p (ties by prompt index); the prompt of class rank r is served at K'_j for
// X_i[j-1] <= r < X_i[j] (X_i = inclusive prefix of row i of the plan x), so exactly x_ij prompts of
// class i go to level j and the ranks are a uniformly random permutation of the class (R18: kappa
// depends only on seed, batch_seq, p -- not on the router GPU count).
//
// Selection instead of sorting: K'_p only depends on how many of the class's nK - 1 split ranks
// X_i[j] lie at or below rank_p, so only the split elements have to be located -- order statistics,
// not a sort.  Two levels:
//   k6_hist    kappa = Philox(p) (stored, 8 B), histogram of (class, top kb bits of kappa) in global
//              atomics (kb = ceil(log2 N) - 6, <= 18: on average <= 64 prompts per bucket of a full
//              class);
//   k6_chunks + k6_bounds  per class: chunk sums of the bucket counts (many CTAs, coalesced), then
//              the bucket holding each split rank and the split's rank inside it (a warp scan over
//              one chunk); each distinct split bucket gets a candidate list;
//   k6_assign  every prompt counts the split buckets below its own bucket -- that IS its K' -- unless
//              its bucket holds a split, then it appends (kappa, p) to that bucket's list;
//   k6_resolve one CTA per split bucket ranks its few entries exactly by (kappa, p) in shared memory.
// Per prompt: level 1 B read twice, kappa 8 B written + read, K' 4 B + K7 class 1 B written; plus one
// L2 atomic.  The previous full counting-sort ranking (scatter + in-bucket rank of all N entries)
// moved 53 B per prompt through scattered accesses (8.8 ms at 64M prompts).
#include "pas_internal.cuh"
#include "philox.cuh"

namespace pas {
namespace {

constexpr int RT = 256;
#ifndef PAS_K6_GRIDCAP
#define PAS_K6_GRIDCAP 1   // k6_assign: grid capped at 8 CTAs per SM (grid-stride); 0: uncapped
#endif
constexpr int kSmemList = 2048;   // k6_resolve: entries staged in shared memory (else read from L2)

__device__ __forceinline__ bool entry_less(uint64_t ka, int32_t pa, uint64_t kb, int32_t pb) {
  return ka < kb || (ka == kb && pa < pb);
}

__device__ __forceinline__ uint32_t top_bits(uint64_t kappa, int kb) {
  return kb ? (uint32_t)(kappa >> (60 - kb)) : 0u;
}

// K' level j of prompt p: K' value and the route-and-batch class (K' level in greedy mode, the
// instance I_j[(u n_j) >> 32] in uniform mode)
__device__ __forceinline__ void emit(const RouteParams& P, const int* grid, const DevPlan* __restrict__ plan,
                                     int64_t p, int j, int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7) {
  K_prime[p] = grid[j];
  if (P.mode == PAS_UNIFORM) {
    const uint4 w = philox_stream(P.seed, batch_seq_of(P), (uint32_t)p, kStreamUniform);
    const uint32_t nj = (uint32_t)plan->n_inst[j];
    cls7[p] = (uint8_t)plan->inst_list[j][(uint32_t)(((uint64_t)w.x * nj) >> 32)];
  } else {
    cls7[p] = (uint8_t)j;
  }
}

__global__ void __launch_bounds__(RT) k6_hist(const uint8_t* __restrict__ level, const RouteParams P,
                                              uint64_t* __restrict__ key, int32_t* __restrict__ hist) {
  pdl_entry();
  const int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x;
  if (p >= P.N) return;
  const uint4 w = philox_stream(P.seed, batch_seq_of(P), (uint32_t)p, kStreamRedirect);
  const uint64_t kappa = (((uint64_t)w.y << 32) | w.x) >> 4;
  key[p] = kappa;
  atomicAdd(&hist[((uint32_t)level[p] << P.kb) | top_bits(kappa, P.kb)], 1);
}

// Per (class, chunk of kChunks) sums of the bucket counts, coalesced, many CTAs.
constexpr int kChunks = 256;
__global__ void __launch_bounds__(RT) k6_chunks(const RouteParams P, const int32_t* __restrict__ hist,
                                                int32_t* __restrict__ csum) {
  pdl_entry();
  __shared__ int32_t ws[RT / 32];
  const int i = blockIdx.x / kChunks, c = blockIdx.x % kChunks;
  const int nb = 1 << P.kb, len = (nb + kChunks - 1) / kChunks;
  const int c0 = c * len, c1 = c0 + len < nb ? c0 + len : nb;
  const int32_t* hc = hist + ((int64_t)i << P.kb);
  int s = 0;
  for (int b = c0 + threadIdx.x; b < c1; b += RT) s += hc[b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < RT / 32; ++w) t += ws[w];
    csum[blockIdx.x] = t;
  }
}

// One CTA per class: the chunk holding each split rank (scan of the chunk sums), then one warp per
// split walks that chunk 32 buckets at a time (warp scan) to the bucket and the split's rank in it.
__global__ void __launch_bounds__(RT) k6_bounds(const RouteParams P, const DevPlan* __restrict__ plan,
                                                const int32_t* __restrict__ hist, const int32_t* __restrict__ csum,
                                                K6Bounds* __restrict__ bnd, K6List* __restrict__ lists,
                                                int32_t* __restrict__ used) {
  pdl_entry();
  __shared__ int32_t cex[kChunks + 1];
  __shared__ int32_t sb[kMaxLevels], so[kMaxLevels];
  const int i = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int nb = 1 << P.kb, len = (nb + kChunks - 1) / kChunks;
  const int32_t* hc = hist + ((int64_t)i << P.kb);
  {   // exclusive scan of the class's kChunks chunk sums (one per thread: warp scans + warp totals)
    static_assert(kChunks == RT, "one chunk sum per thread");
    __shared__ int32_t wtot[RT / 32];
    const int v = csum[i * kChunks + t];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wtot[w] = incl;
    __syncthreads();
    int before = 0;
    for (int q = 0; q < w; ++q) before += wtot[q];
    cex[t] = before + incl - v;
    if (t == RT - 1) cex[kChunks] = before + incl;
  }
  if (t < kMaxLevels) sb[t] = INT32_MAX;
  __syncthreads();
  const int h = plan->h[i];
  for (int j = w; j + 1 < P.nK; j += RT / 32) {   // split rank X_i[j]: the first prompt of group j + 1
    const int X = plan->X[i][j];
    if (X >= h) continue;                          // no such prompt
    int c = 0;   // the chunk holding rank X: the last c with cex[c] <= X (binary search, cex ascending)
    for (int step = kChunks / 2; step > 0; step >>= 1)
      if (c + step < kChunks && cex[c + step] <= X) c += step;
    const int c0 = c * len, c1 = c0 + len < nb ? c0 + len : nb;
    int run = cex[c];
    for (int base = c0; base < c1; base += 32) {   // 32 buckets at a time, warp scan
      const int v = base + lane < c1 ? hc[base + lane] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (run + tot > X) {
        const unsigned hit = __ballot_sync(0xffffffffu, run + incl > X);
        const int L = __ffs(hit) - 1;
        if (lane == L) {
          sb[j] = base + L;
          so[j] = X - (run + incl - v);
        }
        break;
      }
      run += tot;
    }
  }
  __syncthreads();
  if (t == 0) {
    int last_bucket = -1, id = -1;
    for (int j = 0; j + 1 < P.nK; ++j) {
      const int b = sb[j];
      bnd->bucket[i][j] = b;
      bnd->off[i][j] = so[j];
      if (b == INT32_MAX) {
        bnd->list[i][j] = -1;
        continue;
      }
      if (b != last_bucket) {   // one candidate list per distinct split bucket (splits are sorted)
        const int cnt = hc[b];
        id = atomicAdd(&used[0], 1);
        K6List L;
        L.cls = i;
        L.bucket = b;
        L.cnt = cnt;
        L.base = atomicAdd(&used[1], cnt);
        L.fill = 0;
        L.below = j;             // splits in lower buckets of the class
        lists[id] = L;
        last_bucket = b;
      }
      bnd->list[i][j] = id;
    }
  }
}

__global__ void __launch_bounds__(RT) k6_assign(const uint8_t* __restrict__ level, const uint64_t* __restrict__ key,
                                                const RouteParams P, const DevPlan* __restrict__ plan,
                                                const K6Bounds* __restrict__ bnd, K6List* __restrict__ lists,
                                                KeyEntry* __restrict__ cand, int32_t* __restrict__ K_prime,
                                                uint8_t* __restrict__ cls7) {
  pdl_entry();
  __shared__ int32_t sb[kMaxLevels][kMaxLevels], sl[kMaxLevels][kMaxLevels];
  __shared__ int grid_s[kMaxLevels];
  if (threadIdx.x < kMaxLevels) grid_s[threadIdx.x] = P.grid[threadIdx.x];
  for (int e = threadIdx.x; e < P.nK * kMaxLevels; e += RT) {   // once per (persistent) CTA
    const int i = e / kMaxLevels, j = e % kMaxLevels;
    sb[i][j] = j + 1 < P.nK ? bnd->bucket[i][j] : INT32_MAX;
    sl[i][j] = j + 1 < P.nK ? bnd->list[i][j] : -1;
  }
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x; p < P.N; p += (int64_t)gridDim.x * RT) {
    const int i = level[p];
    const uint64_t kappa = key[p];
    const int b = (int)top_bits(kappa, P.kb);
    int below = 0, list = -1;
    for (int j = 0; j + 1 < P.nK; ++j) {
      below += sb[i][j] < b;
      if (sb[i][j] == b) list = sl[i][j];
    }
    if (list < 0) {
      emit(P, grid_s, plan, p, below, K_prime, cls7);
      continue;
    }
    K6List* L = lists + list;
    const int slot = atomicAdd(&L->fill, 1);
    cand[L->base + slot] = KeyEntry{kappa, (int32_t)p, 0};
  }
}

__global__ void __launch_bounds__(RT) k6_resolve(const RouteParams P, const DevPlan* __restrict__ plan,
                                                 const K6Bounds* __restrict__ bnd, const K6List* __restrict__ lists,
                                                 const int32_t* __restrict__ used, const KeyEntry* __restrict__ cand,
                                                 int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7) {
  pdl_entry();
  __shared__ uint64_t sk[kSmemList];
  __shared__ int32_t sp[kSmemList];
  __shared__ int grid_s[kMaxLevels];
  if (threadIdx.x < kMaxLevels) grid_s[threadIdx.x] = P.grid[threadIdx.x];
  if ((int)blockIdx.x >= used[0]) return;
  const K6List L = lists[blockIdx.x];
  const KeyEntry* E = cand + L.base;
  const bool staged = L.cnt <= kSmemList;
  if (staged)
    for (int e = threadIdx.x; e < L.cnt; e += RT) {
      sk[e] = E[e].key;
      sp[e] = E[e].p;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < L.cnt; e += RT) {
    const uint64_t k = staged ? sk[e] : E[e].key;
    const int32_t p = staged ? sp[e] : E[e].p;
    int r = 0;   // rank inside the bucket by (kappa, p)
    for (int f = 0; f < L.cnt; ++f)
      r += staged ? entry_less(sk[f], sp[f], k, p) : entry_less(E[f].key, E[f].p, k, p);
    int j = L.below;
    for (int q = 0; q + 1 < P.nK; ++q)
      j += (bnd->bucket[L.cls][q] == L.bucket && r >= bnd->off[L.cls][q]) ? 1 : 0;
    emit(P, grid_s, plan, p, j, K_prime, cls7);
  }
}

}  // namespace

int redirect_kb(int64_t N) {
  int b = 0;
  while (((int64_t)1 << b) < N) ++b;
  b -= 6;
  return b < 0 ? 0 : (b > kMaxK6Bits ? kMaxK6Bits : b);
}

cudaError_t launch_redirect(const uint8_t* level, const RouteParams& p, const DevPlan* plan, const RedirectWs& w,
                            int32_t* K_prime, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  cudaError_t e;
  if ((e = launch_zero(w.hist, (int64_t)p.nK << p.kb, w.used, 2, nullptr, 0, st))) return e;
  const unsigned blocks = (unsigned)((p.N + RT - 1) / RT);
  launch_pdl(k6_hist, blocks, RT, 0, st, level, p, w.key, w.hist);
  launch_pdl(k6_chunks, p.nK * kChunks, RT, 0, st, p, w.hist, w.csum);
  launch_pdl(k6_bounds, p.nK, RT, 0, st, p, plan, w.hist, w.csum, w.bnd, w.lists, w.used);
  const unsigned ablocks = (!PAS_K6_GRIDCAP || blocks < (unsigned)kNumSMs * 8) ? blocks : (unsigned)kNumSMs * 8;
  launch_pdl(k6_assign, ablocks, RT, 0, st, level, w.key, p, plan, w.bnd, w.lists, w.cand, K_prime, w.cls7);
  launch_pdl(k6_resolve, p.nK * (p.nK - 1) > 0 ? p.nK * (p.nK - 1) : 1, RT, 0, st, p, plan, w.bnd, w.lists, w.used,
             w.cand, K_prime, w.cls7);
  *launches += 6;
  return cudaGetLastError();
}

}  // namespace pas
