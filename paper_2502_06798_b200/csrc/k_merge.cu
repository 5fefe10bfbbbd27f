// K3 -- warp-level merge of per-range / per-GPU top-k candidates, and
// K4 -- best similarity -> optimal-K level, flags and the H_K histogram (fused into the final merge).
//
// Paper: the Optimal-K Selector "first retrieves the nearest cache and determines the optimal K"
// (PAPER.md P:102); the optimal-K distribution H_K enters Eq. 1.  Level of a prompt =
// #{m : s1 >= t_m} over the similarity bands (R8, closed below); cold cache or invalid
// embedding -> level 0 = vanilla (R16).  Only top-1 sets K (R9).
//
// Input candidates [S][N][k] (each list sorted by score desc, gid asc).  One warp per prompt: lane s
// holds the head of source s (lanes loop when S > 32); k rounds of a warp arg-max on (score, gid)
// emit the merged list.  H_K: shared-memory histogram per CTA, one global atomic per non-zero bin.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int WARPS = 8;

struct Head {
  Cand c;
  int src;   // source index (-1 = none)
};

__device__ __forceinline__ Head warp_best(Head h) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Head t;
    t.c.s = __shfl_xor_sync(0xffffffffu, h.c.s, o);
    t.c.g = __shfl_xor_sync(0xffffffffu, h.c.g, o);
    t.src = __shfl_xor_sync(0xffffffffu, h.src, o);
    const bool take = (t.src >= 0) && (h.src < 0 || cand_better(t.c, h.c) ||
                                       (!cand_better(h.c, t.c) && t.src < h.src));
    if (take) h = t;
  }
  return h;
}

// Merge of one prompt's S sorted lists; lane 0 ends with the result in out (registers of all lanes
// are used for the heads).  Returns nothing; writes out[0..k) via lane 0.
__device__ __forceinline__ void merge_prompt(const Cand* __restrict__ in, int S, int64_t N, int k, int64_t p,
                                             Cand* res /*[k] in shared or global*/, int lane) {
  // per-lane cursor over its sources: sources lane, lane+32, ...; keep pos per source in a small array
  constexpr int MAXSRC_PER_LANE = 4;   // S <= 128
  int pos[MAXSRC_PER_LANE];
#pragma unroll
  for (int j = 0; j < MAXSRC_PER_LANE; ++j) pos[j] = 0;
  for (int i = 0; i < k; ++i) {
    Head h;
    h.src = -1;
    h.c = Cand{-INFINITY, -1};
#pragma unroll
    for (int j = 0; j < MAXSRC_PER_LANE; ++j) {
      const int s = lane + 32 * j;
      if (s < S && pos[j] < k) {
        const Cand c = in[((int64_t)s * N + p) * k + pos[j]];
        if (h.src < 0 || cand_better(c, h.c)) { h.c = c; h.src = s; }
      }
    }
    const Head b = warp_best(h);
    if (b.src >= 0 && (b.src & 31) == lane) pos[b.src >> 5]++;
    if (lane == 0) res[i] = (b.src >= 0) ? b.c : Cand{-INFINITY, -1};
  }
}

__global__ void __launch_bounds__(WARPS * 32) k_merge(const Cand* __restrict__ in, int S, int64_t N, int k,
                                                      Cand* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (p >= N) return;
  merge_prompt(in, S, N, k, p, out + p * k, lane);
}

__global__ void __launch_bounds__(WARPS * 32) k_merge_select(const Cand* __restrict__ in, int S,
                                                             const uint8_t* __restrict__ pflags,
                                                             const RouteParams P, SelectOut o) {
  __shared__ Cand res[WARPS][PAS_MAX_TOPK];
  __shared__ int hist[kMaxLevels];
  __shared__ int cnt[3];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x < kMaxLevels) hist[threadIdx.x] = 0;
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * WARPS + w;
  const int k = P.topk;
  if (p < P.N) {
    const bool invalid = pflags && (pflags[p] & PAS_FLAG_INVALID);
    const bool cold = (P.M_total == 0);
    if (invalid || cold) {
      if (lane == 0)
        for (int i = 0; i < k; ++i) res[w][i] = Cand{-INFINITY, -1};
    } else {
      merge_prompt(in, S, P.N, k, p, res[w], lane);
    }
    __syncwarp();
    // lanes write the k results (coalesced)
    for (int i = lane; i < k; i += 32) {
      const Cand c = res[w][i];
      if (o.topk_id) o.topk_id[p * k + i] = c.g;
      if (o.topk_score) o.topk_score[p * k + i] = c.s;
      if (o.cand_out) o.cand_out[p * k + i] = c;
    }
    if (lane == 0) {
      int lvl = 0;
      uint8_t fl = 0;
      if (invalid) fl |= PAS_FLAG_INVALID;
      else if (cold) fl |= PAS_FLAG_COLD;
      else {
        const float s1 = res[w][0].s;
        for (int m = 0; m < P.nK - 1; ++m) lvl += (s1 >= P.thr[m]) ? 1 : 0;
        const float s2 = (k > 1) ? res[w][1].s : -INFINITY;
        if (s2 != -INFINITY && s1 - s2 < 2e-2f) fl |= PAS_FLAG_NEAR_TOP1;
        for (int m = 0; m < P.nK - 1; ++m)
          if (fabsf(s1 - P.thr[m]) < 2e-2f) fl |= PAS_FLAG_NEAR_THRESHOLD;
      }
      o.level[p] = (uint8_t)lvl;
      o.K[p] = P.grid[lvl];
      if (o.flags) o.flags[p] = fl;
      atomicAdd(&hist[lvl], 1);
      if (fl & PAS_FLAG_INVALID) atomicAdd(&cnt[0], 1);
      if (fl & PAS_FLAG_NEAR_TOP1) atomicAdd(&cnt[1], 1);
      if (fl & PAS_FLAG_NEAR_THRESHOLD) atomicAdd(&cnt[2], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < P.nK && hist[threadIdx.x]) atomicAdd(&o.hist[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0) {
    if (cnt[0]) atomicAdd(&o.plan->n_invalid, cnt[0]);
    if (cnt[1]) atomicAdd(&o.plan->n_near_top1, cnt[1]);
    if (cnt[2]) atomicAdd(&o.plan->n_near_threshold, cnt[2]);
  }
}

__global__ void k_fill_sentinel(Cand* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = Cand{-INFINITY, -1};
}

}  // namespace

cudaError_t launch_merge(const Cand* in, int S, int64_t N, int k, Cand* out, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const int64_t blocks = (N + WARPS - 1) / WARPS;
  k_merge<<<(unsigned)blocks, WARPS * 32, 0, st>>>(in, S, N, k, out);
  return cudaGetLastError();
}

cudaError_t launch_merge_select(const Cand* in, int S, const uint8_t* pflags, const RouteParams& p,
                                const SelectOut& o, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  const int64_t blocks = (p.N + WARPS - 1) / WARPS;
  k_merge_select<<<(unsigned)blocks, WARPS * 32, 0, st>>>(in, S, pflags, p, o);
  return cudaGetLastError();
}

cudaError_t launch_fill_sentinel(Cand* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_fill_sentinel<<<(unsigned)blocks, 256, 0, st>>>(out, n);
  return cudaGetLastError();
}

}  // namespace pas
