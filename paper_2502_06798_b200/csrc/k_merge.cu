// K3 -- warp-level merge of per-range / per-GPU top-k candidates, and
// K4 -- best similarity -> optimal-K level, flags and the H_K histogram (fused into the final merge).
//
// Paper: the Optimal-K Selector "first retrieves the nearest cache and determines the optimal K"
// (PAPER.md P:102); the optimal-K distribution H_K enters Eq. 1.  Level of a prompt =
// #{m : s1 >= t_m} over the similarity bands (R8, closed below); cold cache or invalid
// embedding -> level 0 = vanilla (R16).  Only top-1 sets K (R9).
//
// Input candidates [S][N][k] (each list sorted by score desc, gid asc).  S * k <= 32 (and S <= 4):
// thread per prompt over candidate rows staged in shared memory with coalesced loads.  Otherwise warp
// per prompt: lane s holds the head of source s (lanes loop when S > 32); k rounds of a warp arg-max
// on (score, gid) emit the merged list.  H_K: shared-memory histogram per CTA, one global atomic per
// non-zero bin.  HBM per prompt: S*k*8 B read, k*8 + 5 B written (+1 flag byte read).
#include "pas_internal.cuh"

#ifndef PAS_S1_GRIDCAP
#define PAS_S1_GRIDCAP 1   // k_select_s1: grid = one resident wave (grid-stride); 0: uncapped
#endif

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
  if (S <= 32 && k <= 8) {
    // one source per lane, its whole list loaded up front (eight independent loads instead of one
    // dependent load per round), then k rounds of the warp tournament; the winner's lane shifts
    Cand L[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      L[i] = (lane < S && i < k) ? in[((int64_t)lane * N + p) * k + i] : Cand{-INFINITY, -1};
    for (int i = 0; i < k; ++i) {
      Head h;
      h.src = lane < S ? lane : -1;
      h.c = L[0];
      const Head b = warp_best(h);
      if (b.src == lane) {
#pragma unroll
        for (int j = 0; j < 7; ++j) L[j] = L[j + 1];
        L[7] = Cand{-INFINITY, -1};
      }
      if (lane == 0) res[i] = (b.src >= 0) ? b.c : Cand{-INFINITY, -1};
    }
    return;
  }
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
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (p >= N) return;
  merge_prompt(in, S, N, k, p, out + p * k, lane);
}

// K4 for one prompt.  Thresholds are padded with +inf to 16 (make_params), so the level
// #{m : s1 >= t_m} is a 4-step binary search, and the near-threshold test only needs the two
// thresholds around s1.  Counts go to per-thread registers (Tally) and are flushed once per CTA.
struct Tally {
  uint64_t lv[4];        // 16 levels x 16-bit counters
  int inv, near1, nearT;
  __device__ __forceinline__ void zero() {
    lv[0] = lv[1] = lv[2] = lv[3] = 0;
    inv = near1 = nearT = 0;
  }
  __device__ __forceinline__ void add_level(int l) {
#pragma unroll
    for (int g = 0; g < 4; ++g) lv[g] += ((l >> 2) == g) ? (1ull << ((l & 3) * 16)) : 0ull;
  }
};

__device__ __forceinline__ void select_one(float s1, float s2, int32_t g1, int64_t p, bool invalid, bool cold,
                                           const RouteParams& P, const SelectOut& o, Tally& ty) {
  int lvl = 0;
  uint8_t fl = 0;
  if (invalid) fl |= PAS_FLAG_INVALID;
  else if (cold) fl |= PAS_FLAG_COLD;
  else {
#pragma unroll
    for (int step = 8; step >= 1; step >>= 1)
      if (s1 >= P.thr[lvl + step - 1]) lvl += step;
    if (s2 != -INFINITY && s1 - s2 < 2e-2f) fl |= PAS_FLAG_NEAR_TOP1;
    if ((lvl > 0 && s1 - P.thr[lvl - 1] < 2e-2f) || (lvl < P.nK - 1 && P.thr[lvl] - s1 < 2e-2f))
      fl |= PAS_FLAG_NEAR_THRESHOLD;
  }
  // f2: the top-1 entry is the one whose state is reused (R26); gids outside the store (e.g. from a
  // caller's candidate lists) are ignored
  if (P.lru_stamp && !invalid && !cold && g1 >= 0 && g1 < P.M_total) P.lru_stamp[g1] = lru_tick_of(P);
  o.level[p] = (uint8_t)lvl;
  o.K[p] = P.grid[lvl];
  if (o.flags) o.flags[p] = fl;
  ty.add_level(lvl);
  ty.inv += (fl & PAS_FLAG_INVALID) ? 1 : 0;
  ty.near1 += (fl & PAS_FLAG_NEAR_TOP1) ? 1 : 0;
  ty.nearT += (fl & PAS_FLAG_NEAR_THRESHOLD) ? 1 : 0;
}

// Block-wide reduction of the per-thread tallies, then one global atomic per non-zero counter.
__device__ __forceinline__ void flush_tally(const RouteParams& P, const SelectOut& o, const Tally& ty) {
  __shared__ int hist[kMaxLevels];
  __shared__ int cnt[3];
  __syncthreads();
  if (threadIdx.x < kMaxLevels) hist[threadIdx.x] = 0;
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int l = 0; l < kMaxLevels; ++l) {
    if (l >= P.nK) break;
    int v = (int)((ty.lv[l >> 2] >> ((l & 3) * 16)) & 0xFFFF);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&hist[l], v);
  }
  int a = ty.inv, b = ty.near1, c = ty.nearT;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(&cnt[0], a);
    if (b) atomicAdd(&cnt[1], b);
    if (c) atomicAdd(&cnt[2], c);
  }
  __syncthreads();
  if (threadIdx.x < P.nK && hist[threadIdx.x]) atomicAdd(&o.hist[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0) {
    if (cnt[0]) atomicAdd(&o.plan->n_invalid, cnt[0]);
    if (cnt[1]) atomicAdd(&o.plan->n_near_top1, cnt[1]);
    if (cnt[2]) atomicAdd(&o.plan->n_near_threshold, cnt[2]);
  }
}

// Warp per prompt (any S <= 128).
__global__ void __launch_bounds__(WARPS * 32) k_merge_select(const Cand* __restrict__ in, int S,
                                                             const uint8_t* __restrict__ pflags,
                                                             const __grid_constant__ RouteParams P, SelectOut o) {
  pdl_entry();
  __shared__ Cand res[WARPS][PAS_MAX_TOPK];
  Tally ty;
  ty.zero();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * WARPS + w;
  const int k = P.topk;
  if (p < P.N) {
    const bool invalid = pflags && (pflags[p] & PAS_FLAG_INVALID);
    const bool cold = (P.M_total == 0);
    if (invalid || cold) {
      if (lane == 0)
        for (int i = 0; i < k; ++i) res[w][i] = Cand{-INFINITY, -1};
    } else {
      merge_prompt(in, S, P.cand_stride ? P.cand_stride : P.N, k, p, res[w], lane);
    }
    __syncwarp();
    for (int i = lane; i < k; i += 32) {
      const Cand c = res[w][i];
      if (o.topk_id) o.topk_id[p * k + i] = c.g;
      if (o.topk_score) o.topk_score[p * k + i] = c.s;
      if (o.cand_out) o.cand_out[p * k + i] = c;
    }
    if (lane == 0) select_one(res[w][0].s, k > 1 ? res[w][1].s : -INFINITY, res[w][0].g, p, invalid, cold, P, o, ty);
  }
  flush_tally(P, o, ty);
}

// Thread per prompt for S * k <= 32 (the common case: R or G small).  All global traffic is
// coalesced 16-byte vectors through shared memory: the CTA's candidate rows of every source are
// staged in, each thread merges its S lists, and the CTA's top-k ids / scores leave as int4 rows.
constexpr int TP_THREADS = 128;
constexpr int TP_MAXSK = 32;

__global__ void __launch_bounds__(TP_THREADS) k_merge_select_thr(const Cand* __restrict__ in, int S,
                                                                 const uint8_t* __restrict__ pflags,
                                                                 const __grid_constant__ RouteParams P, SelectOut o) {
  pdl_entry();
  extern __shared__ __align__(16) Cand sm[];   // S * 128 * (k + 1) pairs (dynamic, padded rows)
  // after the merge the staging buffer is reused for the outgoing ids and scores (rows padded to k+1
  // words so the per-thread rows fall in different banks)
  const int kp = P.topk + 1;
  int32_t* sid = reinterpret_cast<int32_t*>(sm);
  float* ssc = reinterpret_cast<float*>(sm) + TP_THREADS * kp;
  Tally ty;
  ty.zero();
  const int k = P.topk;
  const bool cold = (P.M_total == 0);
  const int64_t stride = P.cand_stride ? P.cand_stride : P.N;
  const int64_t ntiles = (P.N + TP_THREADS - 1) / TP_THREADS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {   // persistent over tiles
    const int64_t p0 = tile * TP_THREADS;
    const int np = (int)min((int64_t)TP_THREADS, P.N - p0);
    __syncthreads();   // previous tile's output copy finished reading the staging buffer
    for (int s = 0; s < S; ++s) {   // coalesced global reads into rows padded to k+1 pairs
      const Cand* src = in + ((int64_t)s * stride + p0) * k;
      Cand* dst = sm + s * TP_THREADS * kp;
      for (int i = threadIdx.x; i < np * k; i += TP_THREADS) dst[(i / k) * kp + i % k] = src[i];
    }
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t p = p0 + t;
    Cand res[PAS_MAX_TOPK];
    bool invalid = false;
    if (t < np) {
      invalid = pflags && (pflags[p] & PAS_FLAG_INVALID);
      if (invalid || cold) {
#pragma unroll
        for (int i = 0; i < PAS_MAX_TOPK; ++i) res[i] = Cand{-INFINITY, -1};
      } else if (S == 1) {
#pragma unroll
        for (int i = 0; i < PAS_MAX_TOPK; ++i)
          if (i < k) res[i] = sm[t * kp + i];
      } else {
        int pos[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < PAS_MAX_TOPK; ++i) {
          if (i >= k) break;
          Cand best{-INFINITY, -1};
          int bs = -1;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            if (s < S && pos[s] < k) {
              const Cand c = sm[(s * TP_THREADS + t) * kp + pos[s]];
              if (bs < 0 || cand_better(c, best)) { best = c; bs = s; }
            }
          }
#pragma unroll
          for (int s = 0; s < 4; ++s)
            if (s == bs) pos[s]++;
          res[i] = best;
        }
      }
    }
    __syncthreads();   // every thread has read its candidates: the staging buffer becomes sid / ssc
    if (t < np) {
#pragma unroll
      for (int i = 0; i < PAS_MAX_TOPK; ++i) {
        if (i >= k) break;
        sid[t * kp + i] = res[i].g;
        ssc[t * kp + i] = res[i].s;
      }
      select_one(res[0].s, k > 1 ? res[1].s : -INFINITY, res[0].g, p, invalid, cold, P, o, ty);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * k; i += TP_THREADS) {   // coalesced global writes
      const int j = (i / k) * kp + i % k;
      if (o.topk_id) o.topk_id[p0 * k + i] = sid[j];
      if (o.topk_score) o.topk_score[p0 * k + i] = ssc[j];
      if (o.cand_out) o.cand_out[p0 * k + i] = Cand{ssc[j], sid[j]};
    }
  }
  flush_tally(P, o, ty);
}

// S == 1 (lists already merged, e.g. one cache range on one GPU): pure streaming.  Thread e owns the
// pair of candidates 2e, 2e+1 (one 16-byte load, two 8-byte stores, all coalesced); the thread that
// owns a prompt's first pair also does K4 for it.  Requires even k.
constexpr int S1_THREADS = 256;
#ifndef PAS_S1_UNROLL
#define PAS_S1_UNROLL 1   // 16-byte loads in flight per thread per step (2 and 4 measured equal, 8 slower)
#endif
constexpr int S1_UNROLL = PAS_S1_UNROLL;
template <int HALF>
__global__ void __launch_bounds__(S1_THREADS) k_select_s1(const int4* __restrict__ in,
                                                          const uint8_t* __restrict__ pflags, const __grid_constant__ RouteParams P,
                                                          SelectOut o) {
  pdl_entry();
  Tally ty;
  ty.zero();
  constexpr uint32_t half = HALF;
  const bool cold = (P.M_total == 0);
  const uint32_t total = (uint32_t)P.N * half;                    // <= 2^30
  const uint32_t stride = gridDim.x * S1_THREADS;
  // persistent grid-stride loop: one smem histogram flush per CTA (global atomics stay O(grid)).
  // S1_UNROLL independent 16-byte loads are issued before any is consumed (memory-level parallelism).
  for (uint32_t e0 = blockIdx.x * S1_THREADS + threadIdx.x; e0 < total; e0 += S1_UNROLL * stride) {
    int4 v[S1_UNROLL];
    uint8_t fl[S1_UNROLL];
#pragma unroll
    for (int u = 0; u < S1_UNROLL; ++u) {
      const uint32_t e = e0 + u * stride;
      if (e < total) {
        v[u] = __ldg(in + e);
        fl[u] = pflags ? __ldg(pflags + e / half) : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < S1_UNROLL; ++u) {
      const uint32_t e = e0 + u * stride;
      if (e >= total) break;
      const uint32_t p = e / half;
      Cand c0{__int_as_float(v[u].x), v[u].y}, c1{__int_as_float(v[u].z), v[u].w};
      const bool invalid = (fl[u] & PAS_FLAG_INVALID) != 0;
      if (invalid || cold) {
        c0 = Cand{-INFINITY, -1};
        c1 = c0;
      }
      if (o.topk_id) reinterpret_cast<int2*>(o.topk_id)[e] = make_int2(c0.g, c1.g);
      if (o.topk_score) reinterpret_cast<float2*>(o.topk_score)[e] = make_float2(c0.s, c1.s);
      if (o.cand_out) reinterpret_cast<int4*>(o.cand_out)[e] = make_int4(__float_as_int(c0.s), c0.g,
                                                                         __float_as_int(c1.s), c1.g);
      if (e == p * half) select_one(c0.s, c1.s, c0.g, p, invalid, cold, P, o, ty);
    }
  }
  flush_tally(P, o, ty);
}

// Explicit-N2 unpack: thread per (prompt, candidate pair); the prompt's first thread copies K / level /
// flags and stamps its top-1.
__global__ void __launch_bounds__(256) k_unpack_slices(const Cand* __restrict__ all_cand,
                                                       const int32_t* __restrict__ all_K,
                                                       const uint8_t* __restrict__ all_level,
                                                       const uint8_t* __restrict__ all_flags, const __grid_constant__ RouteParams P,
                                                       SelectOut o) {
  pdl_entry();
  const int k = P.topk;
  const int64_t total = P.N * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const Cand c = all_cand[e];
    PAS_CHECK(c.g < P.M_total, "explicit-N2 gathered candidate");
    if (o.topk_id) o.topk_id[e] = c.g;
    if (o.topk_score) o.topk_score[e] = c.s;
    const int64_t p = e / k;
    if (e == p * k) {
      const uint8_t fl = all_flags[p];
      o.K[p] = all_K[p];
      o.level[p] = all_level[p];
      if (o.flags) o.flags[p] = fl;
      if (P.lru_stamp && !(fl & (PAS_FLAG_INVALID | PAS_FLAG_COLD)) && c.g >= 0 && c.g < P.M_total)
        P.lru_stamp[c.g] = lru_tick_of(P);
    }
  }
}

__global__ void k_fill_sentinel(Cand* out, int64_t n) {
  pdl_entry();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = Cand{-INFINITY, -1};
}

}  // namespace

cudaError_t launch_merge(const Cand* in, int S, int64_t N, int k, Cand* out, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const int64_t blocks = (N + WARPS - 1) / WARPS;
  launch_pdl(k_merge, (unsigned)blocks, WARPS * 32, 0, st, in, S, N, k, out);
  return cudaGetLastError();
}

cudaError_t launch_merge_select(const Cand* in, int S, const uint8_t* pflags, const RouteParams& p,
                                const SelectOut& o, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  if (S == 1 && (p.topk & 1) == 0) {
    const int64_t threads = p.N * (p.topk >> 1);
    int64_t blocks = (threads + S1_THREADS - 1) / S1_THREADS;
    static const int per_sm = [] {   // resident CTAs per SM at this kernel's register count
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_select_s1<4>, S1_THREADS, 0) != cudaSuccess || n < 1)
        n = 4;
      return n;
    }();
    if (PAS_S1_GRIDCAP && blocks > (int64_t)kNumSMs * per_sm) blocks = (int64_t)kNumSMs * per_sm;   // one resident wave
    const unsigned g = (unsigned)blocks;
    const int4* in4 = reinterpret_cast<const int4*>(in);
    switch (p.topk >> 1) {
      case 1: launch_pdl(k_select_s1<1>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 2: launch_pdl(k_select_s1<2>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 3: launch_pdl(k_select_s1<3>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 4: launch_pdl(k_select_s1<4>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 5: launch_pdl(k_select_s1<5>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 6: launch_pdl(k_select_s1<6>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      case 7: launch_pdl(k_select_s1<7>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
      default: launch_pdl(k_select_s1<8>, g, S1_THREADS, 0, st, in4, pflags, p, o); break;
    }
  } else if (S <= 4 && S * p.topk <= TP_MAXSK) {
    int64_t blocks = (p.N + TP_THREADS - 1) / TP_THREADS;
    if (blocks > (int64_t)kNumSMs * 8) blocks = (int64_t)kNumSMs * 8;   // persistent CTAs
    // staging for S lists in, and ids + scores (= 1 list of pairs) out, rows padded to k+1 pairs
    const size_t smem = (size_t)(S > 1 ? S : 1) * TP_THREADS * (p.topk + 1) * sizeof(Cand);
    launch_pdl(k_merge_select_thr, (unsigned)blocks, TP_THREADS, smem, st, in, S, pflags, p, o);
  } else {
    const int64_t blocks = (p.N + WARPS - 1) / WARPS;
    launch_pdl(k_merge_select, (unsigned)blocks, WARPS * 32, 0, st, in, S, pflags, p, o);
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack_slices(const Cand* all_cand, const int32_t* all_K, const uint8_t* all_level,
                                 const uint8_t* all_flags, const RouteParams& p, const SelectOut& o,
                                 cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  int64_t blocks = (p.N * p.topk + 255) / 256;
  if (blocks > (int64_t)kNumSMs * 8) blocks = (int64_t)kNumSMs * 8;
  launch_pdl(k_unpack_slices, (unsigned)blocks, 256, 0, st, all_cand, all_K, all_level, all_flags, p, o);
  return cudaGetLastError();
}

cudaError_t launch_fill_sentinel(Cand* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  launch_pdl(k_fill_sentinel, (unsigned)blocks, 256, 0, st, out, n);
  return cudaGetLastError();
}

}  // namespace pas
