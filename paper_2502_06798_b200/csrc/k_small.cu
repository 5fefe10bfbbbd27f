// K3..K7 fused for small batches -- the latency path (low loads are served for
// latency).  For N <= kSmallMax prompts the multi-kernel downstream (merge +
// optimal-K, plan, 6 redirect kernels, count / scan / rank) is a chain of ~11 launches of a few
// microseconds each; here ONE CTA of 1024 threads runs all of it from the K2 candidates:
//   a4/a5  S-way merge of the sorted candidate lists (score desc, gid asc, ties to the lower source,
//          R10) -- eight lanes per prompt with a shuffle tournament per output when S, k <= 8, else a
//          thread per prompt --, optimal-K level #{m : s1 >= t_m}, flags, LRU stamp of the top-1
//          (R26), H_K and the flag counters in shared memory;
//   a6     warp 0: the Eq. 1 plan (plan_body: the same code as K5);
//   a7     kappa_p = Philox(p) (stream 1), the class rank of (kappa, p) by counting (O(N) per prompt over
//          shared memory), K' from the plan's row prefix (R3) -- the order statistic K6 selects;
//   a8     greedy: t = #{q < p : K'_q = K'_p}, instance I_j[(t div b*) mod n_j], slot (R13); uniform:
//          instance by Philox stream 2, slot = FIFO rank (R14); per-instance counts, offsets and the
//          batch lists.
// Same definitions, same fp32 / fp64 operations as the multi-kernel path: the outputs are byte-
// identical to it (tests/test_gpu_graph.py forces both paths on the same batches).  Stateless
// exact-plan modes only (the forecast f1 and dispatcher f3 modes take the multi-kernel path).
#include "philox.cuh"
#include "plan_body.cuh"

namespace pas {
namespace {

constexpr int SM_THREADS = 1024;
constexpr int kStageCands = 2048;   // candidate pairs staged in shared memory (16 KB) when they fit

__global__ void __launch_bounds__(SM_THREADS, 1) k_small_route(const Cand* __restrict__ in, int S,
                                                               const uint8_t* __restrict__ pflags,
                                                               const RouteParams P, SmallOut o) {
  pdl_entry();
  __shared__ uint8_t lvl_s[kSmallMax], cls_s[kSmallMax];
  __shared__ uint64_t kap_s[kSmallMax];
  __shared__ int hist_s[kMaxLevels];
  __shared__ int cnt_s[3];
  __shared__ DevPlan plan_s;          // the batch's plan lives in shared memory, copied out at the end
  __shared__ int icount_s[kMaxInst], ioff_s[kMaxInst + 1];
  __shared__ Cand cand_s[kStageCands];
  const int tid = threadIdx.x;
  const int N = (int)P.N, k = P.topk, nK = P.nK;
  const bool cold = P.M_total == 0;
  {   // zero the plan (as launch_zero does for the multi-kernel path) and the shared tallies
    int32_t* w = reinterpret_cast<int32_t*>(&plan_s);
    for (int i = tid; i < (int)(sizeof(DevPlan) / 4); i += SM_THREADS) w[i] = 0;
    if (tid < kMaxLevels) hist_s[tid] = 0;
    if (tid < 3) cnt_s[tid] = 0;
    if (tid < kMaxInst) icount_s[tid] = 0;
  }
  __syncthreads();
  const uint32_t tick = lru_tick_of(P);
  const int64_t stride = P.cand_stride ? P.cand_stride : P.N;
  // all S x N x k candidates in shared memory when they fit (one coalesced pass, every load in flight),
  // else the merge reads them from L2
  const bool staged = (int64_t)S * N * k <= kStageCands;
  if (staged) {
    const int per = N * k;
    for (int e = tid; e < S * per; e += SM_THREADS) {
      const int s = e / per, r = e - s * per;
      cand_s[e] = in[(int64_t)s * stride * k + r];
    }
  }
  __syncthreads();
  // ---- a4 + a5: merge, optimal-K, flags, stamps, H_K
  // select_one of k_merge.cu for prompt p with its merged s1, s2 (-inf for k = 1) and top-1 id
  auto finish = [&](int p, bool invalid, float s1, float s2, int32_t g1) {
    int lv = 0;
    uint8_t fl = 0;
    if (invalid) fl |= PAS_FLAG_INVALID;
    else if (cold) fl |= PAS_FLAG_COLD;
    else {
#pragma unroll
      for (int step = 8; step >= 1; step >>= 1)
        if (s1 >= P.thr[lv + step - 1]) lv += step;
      if (s2 != -INFINITY && s1 - s2 < 2e-2f) fl |= PAS_FLAG_NEAR_TOP1;
      if ((lv > 0 && s1 - P.thr[lv - 1] < 2e-2f) || (lv < nK - 1 && P.thr[lv] - s1 < 2e-2f))
        fl |= PAS_FLAG_NEAR_THRESHOLD;
    }
    if (P.lru_stamp && !invalid && !cold && g1 >= 0 && g1 < P.M_total) P.lru_stamp[g1] = tick;
    lvl_s[p] = (uint8_t)lv;
    o.level[p] = (uint8_t)lv;
    o.K[p] = P.grid[lv];
    if (o.flags) o.flags[p] = fl;
    atomicAdd(&hist_s[lv], 1);
    if (fl & PAS_FLAG_INVALID) atomicAdd(&cnt_s[0], 1);
    if (fl & PAS_FLAG_NEAR_TOP1) atomicAdd(&cnt_s[1], 1);
    if (fl & PAS_FLAG_NEAR_THRESHOLD) atomicAdd(&cnt_s[2], 1);
  };
  if (S <= 8 && k <= 8) {
    // eight lanes per prompt, lane g holding source list g in registers; each round a width-8
    // shuffle tournament takes the best head (score desc, gid asc, then the lower source, R10) and its
    // lane advances -- k rounds of three shuffle steps instead of k * S dependent shared loads on one
    // thread (64 prompts: all of them at once on 512 threads)
    const int g = tid & 7;
    for (int base = 0; base < N * 8; base += SM_THREADS) {
      const int p = (base + tid) >> 3;
      const bool act = p < N;   // group-uniform; whole warps shuffle (inactive groups carry padding)
      const bool invalid = act && pflags && (pflags[p] & PAS_FLAG_INVALID);
      const bool live = act && !invalid && !cold && g < S;
      Cand L[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        L[i] = (live && i < k) ? (staged ? cand_s[(g * N + p) * k + i] : in[((int64_t)g * stride + p) * k + i])
                               : Cand{-INFINITY, -1};
      float s1 = -INFINITY, s2 = -INFINITY;
      int32_t g1 = -1;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i >= k) break;
        float bs = L[0].s;
        int32_t bg = L[0].g;
        int bsrc = g;
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
          const float os = __shfl_xor_sync(0xffffffffu, bs, off, 8);
          const int32_t og = __shfl_xor_sync(0xffffffffu, bg, off, 8);
          const int osrc = __shfl_xor_sync(0xffffffffu, bsrc, off, 8);
          if (os > bs || (os == bs && ((unsigned)og < (unsigned)bg || (og == bg && osrc < bsrc)))) {
            bs = os;
            bg = og;
            bsrc = osrc;
          }
        }
        if (bsrc == g) {   // this lane's head was taken: advance
#pragma unroll
          for (int j = 0; j < 7; ++j) L[j] = L[j + 1];
          L[7] = Cand{-INFINITY, -1};
        }
        if (act && g == (i & 7)) {
          if (o.topk_id) o.topk_id[(int64_t)p * k + i] = bg;
          if (o.topk_score) o.topk_score[(int64_t)p * k + i] = bs;
        }
        if (i == 0) {
          s1 = bs;
          g1 = bg;
        } else if (i == 1) {
          s2 = bs;
        }
      }
      if (act && g == 0) finish(p, invalid, s1, s2, g1);
    }
  } else {   // a thread per prompt
    for (int p = tid; p < N; p += SM_THREADS) {
      const bool invalid = pflags && (pflags[p] & PAS_FLAG_INVALID);
      // each merged entry goes straight to the outputs; s1, s2 and the top-1 id stay in registers
      // (a per-thread result array would live in local memory)
      float s1 = -INFINITY, s2 = -INFINITY;
      int32_t g1 = -1;
      auto emit = [&](int i, const Cand& c) {
        if (o.topk_id) o.topk_id[(int64_t)p * k + i] = c.g;
        if (o.topk_score) o.topk_score[(int64_t)p * k + i] = c.s;
        if (i == 0) {
          s1 = c.s;
          g1 = c.g;
        } else if (i == 1) {
          s2 = c.s;
        }
      };
      if (invalid || cold) {
        for (int i = 0; i < k; ++i) emit(i, Cand{-INFINITY, -1});
      } else if (S <= 8) {
        int pos[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < k; ++i) {
          Cand best{-INFINITY, -1};
          int bs = -1;
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            if (s >= S || pos[s] >= k) continue;
            const Cand c = staged ? cand_s[(s * N + p) * k + pos[s]] : in[((int64_t)s * stride + p) * k + pos[s]];
            if (bs < 0 || cand_better(c, best)) {
              best = c;
              bs = s;
            }
          }
#pragma unroll
          for (int s = 0; s < 8; ++s) pos[s] += s == bs ? 1 : 0;
          emit(i, bs >= 0 ? best : Cand{-INFINITY, -1});
        }
      } else {
        uint8_t pos[128];
        for (int s = 0; s < S; ++s) pos[s] = 0;
        for (int i = 0; i < k; ++i) {
          Cand best{-INFINITY, -1};
          int bs = -1;
          for (int s = 0; s < S; ++s) {
            if (pos[s] >= k) continue;
            PAS_CHECK(p < stride, "small path candidate row");
            const Cand c = staged ? cand_s[(s * N + p) * k + pos[s]] : in[((int64_t)s * stride + p) * k + pos[s]];
            if (bs < 0 || cand_better(c, best)) {
              best = c;
              bs = s;
            }
          }
          if (bs >= 0) pos[bs]++;
          emit(i, bs >= 0 ? best : Cand{-INFINITY, -1});
        }
      }
      finish(p, invalid, s1, s2, g1);
    }
  }
  __syncthreads();
  // ---- a6: the plan, one warp (the same code as K5)
  if (tid < 32) plan_body(hist_s, P, &plan_s, false);   // no K6 windows: a7 ranks by counting
  if (tid == 0) {
    plan_s.n_invalid = cnt_s[0];
    plan_s.n_near_top1 = cnt_s[1];
    plan_s.n_near_threshold = cnt_s[2];
  }
  const uint64_t bseq = batch_seq_of(P);
  for (int p = tid; p < N; p += SM_THREADS) {
    const uint4 w = philox_stream(P.seed, bseq, (uint32_t)p, kStreamRedirect);
    kap_s[p] = (((uint64_t)w.y << 32) | w.x) >> 4;
  }
  __syncthreads();
  // ---- a7: class rank of (kappa, p), K' from the row prefix of the plan.  G threads per prompt
  // (G = 1024 / N rounded down to a power of two, <= 32) split the count and reduce by shuffles.
  int G = 1;
  while (G < 32 && G * 2 * N <= SM_THREADS) G *= 2;
  const int sub = tid & (G - 1);
  for (int base = 0; base < N * G; base += SM_THREADS) {
    const int p = (base + tid) / G;
    const bool act = p < N;
    const int i = act ? lvl_s[p] : 0;
    const uint64_t kp = act ? kap_s[p] : 0;
    int r = 0;
    if (act)
      for (int q = sub; q < N; q += G)
        r += (lvl_s[q] == i && (kap_s[q] < kp || (kap_s[q] == kp && q < p))) ? 1 : 0;
    for (int off = G >> 1; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    if (!act || sub != 0) continue;
    int j = 0;
    while (j + 1 < nK && plan_s.X[i][j] <= r) ++j;
    o.K_prime[p] = P.grid[j];
    int c = j;
    if (P.mode == PAS_UNIFORM) {
      const uint4 u = philox_stream(P.seed, bseq, (uint32_t)p, kStreamUniform);
      c = plan_s.inst_list[j][(uint32_t)(((uint64_t)u.x * (uint32_t)plan_s.n_inst[j]) >> 32)];
    }
    cls_s[p] = (uint8_t)c;
  }
  __syncthreads();
  // ---- a8: instance and slot (FIFO rank within the class), then the batch lists
  for (int base = 0; base < N * G; base += SM_THREADS) {
    const int p = (base + tid) / G;
    const bool act = p < N;
    const int c = act ? cls_s[p] : 0;
    int t = 0;
    if (act)
      for (int q = sub; q < p; q += G) t += cls_s[q] == c ? 1 : 0;
    for (int off = G >> 1; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (!act || sub != 0) continue;
    int inst, sl;
    if (P.mode == PAS_UNIFORM) {
      inst = c;
      sl = t;
    } else {
      const int b = P.bstar, nj = plan_s.n_inst[c];
      const int q1 = t / b;
      inst = plan_s.inst_list[c][q1 % nj];
      sl = (q1 / nj) * b + t % b;
    }
    PAS_CHECK(inst >= 0 && inst < P.W && sl >= 0, "small path instance / slot");
    o.instance[p] = inst;
    o.slot[p] = sl;
    atomicAdd(&icount_s[inst], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < P.W; ++w) {
      ioff_s[w] = acc;
      acc += icount_s[w];
      plan_s.inst_count[w] = icount_s[w];
    }
    ioff_s[P.W] = acc;
  }
  __syncthreads();
  if (o.bucket_offsets && tid <= P.W) o.bucket_offsets[tid] = ioff_s[tid];
  if (o.bucket_prompts)
    for (int p = tid; p < N; p += SM_THREADS) o.bucket_prompts[ioff_s[o.instance[p]] + o.slot[p]] = p;
  {   // the plan and counters for pas_plan_stats
    const int32_t* src = reinterpret_cast<const int32_t*>(&plan_s);
    int32_t* dst = reinterpret_cast<int32_t*>(o.plan);
    for (int i = tid; i < (int)(sizeof(DevPlan) / 4); i += SM_THREADS) dst[i] = src[i];
  }
  __syncthreads();
  advance_batch_counters(P);   // after every read of the counters in this batch
}

}  // namespace

cudaError_t launch_small_route(const Cand* in, int S, const uint8_t* pflags, const RouteParams& p, const SmallOut& o,
                               cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  launch_pdl(k_small_route, 1, SM_THREADS, 0, st, in, S, pflags, p, o);
  return cudaGetLastError();
}

}  // namespace pas
