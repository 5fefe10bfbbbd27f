// K7 -- load-aware route-and-batch: per prompt a serving instance and a FIFO slot,
// then per-instance batch lists (counting sort).
//
// Greedy (high load, R13): t_p = #{p' < p : K'_p' = K'_p}; instance = I_j[(t div b*) mod n_j],
//   slot = (t div (b* n_j)) b* + t mod b* -- fill I_j[0] up to b*, then I_j[1], ..., then wrap, so
//   every instance's queue fires at the optimal batch size b* ("selecting the worker likely to be
//   fired soonest at optimal batch size").
// Uniform (low load, R14): instance chosen by Philox in K6; slot = FIFO rank among the prompts of that
//   instance (batch size 1).
// Both need a stable rank of every prompt among the prompts of its class (C <= 64 classes) in prompt
// order: k_cls_count (per-CTA class counts, 1024 prompts per CTA), k_cls_scan (per-class exclusive
// scan over CTAs), k_cls_rank (warp __match_any_sync + per-warp counts in smem); then k_offsets (one
// CTA, exclusive scan of the W instance counts) and k_bucket (scatter prompt ids to
// offsets[instance] + slot).
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int TILE = 1024;
constexpr int NCLS = 64;

__global__ void __launch_bounds__(TILE) k_cls_count(const int32_t* __restrict__ cls, int64_t N,
                                                    int32_t* __restrict__ blk_counts) {
  __shared__ int32_t cnt[NCLS];
  if (threadIdx.x < NCLS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * TILE + threadIdx.x;
  if (p < N) atomicAdd(&cnt[cls[p]], 1);
  __syncthreads();
  if (threadIdx.x < NCLS) blk_counts[(int64_t)blockIdx.x * NCLS + threadIdx.x] = cnt[threadIdx.x];
}

__global__ void k_cls_scan(const int32_t* __restrict__ blk_counts, int nblk, int32_t* __restrict__ blk_off) {
  const int c = threadIdx.x;   // one thread per class
  if (c >= NCLS) return;
  int run = 0;
  for (int b = 0; b < nblk; ++b) {
    const int v = blk_counts[(int64_t)b * NCLS + c];
    blk_off[(int64_t)b * NCLS + c] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(TILE) k_cls_rank(const int32_t* __restrict__ cls, RouteParams P,
                                                   const int32_t* __restrict__ blk_off, DevPlan* __restrict__ plan,
                                                   int32_t* __restrict__ instance, int32_t* __restrict__ slot) {
  __shared__ int32_t wcnt[TILE / 32][NCLS];
  __shared__ int32_t icnt[NCLS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (TILE / 32) * NCLS; i += TILE) (&wcnt[0][0])[i] = 0;
  if (threadIdx.x < NCLS) icnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * TILE + threadIdx.x;
  const bool live = p < P.N;
  const int c = live ? cls[p] : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, c);
  const int inwarp = __popc(peers & ((1u << lane) - 1));
  if (live && inwarp == 0) wcnt[w][c] = __popc(peers);
  __syncthreads();
  if (live) {
    int t = blk_off[(int64_t)blockIdx.x * NCLS + c] + inwarp;
    for (int v = 0; v < w; ++v) t += wcnt[v][c];
    int inst, sl;
    if (P.mode == PAS_UNIFORM) {
      inst = c;
      sl = t;
    } else {
      const int nj = plan->n_inst[c];
      const int b = P.bstar;
      inst = plan->inst_list[c][(t / b) % nj];
      sl = (t / (b * nj)) * b + t % b;
    }
    instance[p] = inst;
    slot[p] = sl;
    atomicAdd(&icnt[inst], 1);
  }
  __syncthreads();
  if (threadIdx.x < P.W && icnt[threadIdx.x]) atomicAdd(&plan->inst_count[threadIdx.x], icnt[threadIdx.x]);
}

__global__ void k_offsets(const DevPlan* __restrict__ plan, int W, int32_t* __restrict__ off,
                          int32_t* __restrict__ user_off) {
  if (threadIdx.x != 0) return;
  int run = 0;
  for (int w = 0; w <= W; ++w) {
    off[w] = run;
    if (user_off) user_off[w] = run;
    if (w < W) run += plan->inst_count[w];
  }
}

__global__ void k_bucket(const int32_t* __restrict__ instance, const int32_t* __restrict__ slot, int64_t N,
                         const int32_t* __restrict__ off, int32_t* __restrict__ prompts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  prompts[off[instance[p]] + slot[p]] = (int32_t)p;
}

}  // namespace

cudaError_t launch_route_and_batch(const RedirectWs& r, const RouteParams& p, DevPlan* plan, const BatchWs& w,
                                   int32_t* instance, int32_t* slot, int32_t* bucket_offsets,
                                   int32_t* bucket_prompts, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  const int nblk = (int)((p.N + TILE - 1) / TILE);
  k_cls_count<<<nblk, TILE, 0, st>>>(r.cls7, p.N, w.blk_counts);
  k_cls_scan<<<1, NCLS, 0, st>>>(w.blk_counts, nblk, w.blk_off);
  k_cls_rank<<<nblk, TILE, 0, st>>>(r.cls7, p, w.blk_off, plan, instance, slot);
  *launches += 3;
  if (bucket_offsets || bucket_prompts) {
    k_offsets<<<1, 32, 0, st>>>(plan, p.W, w.offsets, bucket_offsets);
    *launches += 1;
    if (bucket_prompts) {
      k_bucket<<<(unsigned)((p.N + 255) / 256), 256, 0, st>>>(instance, slot, p.N, w.offsets, bucket_prompts);
      *launches += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace pas
