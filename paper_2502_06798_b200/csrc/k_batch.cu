// K7 -- load-aware route-and-batch: per prompt a serving instance and a FIFO slot,
// then per-instance batch lists (counting sort).
//
// Greedy (high load, R13): t_p = #{p' < p : K'_p' = K'_p}; instance = I_j[(t div b*) mod n_j],
//   slot = (t div (b* n_j)) b* + t mod b* -- fill I_j[0] up to b*, then I_j[1], ..., then wrap, so
//   every instance's queue fires at the optimal batch size b* ("selecting the worker likely to be
//   fired soonest at optimal batch size").
// Uniform (low load, R14): instance chosen by Philox in K6; slot = FIFO rank among the prompts of that
//   instance (batch size 1).
// Both need the stable rank t of every prompt among the prompts of its class (C classes: the nK <= 16
// K' levels in greedy mode, the W <= 64 instances in uniform mode) in prompt order.  Tiles of 1024
// prompts, 4 consecutive prompts per thread (16-byte loads and stores, no shared-memory staging):
//   k_cls_count  per-tile class counts, written class-major [64][tiles]
//   scan         device-wide exclusive scan of that array: entry (c, b) = prompts of classes < c plus
//                prompts of class c in tiles < b
//   k_cls_rank   t = scan(c, b) - scan(c, 0) + rank inside the tile: per warp, one ballot per class and
//                element slot (popc of the lanes below), per block an exclusive prefix over the 8 warps.
//   k_offsets    per-instance counts in closed form from the class totals (greedy: each I_j[m] gets
//                the t's whose (t div b*) mod n_j = m), their exclusive scan (the batch-list offsets)
//   k_bucket     scatter prompt ids to offsets[instance] + slot.
// HBM per prompt: class 4 B read twice, instance + slot 8 B written, bucket list 8 B read + 4 B written.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int THREADS = 256;
constexpr int PER = 4;                   // prompts per thread
constexpr int TILE = THREADS * PER;      // prompts per CTA
constexpr int NCLS = 64;
constexpr int WARPS = THREADS / 32;

__device__ __forceinline__ void load4(const int32_t* __restrict__ src, int64_t base, int n, int (&v)[PER]) {
  const int i0 = PER * threadIdx.x;
  if (i0 + PER - 1 < n) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(src + base) + threadIdx.x);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = (i0 + j < n) ? src[base + i0 + j] : -1;
  }
}
__device__ __forceinline__ void store4(int32_t* __restrict__ dst, int64_t base, int n, const int (&v)[PER]) {
  const int i0 = PER * threadIdx.x;
  if (i0 + PER - 1 < n) {
    reinterpret_cast<int4*>(dst + base)[threadIdx.x] = make_int4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (i0 + j < n) dst[base + i0 + j] = v[j];
  }
}

// Warp-level class ranking by ballots (uniform loop over the C <= 64 classes): for an element of
// class c held by lane l at position j of its 4, the number of earlier class-c elements in the warp
// is  sum_k popc(ballot_k(class == c) & lanes_below(l))  +  #{k < j : v[k] == c}.  Lane (c mod 32)
// ends with the warp's total of class c in lane_total[c / 32].
__device__ __forceinline__ void warp_class_rank(const int (&v)[PER], int nC, int (&r)[PER], int (&lane_total)[2]) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
#pragma unroll
  for (int j = 0; j < PER; ++j) r[j] = 0;
  lane_total[0] = lane_total[1] = 0;
  for (int c = 0; c < nC; ++c) {
    int before = 0, tot = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const unsigned b = __ballot_sync(0xffffffffu, v[j] == c);
      before += __popc(b & lt);
      tot += __popc(b);
    }
    int mine = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (v[j] == c) r[j] = before + mine;
      mine += (v[j] == c) ? 1 : 0;
    }
    if (lane == (c & 31)) lane_total[c >> 5] = tot;
  }
}

__global__ void __launch_bounds__(THREADS) k_cls_count(const int32_t* __restrict__ cls, int64_t N, int ntiles,
                                                       int nC, int32_t* __restrict__ counts /*[64][ntiles]*/) {
  pdl_entry();
  __shared__ int32_t cnt[NCLS];
  if (threadIdx.x < NCLS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * TILE;
  const int n = (int)min((int64_t)TILE, N - base);
  int v[PER];
  load4(cls, base, n, v);
  const int lane = threadIdx.x & 31;
  int r[PER], tot[2];
  warp_class_rank(v, nC, r, tot);
  if (lane < nC && tot[0]) atomicAdd(&cnt[lane], tot[0]);
  if (lane + 32 < nC && tot[1]) atomicAdd(&cnt[lane + 32], tot[1]);
  __syncthreads();
  if (threadIdx.x < NCLS) counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(THREADS) k_cls_rank(const int32_t* __restrict__ cls, const RouteParams P,
                                                      int ntiles, int nC, const int32_t* __restrict__ scanned,
                                                      const DevPlan* __restrict__ plan, int32_t* __restrict__ instance,
                                                      int32_t* __restrict__ slot) {
  pdl_entry();
  __shared__ int32_t wcnt[WARPS][NCLS];    // per-warp class totals, then exclusive prefix over warps
  __shared__ int32_t tile_off[NCLS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * TILE;
  const int n = (int)min((int64_t)TILE, P.N - base);
  if (threadIdx.x < NCLS) {
    const int64_t row = (int64_t)threadIdx.x * ntiles;
    tile_off[threadIdx.x] = scanned[row + tile] - scanned[row];
  }
  int c[PER];
  load4(cls, base, n, c);
  int r[PER], tot[2];
  warp_class_rank(c, nC, r, tot);
  wcnt[w][lane] = lane < nC ? tot[0] : 0;
  wcnt[w][lane + 32] = lane + 32 < nC ? tot[1] : 0;
  __syncthreads();
  if (threadIdx.x < NCLS) {   // exclusive prefix over warps, per class
    int run = 0;
    for (int v2 = 0; v2 < WARPS; ++v2) {
      const int x = wcnt[v2][threadIdx.x];
      wcnt[v2][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
  int inst[PER], sl[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    inst[j] = -1;
    sl[j] = 0;
    if (c[j] < 0) continue;
    const int t = tile_off[c[j]] + wcnt[w][c[j]] + r[j];
    if (P.mode == PAS_UNIFORM) {
      inst[j] = c[j];
      sl[j] = t;
    } else {
      // q1 = t div b*, q2 = q1 div n_j (exact multiply-high, t < 2^26, n_j <= 64):
      // instance I_j[q1 mod n_j], slot q2 * b* + t mod b*
      const uint32_t b = (uint32_t)P.bstar;
      const uint32_t q1 = P.bstar_shift >= 0 ? ((uint32_t)t >> P.bstar_shift) : (uint32_t)t / b;
      const uint32_t q2 = (uint32_t)(((uint64_t)q1 * plan->n_inst_magic[c[j]]) >> 32);
      inst[j] = plan->inst_list[c[j]][q1 - q2 * (uint32_t)plan->n_inst[c[j]]];
      sl[j] = (int)(q2 * b + ((uint32_t)t - q1 * b));
    }
  }
  store4(instance, base, n, inst);
  store4(slot, base, n, sl);
}

// Per-instance counts from the class totals (scan of the class-major counts), then offsets.
__global__ void k_offsets(const int32_t* __restrict__ scanned, int ntiles, int64_t N, const RouteParams P,
                          DevPlan* __restrict__ plan, int32_t* __restrict__ off, int32_t* __restrict__ user_off) {
  pdl_entry();
  if (threadIdx.x != 0) return;
  const int nC = P.mode == PAS_UNIFORM ? P.W : P.nK;
  int count[kMaxInst];
  for (int w = 0; w < P.W; ++w) count[w] = 0;
  for (int c = 0; c < nC; ++c) {
    const int64_t start = scanned[(int64_t)c * ntiles];
    const int64_t end = c + 1 < NCLS ? scanned[(int64_t)(c + 1) * ntiles] : N;
    const int total = (int)(end - start);
    if (P.mode == PAS_UNIFORM) {
      count[c] = total;
    } else {
      const int nj = plan->n_inst[c], b = P.bstar;
      if (nj == 0) continue;
      const int full = total / (b * nj), rem = total % (b * nj);
      for (int m = 0; m < nj; ++m) {
        const int extra = rem - m * b;
        count[plan->inst_list[c][m]] = full * b + (extra < 0 ? 0 : (extra > b ? b : extra));
      }
    }
  }
  int run = 0;
  for (int w = 0; w <= P.W; ++w) {
    off[w] = run;
    if (user_off) user_off[w] = run;
    if (w < P.W) {
      plan->inst_count[w] = count[w];
      run += count[w];
    }
  }
}

// 4 prompts per thread (16-byte loads of instance and slot), scattered 4-byte stores.
__global__ void k_bucket(const int32_t* __restrict__ instance, const int32_t* __restrict__ slot, int64_t N,
                         const int32_t* __restrict__ off, int32_t* __restrict__ prompts) {
  pdl_entry();
  __shared__ int32_t soff[NCLS + 1];
  if (threadIdx.x <= NCLS) soff[threadIdx.x] = off[threadIdx.x];
  __syncthreads();
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (p0 + 3 < N) {
    const int4 in = __ldg(reinterpret_cast<const int4*>(instance + p0));
    const int4 sl = __ldg(reinterpret_cast<const int4*>(slot + p0));
    prompts[soff[in.x] + sl.x] = (int32_t)p0;
    prompts[soff[in.y] + sl.y] = (int32_t)(p0 + 1);
    prompts[soff[in.z] + sl.z] = (int32_t)(p0 + 2);
    prompts[soff[in.w] + sl.w] = (int32_t)(p0 + 3);
  } else {
    for (int64_t p = p0; p < N; ++p) prompts[soff[instance[p]] + slot[p]] = (int32_t)p;
  }
}

}  // namespace

int batch_tiles(int64_t N) { return (int)((N + TILE - 1) / TILE); }

cudaError_t launch_route_and_batch(const RedirectWs& r, const RouteParams& p, DevPlan* plan, const BatchWs& w,
                                   int32_t* instance, int32_t* slot, int32_t* bucket_offsets,
                                   int32_t* bucket_prompts, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  const int ntiles = batch_tiles(p.N);
  const int nclasses = p.mode == PAS_UNIFORM ? p.W : p.nK;
  launch_pdl(k_cls_count, ntiles, THREADS, 0, st, r.cls7, p.N, ntiles, nclasses, w.blk_counts);
  cudaError_t e = launch_exclusive_scan(w.blk_counts, w.blk_off, NCLS * ntiles, w.scan_tmp, st, launches);
  if (e != cudaSuccess) return e;
  launch_pdl(k_cls_rank, ntiles, THREADS, 0, st, r.cls7, p, ntiles, nclasses, w.blk_off, plan, instance, slot);
  *launches += 2;
  if (e != cudaSuccess) return e;
  launch_pdl(k_offsets, 1, 32, 0, st, w.blk_off, ntiles, p.N, p, plan, w.offsets, bucket_offsets);
  *launches += 1;
  if (bucket_prompts) {
    launch_pdl(k_bucket, (unsigned)((p.N + 1023) / 1024), 256, 0, st, instance, slot, p.N, w.offsets, bucket_prompts);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace pas
