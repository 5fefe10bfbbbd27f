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
// K' levels in greedy mode, the W <= 64 instances in uniform mode) in prompt order.  The class is a
// byte per prompt.  Tiles of 4096 prompts; each warp takes 512 consecutive prompts as ROWS = 16 rows
// of 32 (lane l of row j holds prompt 32 j + l; coalesced loads, all 16 in flight before any compute):
//   k_cls_count  per-tile class counts, written class-major [C][tiles]
//   scan         device-wide exclusive scan of that array: entry (c, b) = prompts of classes < c plus
//                prompts of class c in tiles < b
//   k_cls_rank   t = scan(c, b) - scan(c, 0) + rank inside the tile.  Inside a warp, row by row:
//                match.any gives the lanes holding the same class, popc of those below a lane is its
//                rank in the row, and a per-warp running count per class (shared memory, bumped by the
//                lowest lane of each match group) carries the earlier rows; per block an exclusive
//                prefix over the 8 warps.  Cost per row is independent of C.  Block 0 also turns the
//                class totals into per-instance counts (closed form, greedy: each I_j[m] gets the t's
//                whose (t div b*) mod n_j = m) and the batch-list offsets.
//   k_bucket     scatter prompt ids to offsets[instance] + slot.
// (A single-pass decoupled look-back variant was 60 % slower at 64M prompts: with ~1200 tiles in
// flight the look-back walks hundreds of predecessors per tile.)
// HBM per prompt: class 1 B read twice, instance + slot 8 B written, bucket list 8 B read + 4 B written.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int ROWS = 16;                       // rows of 32 prompts per warp
constexpr int TILE = THREADS * ROWS;           // prompts per CTA
constexpr int NCLS = 64;

// Row j of this warp's chunk: prompt base + 32 j + lane (-1 past the end).
__device__ __forceinline__ void load_rows(const uint8_t* __restrict__ src, int64_t base, int64_t N, int (&v)[ROWS]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const int64_t p = base + 32 * j + lane;
    v[j] = p < N ? (int)__ldg(src + p) : -1;
  }
}

__global__ void __launch_bounds__(THREADS) k_cls_count(const uint8_t* __restrict__ cls, int64_t N, int ntiles,
                                                       int nC, int32_t* __restrict__ counts /*[nC][ntiles]*/) {
  pdl_entry();
  __shared__ int32_t cnt[NCLS];
  if (threadIdx.x < NCLS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int v[ROWS];
  load_rows(cls, (int64_t)blockIdx.x * TILE + w * 32 * ROWS, N, v);
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const unsigned m = __match_any_sync(0xffffffffu, v[j]);
    if (v[j] >= 0 && lane == __ffs(m) - 1) atomicAdd(&cnt[v[j]], __popc(m));
  }
  __syncthreads();
  if (threadIdx.x < nC) counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(THREADS) k_cls_rank(const uint8_t* __restrict__ cls, const RouteParams P,
                                                      int ntiles, int nC, const int32_t* __restrict__ scanned,
                                                      DevPlan* __restrict__ plan, int32_t* __restrict__ instance,
                                                      int32_t* __restrict__ slot, int32_t* __restrict__ off,
                                                      int32_t* __restrict__ user_off) {
  pdl_entry();
  __shared__ int32_t wcnt[WARPS][NCLS];    // per-warp running class counts, then exclusive prefix over warps
  __shared__ int32_t tile_off[NCLS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * TILE + w * 32 * ROWS;
  int c[ROWS];
  load_rows(cls, base, P.N, c);
  for (int i = threadIdx.x; i < WARPS * NCLS; i += THREADS) (&wcnt[0][0])[i] = 0;
  if (threadIdx.x < nC) {
    const int64_t row = (int64_t)threadIdx.x * ntiles;
    tile_off[threadIdx.x] = scanned[row + tile] - scanned[row];
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1;
  int r[ROWS];
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const unsigned m = __match_any_sync(0xffffffffu, c[j]);
    const bool lead = lane == __ffs(m) - 1;
    r[j] = c[j] >= 0 ? wcnt[w][c[j]] + __popc(m & lt) : 0;
    __syncwarp();
    if (lead && c[j] >= 0) wcnt[w][c[j]] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < nC) {   // exclusive prefix over warps, per class
    int run = 0;
    for (int v2 = 0; v2 < WARPS; ++v2) {
      const int x = wcnt[v2][threadIdx.x];
      wcnt[v2][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const int64_t p = base + 32 * j + lane;
    if (c[j] < 0) continue;
    const int t = tile_off[c[j]] + wcnt[w][c[j]] + r[j];
    int inst, sl;
    if (P.mode == PAS_UNIFORM) {
      inst = c[j];
      sl = t;
    } else {
      // q1 = t div b*, q2 = q1 div n_j (exact multiply-high, t < 2^26, n_j <= 64):
      // instance I_j[q1 mod n_j], slot q2 * b* + t mod b*
      const uint32_t b = (uint32_t)P.bstar;
      const uint32_t q1 = P.bstar_shift >= 0 ? ((uint32_t)t >> P.bstar_shift) : (uint32_t)t / b;
      const uint32_t q2 = (uint32_t)(((uint64_t)q1 * plan->n_inst_magic[c[j]]) >> 32);
      inst = plan->inst_list[c[j]][q1 - q2 * (uint32_t)plan->n_inst[c[j]]];
      sl = (int)(q2 * b + ((uint32_t)t - q1 * b));
    }
    instance[p] = inst;
    slot[p] = sl;
  }
  if (tile == 0 && threadIdx.x == 0) {
    // class totals (from the scanned counts) -> per-instance counts (closed form) -> offsets
    int count[kMaxInst];
    for (int i = 0; i < P.W; ++i) count[i] = 0;
    for (int cc = 0; cc < nC; ++cc) {
      const int64_t start = scanned[(int64_t)cc * ntiles];
      const int64_t end = cc + 1 < nC ? scanned[(int64_t)(cc + 1) * ntiles] : P.N;
      const int total = (int)(end - start);
      if (P.mode == PAS_UNIFORM) {
        count[cc] = total;
      } else {
        const int nj = plan->n_inst[cc], b = P.bstar;
        if (nj == 0) continue;
        const int full = total / (b * nj), rem = total % (b * nj);
        for (int m = 0; m < nj; ++m) {
          const int extra = rem - m * b;
          count[plan->inst_list[cc][m]] = full * b + (extra < 0 ? 0 : (extra > b ? b : extra));
        }
      }
    }
    int run = 0;
    for (int i = 0; i <= P.W; ++i) {
      off[i] = run;
      if (user_off) user_off[i] = run;
      if (i < P.W) {
        plan->inst_count[i] = count[i];
        run += count[i];
      }
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
  cudaError_t e = launch_exclusive_scan(w.blk_counts, w.blk_off, nclasses * ntiles, w.scan_tmp, st, launches);
  if (e != cudaSuccess) return e;
  launch_pdl(k_cls_rank, ntiles, THREADS, 0, st, r.cls7, p, ntiles, nclasses, w.blk_off, plan, instance, slot,
             w.offsets, bucket_offsets);
  *launches += 2;
  if (bucket_prompts) {
    launch_pdl(k_bucket, (unsigned)((p.N + 1023) / 1024), 256, 0, st, instance, slot, p.N, w.offsets, bucket_prompts);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace pas
