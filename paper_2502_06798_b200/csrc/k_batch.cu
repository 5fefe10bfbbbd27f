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
// byte per prompt.  Tiles of 4096 prompts:
//   k_cls_count  per-tile class counts, written class-major [C][tiles]: 16 consecutive prompts per
//                thread (one 16-byte load), counted in a private shared-memory column cnt[c][thread]
//                (conflict-free: the column is the bank), rows summed by one warp per class.
//   scan         device-wide exclusive scan of that array: entry (c, b) = prompts of classes < c plus
//                prompts of class c in tiles < b
//   k_cls_rank   t = scan(c, b) - scan(c, 0) + rank inside the tile.  Each warp takes 512 consecutive
//                prompts as 16 rows of 32 (coalesced loads and stores); row by row, match.any gives the
//                lanes of one class, popc of those below a lane is its rank in the row, a per-warp
//                running count per class carries the earlier rows; per block an exclusive prefix over
//                the 8 warps.  Every block turns the class totals into per-instance counts (closed
//                form, greedy: each I_j[m] gets the t's whose (t div b*) mod n_j = m) and batch-list
//                offsets (W <= 64, in shared memory), so the same pass also scatters each prompt id to
//                offsets[instance] + slot (the counting sort's scatter; block 0 publishes the offsets).
// Measured alternatives (64M prompts, profiles/r01_stream): match.any counting is ADU-bound (98 %);
// one ballot per class bit is slower still; the column scheme ranks slower than match.any (262 vs
// 207 us); 16 consecutive prompts per thread with register-packed counters and a shuffle scan
// ranks without votes but scatters the batch lists far worse (463 vs 305 us with the scatter); a
// single-pass decoupled look-back is 60 % slower than count + scan + rank; (round 2) byte-packed class
// counters with 4 prompts per lane and a 5-step warp scan of 4 packed registers per 128 prompts, int4
// stores of instance and slot, executes MORE instructions per prompt (144 vs 97 warp instructions per 32
// prompts: register selects for the packed fields, divergent per-prompt branches) and is slower at 64M
// prompts (407 vs 260 us, profiles/r02_k7/): removed.  Round 2 rework of the rank kernel (profiles/r02_k7b/):
// the per-instance counts in closed form from K5's inst_pos (no W-step loop per instance, no 64-bit
// division), a past-the-end dump class so the rank loop has no range tests and the group leader writes
// its count without a reload, the emit specialised on a full chunk and on the scatter with the scalars
// hoisted, and {instance, list offset} in one 8-byte table entry: 176M -> 102M warp instructions,
// 255 -> 224 us at 64M prompts.  Now latency-bound (issue 40 %, short-scoreboard and barrier stalls),
// not write-bound (a write-only fill reaches 7.1 TB/s here): measured and not kept -- one block barrier
// instead of three (230 us), the batch-list scatter staged through shared memory in (class, t) order
// and written coalesced (231 us; the direct scatter's partial sectors merge in L2: DRAM writes equal
// the algorithmic bytes), 4 or 6 resident CTAs instead of 5 (226 / 265 us), a persistent grid (740 CTAs) that
// builds the per-batch tables once per CTA and stages each warp's next 512 classes with cp.async (299 us).
// HBM per prompt: class 1 B read twice, instance + slot 8 B written, bucket list 4 B written.
#include "dispatch.cuh"

namespace pas {
namespace {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int PER = 16;                        // consecutive prompts per thread (k_cls_count)
constexpr int ROWS = 16;                       // rows of 32 prompts per warp (k_cls_rank)
constexpr int TILE = THREADS * PER;            // prompts per CTA (both kernels: same tiles)
static_assert(PER == ROWS, "k_cls_count and k_cls_rank must cut the same tiles");
constexpr int NCLS = 64;

// This thread's 16 consecutive classes (-1 past the end): one 16-byte load.
__device__ __forceinline__ void load_cls(const uint8_t* __restrict__ src, int64_t p0, int64_t N, int (&v)[PER]) {
  if (p0 + PER <= N) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(src + p0));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < PER; ++e) v[e] = (int)((w[e >> 2] >> (8 * (e & 3))) & 0xFFu);
  } else {
#pragma unroll
    for (int e = 0; e < PER; ++e) v[e] = p0 + e < N ? (int)src[p0 + e] : -1;
  }
}

// Row j of this warp's chunk for k_cls_rank: prompt base + 32 j + lane (NCLS past the end: a dump class
// with its own counter, so the rank loop needs no range test).
__device__ __forceinline__ void load_rows(const uint8_t* __restrict__ src, int64_t base, int64_t N, int (&v)[ROWS]) {
  const int lane = threadIdx.x & 31;
  if (base + 32 * ROWS <= N) {   // the whole chunk in range: one base address, immediate offsets
    const uint8_t* __restrict__ q = src + base + lane;
#pragma unroll
    for (int j = 0; j < ROWS; ++j) v[j] = (int)__ldg(q + 32 * j);
    return;
  }
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const int64_t p = base + 32 * j + lane;
    v[j] = p < N ? (int)__ldg(src + p) : NCLS;
  }
}

// Per-thread class counts in the private column cnt[c * THREADS + tid]; r[e] = rank of element e
// among this thread's earlier elements of its class.
__device__ __forceinline__ void column_counts(int32_t* cnt, int nC, const int (&v)[PER], int (&r)[PER]) {
  const int t = threadIdx.x;
  for (int c = 0; c < nC; ++c) cnt[c * THREADS + t] = 0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    if (v[e] < 0) continue;
    int32_t* a = cnt + v[e] * THREADS + t;
    r[e] = *a;
    *a = r[e] + 1;
  }
}

__global__ void __launch_bounds__(THREADS) k_cls_count(const uint8_t* __restrict__ cls, int64_t N, int ntiles,
                                                       int nC, int32_t* __restrict__ counts /*[nC][ntiles]*/,
                                                       const int* __restrict__ gate) {
  pdl_entry();
  // gate: K6's windowed pass already wrote the counts unless it fell back to the exact path
  if (gate && *reinterpret_cast<const volatile int*>(gate) == 0) return;
  extern __shared__ int32_t cnt[];      // [nC][THREADS]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {   // gated launches use a capped grid
    int v[PER], r[PER];
    load_cls(cls, (int64_t)tile * TILE + (int64_t)threadIdx.x * PER, N, v);
    __syncthreads();   // the previous tile's row sums have read the columns
    column_counts(cnt, nC, v, r);
    __syncthreads();
    for (int c = w; c < nC; c += WARPS) {   // one warp per class: sum its row
      int sum = 0;
#pragma unroll
      for (int i = 0; i < THREADS / 32; ++i) sum += cnt[c * THREADS + lane + 32 * i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) counts[(int64_t)c * ntiles + tile] = sum;
    }
  }
}

#ifndef PAS_K7_MINB
#define PAS_K7_MINB 5     // resident CTAs per SM the rank kernel is compiled for: 48 registers (a few once-per-warp spills)
#endif

// The stateless per-row emit of k_cls_rank: t = wb[class] + in-warp rank; greedy (MODE 0/1): q1 = t div b*,
// q2 = q1 div n_j (exact multiply-high, t < 2^26, n_j <= 64), instance I_j[q1 mod n_j], slot
// q2 * b* + t mod b*; uniform (MODE 2): instance = class, slot = t.  SCATTER: also write the batch lists;
// FULL: all 16 rows of the warp's chunk are in range (no per-row end test).
template <int MODE, bool SCATTER, bool FULL>
__device__ __forceinline__ void emit_rows(const int (&c)[ROWS], const int32_t* __restrict__ wb, const uint4* cinfo_s,
                                          const int2* flat_s, const int32_t* ioff,
                                          int32_t* __restrict__ inst_w, int32_t* __restrict__ slot_w,
                                          int32_t* __restrict__ prompts, int32_t p_w, uint32_t b, uint32_t sh, int W) {
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const int cj = c[j] & 0xFF, rj = c[j] >> 8;
    if (!FULL && cj == NCLS) continue;
    const int t = wb[cj] + rj;
    int inst, sl, off;
    if (MODE == 2) {
      inst = cj;
      sl = t;
      off = ioff[cj];
    } else {
      const uint32_t q1 = MODE == 0 ? ((uint32_t)t >> sh) : (uint32_t)t / b;
      const uint4 ci = cinfo_s[cj];
      const uint32_t q2 = ci.x ? __umulhi(q1, ci.x) : q1;
      const int2 e = flat_s[ci.z + (q1 - q2 * ci.y)];   // I_j[q1 mod n_j] and its list offset
      inst = e.x;
      off = e.y;
      sl = (int)(q2 * b + ((uint32_t)t - q1 * b));
    }
    PAS_CHECK(inst >= 0 && inst < W && sl >= 0 && off == ioff[inst] && off + sl < ioff[inst + 1], "K7 batch-list position");
    inst_w[32 * j] = inst;
    slot_w[32 * j] = sl;
    if (SCATTER) prompts[off + sl] = p_w + 32 * j;   // the batch lists (counting-sort scatter)
  }
}

// DISP: the f3 stateful dispatcher picks (a separate instantiation keeps R13 lean).  MODE (the stateless
// path; compile-time so the per-row loop carries no mode branches or parameter reloads): 0 greedy with
// b* a power of two, 1 greedy with any b*, 2 uniform.  The DISP instantiation reads P.mode.
template <bool DISP, int MODE>
__global__ void __launch_bounds__(THREADS, DISP ? 1 : PAS_K7_MINB) k_cls_rank(const uint8_t* __restrict__ cls, const __grid_constant__ RouteParams P,
                                                      int ntiles, int nC, const int32_t* __restrict__ scanned,
                                                      DevPlan* __restrict__ plan, int32_t* __restrict__ instance,
                                                      int32_t* __restrict__ slot, int32_t* __restrict__ prompts,
                                                      int32_t* __restrict__ user_off) {
  pdl_entry();
  advance_batch_counters(P);   // the batch's last kernel: every reader of the counters has finished
  __shared__ int32_t wcnt[WARPS][NCLS + 1];   // per-warp class counts of this tile (+ the past-the-end dump)
  __shared__ int32_t wbase[WARPS][NCLS];   // per warp and class: t of the warp's first prompt of the class
  __shared__ int32_t tile_off[NCLS];
  __shared__ int32_t icount[kMaxInst], fpos[kMaxInst], ioff[kMaxInst + 1];   // per instance: count, flat_s slot, list offset
  // per K' level j: {32-bit reciprocal of n_j (0 for n_j = 1), n_j, first entry of I_j in flat_s, -}
  __shared__ uint4 cinfo_s[kMaxLevels];
  // {instance, batch-list offset} of I_0[0..n_0), I_1[0..n_1), ...: W <= 64 entries (each instance sits
  // at exactly one level), so the per-prompt instance pick and its list offset are one 8-byte load
  __shared__ int2 flat_s[kMaxInst];
  __shared__ __align__(16) int32_t ilist_s[DISP ? kMaxLevels : 1][kMaxInst];   // f3 only: I_j per level
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * TILE + w * 32 * ROWS;
  const bool uniform = DISP ? P.mode == PAS_UNIFORM : MODE == 2;
  int c[ROWS];
  load_rows(cls, base, P.N, c);
  for (int i = threadIdx.x; i < WARPS * (NCLS + 1); i += THREADS) (&wcnt[0][0])[i] = 0;
  if (!uniform) {
    // K5 wrote n_j's reciprocal (q div n_j = umulhi(q, ceil(2^32 / n_j)), exact for q < 2^26 and
    // n_j <= 64) and I_j's start in the level-ordered instance list
    if (threadIdx.x < nC)
      cinfo_s[threadIdx.x] = make_uint4(plan->n_inst_recip[threadIdx.x], (uint32_t)plan->n_inst[threadIdx.x],
                                        (uint32_t)plan->inst_base[threadIdx.x], 0u);
    if (DISP) {   // the instance lists of the K' levels (the f3 picks walk them)
#pragma unroll 1
      for (int i = threadIdx.x; i < nC * (kMaxInst / 4); i += THREADS)   // 16-byte copies
        reinterpret_cast<int4*>(&ilist_s[0][0])[i] = reinterpret_cast<const int4*>(&plan->inst_list[0][0])[i];
    }
  }
  if (threadIdx.x < nC) {
    const int64_t row = (int64_t)threadIdx.x * ntiles;
    tile_off[threadIdx.x] = scanned[row + tile] - scanned[row];
  }
  if (threadIdx.x < P.W) {
    // class totals (from the scanned counts) -> this instance's count (closed form, R13 / R14): instance
    // i is I_j[m] (m = its position among the n_j instances of its level j, from K5)
    const int i = threadIdx.x;
    const int cc = uniform ? i : P.inst_level[i];
    const int64_t start = scanned[(int64_t)cc * ntiles];
    const int64_t end = cc + 1 < nC ? scanned[(int64_t)(cc + 1) * ntiles] : P.N;
    const int total = (int)(end - start);
    int cnt = total;
    if (DISP) {
      cnt = P.dplan->cnt[i];   // f3: counted by k_disp_prep from the same class totals
    } else if (!uniform) {
      const int m = plan->inst_pos[i], nj = plan->n_inst[cc];
      const int b = P.bstar, full = total / (b * nj), rem = total - full * (b * nj), extra = rem - m * b;
      cnt = full * b + (extra < 0 ? 0 : (extra > b ? b : extra));
      fpos[i] = plan->inst_base[cc] + m;
    }
    icount[i] = cnt;
  }
  // in-warp rank, row by row: match.any groups the lanes of one class; a per-warp running count per
  // class (advanced by the group's lowest lane, whose rank is the count itself) carries the earlier
  // rows.  The rank is packed above the class byte (c[j] = rank << 8 | class): one register per row.
  __syncthreads();   // wcnt zeroed
  const unsigned lt = (1u << lane) - 1;
#pragma unroll
  for (int j = 0; j < ROWS; ++j) {
    const unsigned m = __match_any_sync(0xffffffffu, c[j]);
    const unsigned below = m & lt;
    const int r = wcnt[w][c[j]] + __popc(below);
    __syncwarp();
    if (below == 0) wcnt[w][c[j]] = r + __popc(m);
    __syncwarp();
    c[j] = (r << 8) | c[j];
  }
  __syncthreads();
  if (w == 0) {   // batch-list offsets: exclusive scan of the W <= 64 instance counts, two per lane
    static_assert(kMaxInst <= 64, "two instances per lane");
    const int i0 = 2 * lane, i1 = 2 * lane + 1;
    const int a = i0 < P.W ? icount[i0] : 0, b = i1 < P.W ? icount[i1] : 0;
    int incl = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const int ex = incl - a - b;
    if (i0 < P.W) ioff[i0] = ex;
    if (i1 < P.W) ioff[i1] = ex + a;
    if (lane == 31) ioff[P.W] = incl;   // the total
    if (!uniform) {
      if (i0 < P.W) flat_s[fpos[i0]] = make_int2(i0, ex);
      if (i1 < P.W) flat_s[fpos[i1]] = make_int2(i1, ex + a);
    }
    if (tile == 0) {
      if (user_off) {
        if (i0 < P.W) user_off[i0] = ex;
        if (i1 < P.W) user_off[i1] = ex + a;
        if (lane == 31) user_off[P.W] = incl;
      }
      if (i0 < P.W) plan->inst_count[i0] = a;
      if (i1 < P.W) plan->inst_count[i1] = b;
    }
  }
  if (threadIdx.x < nC) {   // per class: the tile's offset plus the exclusive prefix over the warps
    int x[WARPS];
#pragma unroll
    for (int v = 0; v < WARPS; ++v) x[v] = wcnt[v][threadIdx.x];   // independent loads, then a short add chain
    int run = tile_off[threadIdx.x];
#pragma unroll
    for (int v = 0; v < WARPS; ++v) {
      wbase[v][threadIdx.x] = run;
      run += x[v];
    }
  }
  __syncthreads();
  // per-warp output bases: the unrolled rows below address them with immediate offsets
  int32_t* const inst_w = instance + base + lane;
  int32_t* const slot_w = slot + base + lane;
  const int32_t p_w = (int32_t)(base + lane);   // prompt ids fit int32 (N <= max_batch < 2^31)
  if constexpr (!DISP) {   // stateless: the per-row emit specialised on the batch-list scatter and a full chunk
    const bool full = base + 32 * ROWS <= P.N;
    const uint32_t bs = (uint32_t)P.bstar, sh = (uint32_t)P.bstar_shift;
    if (prompts) {
      if (full) emit_rows<MODE, true, true>(c, wbase[w], cinfo_s, flat_s, ioff, inst_w, slot_w, prompts, p_w, bs, sh, P.W);
      else emit_rows<MODE, true, false>(c, wbase[w], cinfo_s, flat_s, ioff, inst_w, slot_w, prompts, p_w, bs, sh, P.W);
    } else {
      if (full) emit_rows<MODE, false, true>(c, wbase[w], cinfo_s, flat_s, ioff, inst_w, slot_w, prompts, p_w, bs, sh, P.W);
      else emit_rows<MODE, false, false>(c, wbase[w], cinfo_s, flat_s, ioff, inst_w, slot_w, prompts, p_w, bs, sh, P.W);
    }
  } else {
#pragma unroll
    for (int j = 0; j < ROWS; ++j) {   // f3 stateful dispatcher: slot = position in the instance's queue (R29, R31)
      const int cj = c[j] & 0xFF, rj = c[j] >> 8;
      if (cj == NCLS) continue;
      const int t = wbase[w][cj] + rj;
      int inst;
      int64_t sl64;
      if (uniform) {
        inst = cj;
        sl64 = P.dplan->Q0[inst] + t;
      } else {
        disp_pick_greedy(P.dplan, ilist_s[cj], (int)cinfo_s[cj].y, cj, t, P.bstar, inst, sl64);
      }
      const int sl = (int)sl64, pos = (int)(sl64 - P.dplan->Q0[inst]);
      PAS_CHECK(inst >= 0 && inst < P.W && pos >= 0 && ioff[inst] + pos < ioff[inst + 1], "K7 batch-list position");
      inst_w[32 * j] = inst;
      slot_w[32 * j] = sl;
      if (prompts) prompts[ioff[inst] + pos] = p_w + 32 * j;   // the batch lists (counting-sort scatter)
    }
  }
}

}  // namespace

int batch_tiles(int64_t N) { return (int)((N + TILE - 1) / TILE); }

// Up to 64 classes x 256 threads of int32 columns (64 KB) needs the > 48 KB opt-in.
cudaError_t batch_init() {
  const int bytes = NCLS * THREADS * (int)sizeof(int32_t);
  cudaError_t e = cudaFuncSetAttribute(k_cls_count, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  return e;
}

cudaError_t launch_route_and_batch(const RedirectWs& r, const RouteParams& p, DevPlan* plan, const int* count_gate,
                                   const BatchWs& w,
                                   int32_t* instance, int32_t* slot, int32_t* bucket_offsets,
                                   int32_t* bucket_prompts, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  const int ntiles = batch_tiles(p.N);
  const int nclasses = p.mode == PAS_UNIFORM ? p.W : p.nK;
  const size_t smem = (size_t)nclasses * THREADS * sizeof(int32_t);
  const int cgrid = count_gate && ntiles > kNumSMs * 4 ? kNumSMs * 4 : ntiles;   // gated: capped, grid-stride
  launch_pdl(k_cls_count, cgrid, THREADS, smem, st, r.cls7, p.N, ntiles, nclasses, w.blk_counts, count_gate);
  cudaError_t e = launch_exclusive_scan(w.blk_counts, w.blk_off, nclasses * ntiles, w.scan_tmp, st, launches);
  if (e != cudaSuccess) return e;
  if (p.disp) {   // f3: queue events since the last batch, pick tables, counts, state after
    e = launch_disp_prep(p, ntiles, nclasses, w.blk_off, st);
    if (e != cudaSuccess) return e;
    *launches += 1;
  }
  auto kern = p.disp ? k_cls_rank<true, 0>
              : p.mode == PAS_UNIFORM ? k_cls_rank<false, 2>
              : p.bstar_shift >= 0 ? k_cls_rank<false, 0> : k_cls_rank<false, 1>;
  launch_pdl(kern, ntiles, THREADS, 0, st, r.cls7, p, ntiles, nclasses, w.blk_off, plan, instance, slot, bucket_prompts,
             bucket_offsets);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace pas
