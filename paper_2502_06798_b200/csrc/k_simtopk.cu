// K2 -- prompt x cache cosine-similarity GEMM on tcgen05 tensor cores with a fused running top-k.
//
// Paper: the Optimal-K Selector "first retrieves the nearest cache" by prompt
// "closeness".  Both operands are unit rows in bf16 (K1), so S = Q_hat C_hat^T is the cosine
// similarity; it is accumulated in fp32 in TMEM and never written to memory: each epilogue thread
// owns one prompt row of the accumulator and keeps the k best (score desc, gid asc; R10) over the
// cache range of its work unit.
//
// Two tile organisations share one source (template parameter), dispatched by batch size
// (simtopk_pair; DESIGN.md section 8 records the A/B on one B200):
//   single CTA (else)     tcgen05.mma.cta_group::1, 128 prompt rows x 256 cache rows x K=16 per
//                         instruction; per stage A 128x64 + B 256x64 bf16 (48 KB), 4 stages.
//   CTA pair (N = 129..256, 385..512)   tcgen05.mma.cta_group::2, 256 x 256 x 16: prompt rows 0..127 in CTA 0,
//                         128..255 in CTA 1; the 256 cache rows of B split 128/128 between the two
//                         CTAs' smem (32 KB / stage, 6 stages); TMA bytes of both CTAs land on the
//                         leader's mbarrier; commits multicast to both CTAs.
//
// Two schedules:
//   dynamic (single-CTA tile, long ranges; simtopk_plan_dynamic): units (chunk step, range, prompt
//     tile) of T cache tiles handed out by a global counter, the top-k lists parked in L2 between a
//     (range, prompt tile)'s chunks -- the CTAs stay within one chunk step of each other whatever
//     their speed, so the cache crosses HBM about once and fast SMs take more units.
//   static (CTA pair, short ranges): unit = (prompt tile m, cache range r); persistent CTAs / pairs
//     walk units u = id + i*count with m fastest, so concurrently running CTAs stream the SAME cache
//     tiles against different prompt tiles.  Progress leash (small N only, simtopk_leash_slack): free
//     running, CTAs drift apart over a range of thousands of tiles by more than L2 holds and tiles are
//     fetched from DRAM again and again, so each producer publishes its tile count (epoch-tagged) and
//     waits while it is more than `slack` tiles ahead of the slowest CTA still working.
//
// Warp roles per CTA (320 threads, 1 CTA/SM):
//   warp 0      TMA producer (128-B swizzle, mbarrier complete_tx); in the dynamic schedule it also
//               takes the units and publishes them through a 4-entry mbarrier ring.
//   warp 1      TMEM allocation (512 columns = two 256-column fp32 accumulators) and one lane issuing
//               tcgen05.mma + tcgen05.commit (smem stage released, accumulator ready).
//   warps 2..9  epilogue over the CTA's 128 TMEM lanes, two warps per lane quarter (column halves
//               0..127 / 128..255 of every tile, each with its own top-k list, merged by a bitonic
//               network at the end of the range): tcgen05.ld of 32 columns, max of the chunk vs the
//               current k-th score, and while it beats it, insert the max and knock it out (epi_tile).
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "pas_internal.cuh"
#include "ptx_sm100.cuh"

// Shape-dispatched tile: the CTA pair (cta_group::2) for N <= PAS_K2_PAIR_MAX_TILES x 128 prompts in an
// even number of 128-row tiles,
// the single-CTA tile above that (A/B in DESIGN.md 8: the pair is faster where K2 is latency- and
// L2-bound, the single CTA where it is power-bound).  0 disables the pair; a huge value forces it.
#ifndef PAS_K2_PAIR_MAX_TILES
#define PAS_K2_PAIR_MAX_TILES 4
#endif


namespace pas {
namespace {

constexpr int BM = 128;                 // prompt rows per CTA
constexpr int BN = 256;                 // cache rows per tile (MMA N)
constexpr int BK = 64;                  // one 128-B swizzle row of bf16
constexpr int EPI_WARPS = 8;                     // 2 per TMEM lane quarter: column halves
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;
constexpr int LIST_BYTES = BM * 16 * 8;             // hand-over of the upper half's lists (KMAX <= 16)
constexpr int WARMUP_TILES = 24;

// BNT: cache rows per tile (MMA N): 256, or 128 for the small-problem tile (simtopk_small)
template <bool P, int BNT = BN>
struct Tile {
  static constexpr int CTAS = P ? 2 : 1;
  static constexpr int BN_CTA = BNT / CTAS;          // cache rows staged per CTA
  static constexpr int STAGES = (P || BNT < BN) ? 6 : 4;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN_CTA * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // per CTA
  static constexpr int NUM_WORKERS = kNumSMs / CTAS;      // persistent CTAs (or pairs)
  static constexpr int UNIT_ROWS = BM * CTAS;             // prompt rows per work unit
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + LIST_BYTES;
};

constexpr int UNIT_RING = 4;   // dynamic schedule: work units fetched ahead by the producer

template <int STAGES>
struct __align__(8) Bars {
  uint64_t full[STAGES];    // TMA bytes landed (leader's barrier in pair mode)
  uint64_t empty[STAGES];   // MMA finished reading the stage
  uint64_t tfull[2];        // accumulator ready
  uint64_t tempty[2];       // epilogue(s) drained the accumulator
  uint64_t ufull[UNIT_RING];    // dynamic schedule: unit id published by the producer
  uint64_t uempty[UNIT_RING];   // ... read by the MMA issuer and every epilogue warp
  int32_t unit[UNIT_RING];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars<6>) <= 256, "barrier block overflows its 256-byte slot");

// Opaque copy: stops the compiler from strength-reducing per-element column ids across chunks.
__device__ __forceinline__ int opaque(int x) {
  asm volatile("" : "+r"(x));
  return x;
}

__device__ __forceinline__ float max32(const uint32_t (&v)[32]) {
  float mx = __uint_as_float(v[0]);
#pragma unroll
  for (int j = 1; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
  return mx;
}

template <int KMAX>
__device__ __forceinline__ void bubble_insert(float x, int32_t g, float (&s)[KMAX], int32_t (&gl)[KMAX]) {
  s[KMAX - 1] = x;
  gl[KMAX - 1] = g;
#pragma unroll
  for (int i = KMAX - 1; i > 0; --i) {
    if (s[i] > s[i - 1]) {
      const float ts = s[i]; s[i] = s[i - 1]; s[i - 1] = ts;
      const int32_t tg = gl[i]; gl[i] = gl[i - 1]; gl[i - 1] = tg;
    }
  }
}

// Epilogue over one accumulator: 32-column chunks (tcgen05.ld), chain max (FMNMX3), the column id
// materialised only inside the insert path, the tail mask only on the last partial tile.
// Insert path: while the chunk max beats the k-th best, insert it and knock it out (lowest column among
// equal values), so a lane pays per candidate, not per column; a warp pays the most candidates of any
// lane.  Inserting in value order (ties: column ascending) with a strict > keeps the list the top-k
// under (score desc, column asc), exactly as a column-order scan would.  Measured and removed
// (DESIGN.md 8): the column-order scan of all 32 columns (a warp pays 32 bubble inserts whenever any
// lane has a candidate), a warp vote per column on top of it, a double-buffered tcgen05.ld + tree max.
template <int KMAX, bool PARTIAL, int NCH = BN / 64>
__device__ __forceinline__ void epi_tile(uint32_t taddr, int col_base, int M_local, float (&s)[KMAX],
                                            int32_t (&gl)[KMAX]) {
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {   // this warp's share of the tile: NCH chunks of 32 columns
    uint32_t v[32];
    ptx::tmem_ld_32x32b_x32(taddr + c * 32, v);
    ptx::tmem_wait_ld();
    const int base = opaque(col_base + c * 32);
    if (PARTIAL) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (base + j >= M_local) v[j] = __float_as_uint(-INFINITY);
    }
    float mx = max32(v);
    while (mx > s[KMAX - 1]) {
      int col = 0;
      bool hit = false;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool h = !hit && __uint_as_float(v[j]) == mx;
        col = h ? j : col;
        v[j] = h ? __float_as_uint(-INFINITY) : v[j];
        hit = hit || h;
      }
      bubble_insert<KMAX>(mx, base + col, s, gl);
      mx = max32(v);
    }
  }
}

// Top-KMAX of two sorted lists (score desc, column asc): bitonic half-cleaner against the reversed
// partner list, then a bitonic sort of the KMAX winners -- static indexing only.
__device__ __forceinline__ bool better(float sa, int ga, float sb, int gb) {
  return sa > sb || (sa == sb && (unsigned)ga < (unsigned)gb);
}
template <int KMAX>
__device__ __forceinline__ void merge_lists(float (&s)[KMAX], int32_t (&gl)[KMAX], const float* ps, const int32_t* pg) {
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    const float bs = ps[KMAX - 1 - i];
    const int32_t bg = pg[KMAX - 1 - i];
    if (!better(s[i], gl[i], bs, bg)) { s[i] = bs; gl[i] = bg; }
  }
#pragma unroll
  for (int len = KMAX / 2; len >= 1; len >>= 1) {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      if ((i & len) == 0) {
        const int j = i + len;
        if (!better(s[i], gl[i], s[j], gl[j])) {
          const float ts = s[i]; s[i] = s[j]; s[j] = ts;
          const int32_t tg = gl[i]; gl[i] = gl[j]; gl[j] = tg;
        }
      }
    }
  }
}

// Whole producer warp: publish `issued` and wait until issued - min(progress of live CTAs) <= slack.
// Bounded (a CTA that never gets a slot cannot deadlock the grid: the leash just lets go).
__device__ __noinline__ void leash_wait(uint64_t* progress, int worker, int nworkers, uint32_t epoch,
                                        uint32_t issued, uint32_t slack) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane == 0)
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(progress + worker),
                 "l"(((uint64_t)epoch << 32) | issued) : "memory");
  if (issued <= slack) return;
  for (int spin = 0; spin < (1 << 16); ++spin) {
    uint32_t mn = 0xFFFFFFFFu;
    for (int w = (int)lane; w < nworkers; w += 32) {
      uint64_t v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(progress + w) : "memory");
      mn = min(mn, (uint32_t)(v >> 32) == epoch ? (uint32_t)v : 0u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (issued - min(mn, issued) <= slack) return;
    __nanosleep(512);
  }
}

// Dynamic schedule (DESIGN.md 8 "K2 schedule"): prompt tiles in groups of MTg; within a group, unit
// u = (chunk step c, range r, prompt tile m), m fastest, then r, then c; chunk c of range r = its tiles
// [t0 + cT, t0 + (c+1)T) (possibly empty).  j = r * MT + m is the (range, prompt tile) slot.
__device__ __forceinline__ void dyn_decode(int u, int MT, int R, int NT, const DynSched& dy, int& c, int& j,
                                           int& ta, int& tb) {
  const int per_group = dy.CS * R * dy.MTg;
  const int g = u / per_group;
  const int ui = u - g * per_group;
  const int m0 = g * dy.MTg;
  const int mg = min(dy.MTg, MT - m0);
  const int P = mg * R;
  c = ui / P;
  const int ji = ui - c * P;
  const int r = ji / mg;
  j = r * MT + m0 + (ji - r * mg);
  const int t0 = (int)((int64_t)r * NT / R), t1 = (int)((int64_t)(r + 1) * NT / R);
  ta = min(t1, t0 + c * dy.T);
  tb = min(t1, ta + dy.T);
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until the lists of (r, m) after chunk c - 1 are published.  Bounded: a broken protocol traps
// (a reported launch failure) instead of hanging the device.
__device__ __noinline__ void dyn_wait_state(const uint64_t* done, uint64_t want) {
  for (uint32_t spin = 0;; ++spin) {
    if (ld_acquire_u64(done) == want) return;
    if (spin > (1u << 26)) __trap();
    __nanosleep(256);
  }
}

__device__ __forceinline__ void epi_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
}

template <int KMAX, bool DUMP, bool PAIR, bool DYN, int BNT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_simtopk(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmC, int64_t N,
              int64_t M_local, int kblocks, int k, int G, int rank, int R, int MT, int NT, Cand* __restrict__ out,
              float* __restrict__ dump, uint64_t* __restrict__ progress, uint32_t epoch_arg,
              const uint32_t* __restrict__ epoch_dev, uint32_t slack, const DynSched dyn, int dup_arg) {
  static_assert(!DYN || (!PAIR && !DUMP), "the dynamic schedule serves the single-CTA top-k tile");
  static_assert(BNT == BN || (!PAIR && !DYN && !DUMP), "the small tile serves the static single-CTA path");
  using TL = Tile<PAIR, BNT>;
  constexpr int CTAS = TL::CTAS, BN_CTA = TL::BN_CTA, STAGES = TL::STAGES, A_BYTES = TL::A_BYTES,
                B_BYTES = TL::B_BYTES, STAGE_BYTES = TL::STAGE_BYTES, UNIT_ROWS = TL::UNIT_ROWS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  Bars<STAGES>* bars = reinterpret_cast<Bars<STAGES>*>(smem + STAGES * STAGE_BYTES);
  float* list_s = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);   // [BM][KMAX]
  int32_t* list_g = reinterpret_cast<int32_t*>(list_s + BM * KMAX);            // [BM][KMAX]

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t crank = PAIR ? ptx::cluster_ctarank() : 0;
  const bool leader = crank == 0;
  const int worker = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nworkers = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int MTu = MT;   // schedule rows: prompt tiles
  const int units = DYN ? dyn.CS * MTu * R : MT * R;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmQ);
    ptx::prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&bars->full[s], 1);
      ptx::mbar_init(&bars->empty[s], 1);
    }
    for (int s = 0; s < UNIT_RING; ++s) {
      ptx::mbar_init(&bars->ufull[s], 1);
      ptx::mbar_init(&bars->uempty[s], 1 + EPI_WARPS);   // released by the MMA issuer + every epilogue warp
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&bars->tfull[a], 1);
      ptx::mbar_init(&bars->tempty[a], EPI_WARPS * CTAS);  // one arrive per epilogue warp (of both CTAs)
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) {
      ptx::tmem_alloc_pair(&bars->tmem_base, TMEM_COLS);
      ptx::tmem_relinquish_pair();
    } else {
      ptx::tmem_alloc(&bars->tmem_base, TMEM_COLS);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  if (PAIR) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = bars->tmem_base;
  pdl_entry();   // prologue (barriers, TMEM, tensor-map prefetch) overlapped with the previous kernel
  // this launch's epoch: bumped on the device by the K1 that precedes it (graph-replayable), else the
  // host's argument
  const uint32_t epoch = epoch_dev ? *reinterpret_cast<const volatile uint32_t*>(epoch_dev) : epoch_arg;

  if (warp == 0) {
    // ------------------------------- TMA producer -------------------------------
    // Lane 0 waits on the ring and issues TMA; with the leash on, the whole warp walks the schedule
    // (the look-up of the other CTAs' progress is warp-parallel).
    if (DYN) {
      // dynamic schedule: lane 0 takes the next unit from the global counter, publishes it to the
      // MMA issuer and the epilogue through the unit ring, then streams its chunk
      if (lane == 0) {
        int stage = 0, us = 0;
        uint32_t phase = 0, uph = 0;
        for (;;) {
          int u = (int)atomicAdd(dyn.sched, 1u);
          if (u >= units) u = -1;
          ptx::mbar_wait(&bars->uempty[us], uph ^ 1);
          bars->unit[us] = u;
          ptx::mbar_arrive(&bars->ufull[us]);
          if (++us == UNIT_RING) { us = 0; uph ^= 1; }
          if (u < 0) break;
          int c, j, ta, tb;
          dyn_decode(u, MTu, R, NT, dyn, c, j, ta, tb);
          const int qrow = (j % MT) * BM;
          for (int t = ta; t < tb; ++t) {
            for (int kb = 0; kb < kblocks; ++kb) {
              ptx::mbar_wait(&bars->empty[stage], phase ^ 1);
              ptx::mbar_arrive_expect_tx(&bars->full[stage], STAGE_BYTES);
              ptx::tma_load_2d(&tmQ, sA + stage * A_BYTES, &bars->full[stage], kb * BK, qrow, ptx::kEvictLast);
              ptx::tma_load_2d(&tmC, sB + stage * B_BYTES, &bars->full[stage], kb * BK, t * BNT,
                               ptx::kEvictNormal);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
        // every worker has taken its last unit once all have arrived here: the last one out re-arms
        // the counter for the next launch (kernel boundaries order this against the next K2)
        if (atomicAdd(dyn.sched + 1, 1u) == (uint32_t)nworkers - 1) {
          dyn.sched[0] = 0;
          dyn.sched[1] = 0;
        }
      }
    } else if (slack || lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t issued = 0;
      for (int u = worker; u < units; u += nworkers) {
        const int m = u % MT, r = u / MT;
        const int t0 = (int)((int64_t)r * NT / R), t1 = (int)((int64_t)(r + 1) * NT / R);
        const int qrow = m * UNIT_ROWS + (int)crank * BM;
        for (int t = t0; t < t1; ++t, ++issued) {
          if (slack) {
            if (leader) leash_wait(progress, worker, nworkers, epoch, issued, slack);
            __syncwarp();
          }
          const int crow = t * BNT + (int)crank * BN_CTA;
          if (lane == 0)
          for (int kb = 0; kb < kblocks; ++kb) {
            ptx::mbar_wait(&bars->empty[stage], phase ^ 1);
            if (PAIR) {
              if (leader) ptx::mbar_arrive_expect_tx(&bars->full[stage], CTAS * STAGE_BYTES);
              ptx::tma_load_2d_pair(&tmQ, sA + stage * A_BYTES, &bars->full[stage], kb * BK, qrow, ptx::kEvictLast);
              ptx::tma_load_2d_pair(&tmC, sB + stage * B_BYTES, &bars->full[stage], kb * BK, crow,
                                    ptx::kEvictNormal);
            } else {
              ptx::mbar_arrive_expect_tx(&bars->full[stage], STAGE_BYTES);
              ptx::tma_load_2d(&tmQ, sA + stage * A_BYTES, &bars->full[stage], kb * BK, qrow, ptx::kEvictLast);
              ptx::tma_load_2d(&tmC, sB + stage * B_BYTES, &bars->full[stage], kb * BK, crow, ptx::kEvictNormal);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (slack) __syncwarp();
        }
      }
      if (slack && leader && lane == 0)   // done: never hold anyone back
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(progress + worker),
                     "l"(((uint64_t)epoch << 32) | 0xFFFFFFFFull) : "memory");
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer ---------------------------------
    // (CTA pair: the leader issues for both CTAs; the single-CTA tile its own)
    if ((!PAIR || leader) && ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(UNIT_ROWS, BNT);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int us = 0;
      uint32_t uph = 0;
      for (int u = worker; DYN || u < units; u += nworkers) {
        int t0, t1;
        if (DYN) {
          ptx::mbar_wait(&bars->ufull[us], uph);
          u = bars->unit[us];
          ptx::mbar_arrive(&bars->uempty[us]);
          if (++us == UNIT_RING) { us = 0; uph ^= 1; }
          if (u < 0) break;
          int c, j;
          dyn_decode(u, MTu, R, NT, dyn, c, j, t0, t1);
        } else {
          const int r = u / MT;
          t0 = (int)((int64_t)r * NT / R);
          t1 = (int)((int64_t)(r + 1) * NT / R);
        }
        for (int t = t0; t < t1; ++t) {
          ptx::mbar_wait(&bars->tempty[acc], acc_phase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BNT;
          for (int kb = 0; kb < kblocks; ++kb) {
            ptx::mbar_wait(&bars->full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(sA + stage * A_BYTES);
            const uint32_t b0 = ptx::smem_u32(sB + stage * B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = ptx::sdesc_kmajor_sw128(a0 + kk * 32);
              const uint64_t bd = ptx::sdesc_kmajor_sw128(b0 + kk * 32);
              if (PAIR) ptx::umma_f16_ss_pair(d_tmem, ad, bd, idesc, (kb | kk) != 0);
              else ptx::umma_f16_ss(d_tmem, ad, bd, idesc, (kb | kk) != 0);
            }
            if (PAIR) ptx::umma_commit_pair(&bars->empty[stage], 0x3);
            else ptx::umma_commit(&bars->empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (PAIR) ptx::umma_commit_pair(&bars->tfull[acc], 0x3);
          else ptx::umma_commit(&bars->tfull[acc]);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------- epilogue -----------------------------------
    const uint32_t q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = (int)(warp - 2) >> 2;    // 0: columns 0..127 of each tile, 1: 128..255
    const int row = (int)(q * 32 + lane);
    // Small batches (dup, N <= 64): K1 wrote every prompt row again 64 rows down, so the MMA computes
    // each prompt's scores in lane quarters q and q + 2 -- which belong to different SM
    // sub-partitions.  The four (quarter pair, half) combinations then take a quarter of the columns
    // each: the epilogue runs on all four schedulers instead of the two the real rows would occupy.
    const bool dup = !PAIR && !DYN && !DUMP && dup_arg;
    const int cpart = dup ? (int)(q >> 1) * 2 + half : half;   // column part of the tile this warp ranks
    const int PCOLS = dup ? BNT / 4 : BNT / 2;
    const int prow = dup ? (row & 63) : row;                   // the prompt row this lane ranks
    const uint32_t lane_addr = tmem_base + ((q * 32u) << 16) + cpart * PCOLS;
    const int Ml = (int)M_local;
    int acc = 0;
    uint32_t acc_phase = 0;
    int us = 0;
    uint32_t uph = 0;
    for (int u = worker; DYN || u < units; u += nworkers) {
      int m, r, t0, t1, c = 0, j = 0;
      if (DYN) {
        ptx::mbar_wait(&bars->ufull[us], uph);
        u = bars->unit[us];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bars->uempty[us]);
        if (++us == UNIT_RING) { us = 0; uph ^= 1; }
        if (u < 0) break;
        dyn_decode(u, MTu, R, NT, dyn, c, j, t0, t1);
        PAS_CHECK(u < units && c < dyn.CS && t0 <= t1 && t1 <= NT, "K2 unit decode");
        m = j % MT;
        r = j / MT;
      } else {
        m = u % MT;
        r = u / MT;
        t0 = (int)((int64_t)r * NT / R);
        t1 = (int)((int64_t)(r + 1) * NT / R);
      }
      const int64_t prompt = (int64_t)m * UNIT_ROWS + (PAIR ? crank * BM : 0) + prow;
      // a warp whose 32 rows are all past the batch (the padding of the last prompt tile) has no lists
      // to keep: it skips the epilogue work (those Q_hat rows are whatever the buffer holds, and a
      // list fed garbage scores inserts on most chunks -- C1: 5.5 us of K2's 18.5)
      const bool warp_live = __any_sync(0xffffffffu, prompt < N);
      float s[KMAX];
      int32_t gl[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) { s[i] = -INFINITY; gl[i] = -1; }
      // dynamic schedule: resume the lists this (range, prompt tile) had after chunk c - 1
      const int64_t st_off = ((int64_t)(j * 2 + half) * KMAX) * BM + row;
      PAS_CHECK(!DYN || j < dyn.slots, "K2 parked-list slot");
      PAS_CHECK(r < R && m < MT, "K2 range / prompt tile");
      if (DYN && c > 0) {
        if (warp == 2 && lane == 0) dyn_wait_state(dyn.done + j, ((uint64_t)epoch << 32) | (uint32_t)c);
        epi_barrier();
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          s[i] = __ldcg(dyn.st_s + st_off + i * BM);
          gl[i] = __ldcg(dyn.st_g + st_off + i * BM);
        }
      }
      for (int t = t0; t < t1; ++t) {
        ptx::mbar_wait(&bars->tfull[acc], acc_phase);
        ptx::tc_fence_after();
        const int col_base = t * BNT + cpart * PCOLS;
        const uint32_t taddr = lane_addr + acc * BNT;
        if (!warp_live) {
          // nothing to rank (the accumulator is released below like any other)
        } else if (DUMP) {
#pragma unroll 1
          for (int c = 0; c < BNT / 64; ++c) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(taddr + c * 32, v);
            ptx::tmem_wait_ld();

            const int64_t col0 = (int64_t)col_base + c * 32;
            if (prompt < N)
              for (int j = 0; j < 32; ++j)
                if (col0 + j < M_local) dump[prompt * M_local + col0 + j] = __uint_as_float(v[j]);
          }
        } else if (dup) {
          if (col_base + BNT / 4 > Ml) epi_tile<KMAX, true, BNT / 128>(taddr, col_base, Ml, s, gl);
          else epi_tile<KMAX, false, BNT / 128>(taddr, col_base, Ml, s, gl);
        } else if (col_base + BNT / 2 > Ml) {
          epi_tile<KMAX, true, BNT / 64>(taddr, col_base, Ml, s, gl);
        } else {
          epi_tile<KMAX, false, BNT / 64>(taddr, col_base, Ml, s, gl);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) ptx::mbar_arrive_cluster(&bars->tempty[acc], 0);
          else ptx::mbar_arrive(&bars->tempty[acc]);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (DYN && c + 1 < dyn.CS) {
        // not the range's last chunk: park both half-lists (coalesced [j][half][i][row]) and publish
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          __stcg(dyn.st_s + st_off + i * BM, s[i]);
          __stcg(dyn.st_g + st_off + i * BM, gl[i]);
        }
        epi_barrier();
        if (warp == 2 && lane == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(dyn.done + j),
                       "l"(((uint64_t)epoch << 32) | (uint32_t)(c + 1)) : "memory");
        }
      } else if (!DUMP) {
        // the upper-half warps hand their lists over; the lower half merges and writes
        if (half == 1) {
#pragma unroll
          for (int i = 0; i < KMAX; ++i) {
            list_s[row * KMAX + i] = s[i];
            list_g[row * KMAX + i] = gl[i];
          }
        }
        epi_barrier();
        if (half == 0) merge_lists<KMAX>(s, gl, list_s + row * KMAX, list_g + row * KMAX);
        if (dup) {   // second round: rows 64..127 (the copies) hand their merged lists to rows 0..63
          if (half == 0 && row >= 64) {
#pragma unroll
            for (int i = 0; i < KMAX; ++i) {
              list_s[row * KMAX + i] = s[i];
              list_g[row * KMAX + i] = gl[i];
            }
          }
          epi_barrier();
          if (half == 0 && row < 64) merge_lists<KMAX>(s, gl, list_s + (row + 64) * KMAX, list_g + (row + 64) * KMAX);
        }
        if (half == 0 && (!dup || row < 64)) {
          if (prompt < N) {
            Cand* dst = out + ((int64_t)r * N + prompt) * k;
#pragma unroll
            for (int i = 0; i < KMAX; ++i) {
              PAS_CHECK(gl[i] < (int64_t)M_local, "K2 top-k row beyond the shard");
              if (i < k) dst[i] = Cand{s[i], gl[i] < 0 ? -1 : gl[i] * G + rank};
            }
          }
        }
        epi_barrier();
      }
    }
  }

  ptx::tc_fence_before();
  if (PAIR) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if (PAIR) ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int KMAX, bool DUMP, bool PAIR, bool DYN = false, int BNT = BN>
cudaError_t launch_variant(const SimTopkArgs& a, int MT, int NT, int grid, uint32_t slack, cudaStream_t st) {
  using TL = Tile<PAIR, BNT>;
  static_assert(TL::NUM_WORKERS > 0 && TL::SMEM_BYTES <= 232448, "tile configuration");
  constexpr int CTAS = PAIR ? 2 : 1;   // cluster size
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = TL::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CTAS;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = PAIR ? 2 : 1;
  // the CTA pair and the B multicast read the cache through the 128-row box map
  return cudaLaunchKernelEx(&cfg, k_simtopk<KMAX, DUMP, PAIR, DYN, BNT>, *a.tmap_q,
                            (PAIR || BNT < BN) ? *a.tmap_c_pair : *a.tmap_c, a.N, a.M_local, a.d / BK, a.k, a.G,
                            a.rank, a.R, MT, NT, a.out, a.dump, a.progress, a.epoch, a.epoch_dev, slack, a.dyn,
                            a.dup ? 1 : 0);
}

}  // namespace

bool simtopk_pair(int64_t N, int d) {
  static const int max_tiles = [] {   // A/B experiments: PAS_K2_PAIR_MAX_TILES in the environment
    const char* v = getenv("PAS_K2_PAIR_MAX_TILES");
    return v ? atoi(v) : PAS_K2_PAIR_MAX_TILES;
  }();
  (void)d;
  // the pair covers 256 prompt rows per unit: with an odd number of 128-row tiles one CTA of a pair
  // computes only padding (C5, 50M rows: N = 128 8.0k vs 10.8k prompts/s single-CTA, N = 384 11.1k vs
  // 14.1k; N = 256 14.3k vs 12.9k), so the pair serves only whole pairs of tiles
  const int64_t tiles = (N + BM - 1) / BM;
  return tiles <= max_tiles && tiles % 2 == 0;
}
// Small problems (one prompt tile, at most 128 cache tiles of 128 rows): the 128-row cache tile, one per
// CTA -- twice the CTAs of the 256-row tile, each pulling half the bytes through its TMA and running half
// the MMA and epilogue (C1: 8 CTAs instead of 4).  Large caches keep 256-row tiles (the prompt tile is
// re-read from L2 once per cache tile).
bool simtopk_small(int64_t N, int64_t M_local, int d) {
  static const bool off = getenv("PAS_K2_NO_SMALL") != nullptr;   // A/B experiments
  return !off && N > 0 && N <= BM && !simtopk_pair(N, d) && M_local > 0 && (M_local + 127) / 128 <= 128;
}
int simtopk_tile_rows(int64_t N, int64_t M_local, int d) { return simtopk_small(N, M_local, d) ? 128 : BN; }

int64_t simtopk_dup_rows(int64_t N, int d) {
  static const bool off = getenv("PAS_K2_NO_DUP") != nullptr;   // A/B experiments
  return !off && N <= 64 && !simtopk_pair(N, d) ? 64 : 0;
}
int simtopk_prompt_rows() { return Tile<true>::UNIT_ROWS; }   // prompt buffers are padded to whole pair tiles
int simtopk_box_q() { return BM; }
int simtopk_box_c(int d) { return (void)d, Tile<false>::BN_CTA; }
int simtopk_box_c_pair() { return Tile<true>::BN_CTA; }
static int tile_rows(int d) { return (void)d, BN; }

// Opt the kernel variants into > 48 KB dynamic shared memory on the current device.
cudaError_t simtopk_init() {
  cudaError_t e;
  const int ss = Tile<false>::SMEM_BYTES, pr = Tile<true>::SMEM_BYTES, sm = Tile<false, 128>::SMEM_BYTES;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, false, false, false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<16, false, false, false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, false, false, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ss))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<16, false, false, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ss))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, false, false, true, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ss))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<16, false, false, true, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ss))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, true, false, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ss))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, false, true, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, pr))) return e;
  return cudaFuncSetAttribute(k_simtopk<16, false, true, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, pr);
}

// Dynamic schedule.  Static units (prompt tile, whole range) let the 148 CTAs drift apart over a range
// of thousands of tiles, so L2 stops covering the spread and tiles come from DRAM again (C4: 418 GB
// read per launch for a 15.4 GB cache); a leash that holds CTAs together costs more than it saves.
// Here units are short (T tiles of one range for one prompt tile), handed out by a global counter in
// (chunk step, range, prompt tile) order: whatever their speed, the CTAs stay within one chunk step of
// each other, so the cache crosses HBM about once, and fast SMs simply take more units.  Top-k lists
// are parked in global memory (L2-resident, 32 KB per unit for k <= 8) between a tile's chunks.
// Conditions: the single-CTA tile; at least PAS_K2_DYN_MIN_PAIRS x 148 (range, prompt tile) pairs, so
// the unit that resumes (r, m) is handed out that many units after the one that parks it (it almost
// never waits); R * N within the candidate buffer and R * MT within the parked-list buffer.
#ifndef PAS_K2_DYN_MB
#define PAS_K2_DYN_MB 100         // L2 budget for the chunks streamed concurrently
#endif
#ifndef PAS_K2_DYN_AMB
#define PAS_K2_DYN_AMB 4096       // L2 budget for one group's prompt tiles (MB; default: one group)
#endif
#ifndef PAS_K2_DYN_TMAX
#define PAS_K2_DYN_TMAX 128       // longest chunk (tiles)
#endif
#ifndef PAS_K2_DYN_MIN_PAIRS
#define PAS_K2_DYN_MIN_PAIRS 2
#endif
#ifndef PAS_K2_DYN_MIN_STEPS
#define PAS_K2_DYN_MIN_STEPS 2    // fewer chunk steps: the static schedule
#endif
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
K2Tuning K2Tuning::from_env() {
  K2Tuning t;
  const char* sched = getenv("PAS_K2_SCHED");
  t.force_static = sched && !strcmp(sched, "static");
  t.ranges = env_int("PAS_K2_RANGES", 0);
  t.no_leash = getenv("PAS_K2_NOLEASH") != nullptr;
  t.dyn_mb = env_int("PAS_K2_DYN_MB", PAS_K2_DYN_MB);
  t.dyn_tmax = env_int("PAS_K2_DYN_TMAX", PAS_K2_DYN_TMAX);
  t.dyn_min_pairs = env_int("PAS_K2_DYN_MIN_PAIRS", PAS_K2_DYN_MIN_PAIRS);
  t.dyn_min_steps = env_int("PAS_K2_DYN_MIN_STEPS", PAS_K2_DYN_MIN_STEPS);
  t.dyn_amb = env_int("PAS_K2_DYN_AMB", PAS_K2_DYN_AMB);
  return t;
}
bool simtopk_plan_dynamic(int64_t N, int64_t M_local, int64_t cand_rows, int64_t state_tiles, int d,
                          const K2Tuning& tune, int* R_out, int* T_out, int* CS_out, int* MTg_out) {
  const int budget_mb = tune.dyn_mb;
  if (budget_mb <= 0 || simtopk_pair(N, d)) return false;
  const int64_t MT = (N + BM - 1) / BM;
  const int64_t NT = (M_local + BN - 1) / BN;
  if (MT <= 0 || NT <= 0) return false;
  const int64_t rows = MT;
  const int64_t workers = Tile<false>::NUM_WORKERS;
  const int64_t want = (int64_t)tune.dyn_min_pairs * workers;
  // prompt-tile groups: every chunk step of a group re-reads all of its prompt tiles (A, kept in L2
  // with evict_last), so a group's A must leave L2 room for the chunks; each group streams the cache
  // once.  Never split below `want` (range, prompt tile) pairs per group.
  const int64_t a_bytes = (int64_t)MT * BM * d * 2;
  const int64_t a_budget = (int64_t)std::max(tune.dyn_amb, 1) << 20;
  int64_t groups = std::min<int64_t>((a_bytes + a_budget - 1) / a_budget, rows), MTg, R;
  const int64_t slots_per_range = MT;   // parked-list slots
  for (;; --groups) {   // fewer groups (more ranges per group) until the candidate buffers hold R ranges
    MTg = (rows + groups - 1) / groups;
    R = std::min<int64_t>((want + MTg - 1) / MTg, 128);   // the S-way merge takes S <= 128 sources
    if (groups == 1 || (R <= NT && R * N <= cand_rows && R * slots_per_range <= state_tiles)) break;
  }
  if (R > NT || R * N > cand_rows || R * slots_per_range > state_tiles) return false;
  if (R * MTg < workers) return false;      // less than one unit per worker per chunk step
  // chunks in flight: the ranges one window of `workers` consecutive units spans, plus the next step's
  const int64_t in_flight = (workers + MTg - 1) / MTg + 1;
  const int64_t tile_bytes = (int64_t)BN * d * 2;
  const int64_t L = (NT + R - 1) / R;             // tiles of the longest range
  int64_t T = ((int64_t)budget_mb << 20) / (in_flight * tile_bytes);
  // short ranges: at least ~kTargetSteps chunk steps, so the units balance across the SMs (C2:
  // 40-tile ranges in 6 chunks of 7 measured 3-5 % faster than the static schedule)
  constexpr int64_t kTargetSteps = 6;
  T = std::min(T, (L + kTargetSteps - 1) / kTargetSteps);
  if (T < 4) T = 4;
  const int tmax = tune.dyn_tmax;
  if (T > tmax) T = tmax;
  if (L < tune.dyn_min_steps * T) return false;   // too short to chunk
  *R_out = (int)R;
  *T_out = (int)T;
  *CS_out = (int)((L + T - 1) / T);
  *MTg_out = (int)MTg;
  return true;
}

// Pick the number of cache ranges R so that (prompt tiles x R) units fill the persistent workers with
// the smallest makespan: waves(R) * (tiles per unit + WARMUP_TILES), subject to the candidate buffer
// (R * N <= cand_rows).  WARMUP_TILES prices a unit's start: while a fresh top-k list is filling,
// nearly every 32-column chunk of some lane takes the insert path (P(insert) ~ 32 k / columns seen),
// which makes the first ~8k columns of a unit epilogue-bound rather than MMA-bound.
int simtopk_choose_ranges(int64_t N, int64_t M_local, int64_t cand_rows, int d) {
  if (simtopk_small(N, M_local, d)) {   // one 128-row tile per CTA (as many as the candidate buffer holds)
    int64_t R = (M_local + 127) / 128;
    while (R > 1 && R * N > cand_rows) --R;
    return (int)R;
  }
  const bool pair = simtopk_pair(N, d);
  const int UNIT_ROWS = pair ? Tile<true>::UNIT_ROWS : Tile<false>::UNIT_ROWS;
  const int NUM_WORKERS = pair ? Tile<true>::NUM_WORKERS : Tile<false>::NUM_WORKERS;
  const int64_t MT = (N + UNIT_ROWS - 1) / UNIT_ROWS;
  const int64_t NT = (M_local + tile_rows(d) - 1) / tile_rows(d);
  const double warmup = (double)WARMUP_TILES * BN / tile_rows(d);
  if (NT <= 1 || MT <= 0) return 1;
  int best = 1;
  double best_cost = 1e300;
  const int64_t rmax = NT < 128 ? NT : 128;   // the S-way merge takes S <= 128 sources
  for (int64_t R = 1; R <= rmax; ++R) {
    if (R > 1 && R * N > cand_rows) break;
    const int64_t waves = (MT * R + NUM_WORKERS - 1) / NUM_WORKERS;
    const double cost = (double)waves * ((double)((NT + R - 1) / R) + warmup);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = (int)R; }
  }
  return best;
}

// Leash slack in tiles (0 = off): the ranges streamed concurrently by one wave of `workers` CTAs,
// each spread over at most `slack` tiles, must fit in PAS_K2_LEASH_MB of L2 next to the prompt tiles.
// Measured on one B200 (profiles/r01_leash/): the leash cuts K2's DRAM reads at C4 from
// 491 GB to 73 GB per launch but costs 9 % throughput there (CTAs wait for the slowest SM; DRAM is
// not K2's bound), and gains 4-6 % only when many ranges are streamed at once (MT <= 16 prompt
// tiles, i.e. N <= 2048).  So it is on only in that regime, and off when units are short or a
// range has a single reader.
#ifndef PAS_K2_LEASH_MB
#define PAS_K2_LEASH_MB 48
#endif
uint32_t simtopk_leash_slack(int MT, int NT, int R, int workers) {
  if (PAS_K2_LEASH_MB <= 0 || MT < 2 || MT > 16 || workers < 2) return 0;
  const int64_t tiles_per_unit = ((int64_t)NT + R - 1) / R;
  const int64_t ranges = MT >= workers ? 2 : (workers + MT - 1) / MT + 1;   // +1: a wave straddles two
  const int64_t tile_bytes = (int64_t)BN * 768 * 2;
  int64_t slack = ((int64_t)PAS_K2_LEASH_MB << 20) / (ranges * tile_bytes);
  if (slack < 2) slack = 2;
  if (slack > 64) slack = 64;
  if (tiles_per_unit < 8 * slack) return 0;
  return (uint32_t)slack;
}

cudaError_t launch_simtopk(const SimTopkArgs& a, cudaStream_t st) {
  const bool pair = !a.dump && simtopk_pair(a.N, a.d);
  const int UNIT_ROWS = pair ? Tile<true>::UNIT_ROWS : Tile<false>::UNIT_ROWS;
  const int NUM_WORKERS = pair ? Tile<true>::NUM_WORKERS : Tile<false>::NUM_WORKERS;
  const int CTAS = pair ? 2 : 1;
  const int MT = (int)((a.N + UNIT_ROWS - 1) / UNIT_ROWS);
  const bool small = !a.dump && a.dyn.T == 0 && simtopk_small(a.N, a.M_local, a.d);
  const int tr = small ? 128 : tile_rows(a.d);
  const int NT = (int)((a.M_local + tr - 1) / tr);
  if (MT == 0 || NT == 0) return cudaSuccess;
  const int units = MT * a.R;
  const int workers = units < NUM_WORKERS ? units : NUM_WORKERS;
  const int grid = CTAS * workers;
  if (a.dyn.T > 0 && !pair && !a.dump) {
    const int g = NUM_WORKERS;   // every SM: units are handed out dynamically
    if (a.k <= 8) return launch_variant<8, false, false, true>(a, MT, NT, g, 0, st);
    return launch_variant<16, false, false, true>(a, MT, NT, g, 0, st);
  }
  const uint32_t slack = a.progress ? simtopk_leash_slack(MT, NT, a.R, workers) : 0;
  if (a.dump) return launch_variant<8, true, false>(a, MT, NT, grid, slack, st);
  if (pair) {
    if (a.k <= 8) return launch_variant<8, false, true>(a, MT, NT, grid, slack, st);
    return launch_variant<16, false, true>(a, MT, NT, grid, slack, st);
  }
  if (small) {
    if (a.k <= 8) return launch_variant<8, false, false, false, 128>(a, MT, NT, grid, 0, st);
    return launch_variant<16, false, false, false, 128>(a, MT, NT, grid, 0, st);
  }
  if (a.k <= 8) return launch_variant<8, false, false>(a, MT, NT, grid, slack, st);
  return launch_variant<16, false, false>(a, MT, NT, grid, slack, st);
}

}  // namespace pas
