// K2 -- prompt x cache cosine-similarity GEMM on tcgen05 tensor cores with a fused running top-k.
//
// Paper: the Optimal-K Selector "first retrieves the nearest cache" by prompt
// "closeness".  Both operands are unit rows in bf16 (K1), so S = Q_hat C_hat^T is the cosine
// similarity; it is accumulated in fp32 in TMEM and never written to memory: each epilogue thread
// owns one prompt row of the accumulator and keeps the k best (score desc, gid asc; R10) over the
// cache range of its work unit.
//
// CTA pairs (cluster of 2, tcgen05 cta_group::2): one MMA instruction computes a 256 x 256 x 16
// tile, prompt rows 0..127 from CTA 0's shared memory and TMEM, rows 128..255 from CTA 1's; the 256
// cache rows of B are split 128 / 128 between the two CTAs' shared memory, so each SM stages half of
// the big operand (half the smem traffic of a 1-CTA 128 x 256 tile for the same per-SM MMA rate).
//
// Work unit = (prompt pair-tile m of 256 rows, cache range r of whole 256-row tiles).  Persistent
// pairs (74 on 148 SMs) walk units u = cluster + i*clusters with m fastest, so concurrently running
// pairs stream the SAME cache tiles (L2 reuse of the big operand) against different prompt tiles.
//
// Warp roles per CTA (192 threads, 1 CTA/SM):
//   warp 0      TMA producer: its 128 prompt rows and its 128 cache rows of each 64-wide k-block
//               (128-B swizzle) into a 6-stage ring (32 KB / stage); completion bytes of BOTH CTAs
//               land on the leader's "full" mbarrier.
//   warp 1      TMEM allocation (cta_group::2, 512 columns = two 256-column fp32 accumulators); in
//               the leader one lane issues tcgen05.mma.cta_group::2 (M=256, N=256, K=16) and
//               commits smem stages (multicast to both CTAs' "empty") and accumulators (both
//               CTAs' "tfull").
//   warps 2..5  epilogue over this CTA's 128 TMEM lanes: tcgen05.ld 32 columns at a time, chunk max
//               vs the current k-th score, branch-free bubble insert only when the chunk can improve
//               the list; then arrive on the leader's "tempty" (8 arrivals: 4 warps x 2 CTAs).
#include <cfloat>
#include <cstdio>

#include "pas_internal.cuh"
#include "ptx_sm100.cuh"

namespace pas {
namespace {

constexpr int BM = 128;           // prompt rows per CTA (256 per pair)
constexpr int BN = 256;           // cache rows per tile (128 staged per CTA)
constexpr int BN_CTA = BN / 2;
constexpr int BK = 64;
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN_CTA * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // per CTA
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;
constexpr int NUM_PAIRS = kNumSMs / 2;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct __align__(8) Bars {
  uint64_t full[STAGES];    // leader: TMA bytes of both CTAs landed
  uint64_t empty[STAGES];   // both: MMA finished reading the stage
  uint64_t tfull[2];        // both: accumulator ready
  uint64_t tempty[2];       // leader: both epilogues drained the accumulator
  uint32_t tmem_base;
};

template <int KMAX, bool DUMP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_simtopk(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmC, int64_t N,
              int64_t M_local, int kblocks, int k, int G, int rank, int R, int MT, int NT, Cand* __restrict__ out,
              float* __restrict__ dump) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  Bars* bars = reinterpret_cast<Bars*>(smem + STAGES * STAGE_BYTES);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t crank = ptx::cluster_ctarank();
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int units = MT * R;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmQ);
    ptx::prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&bars->full[s], 1);
      ptx::mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&bars->tfull[a], 1);
      ptx::mbar_init(&bars->tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc_pair(&bars->tmem_base, TMEM_COLS);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------- TMA producer (both CTAs) -------------------------------
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < units; u += npairs) {
        const int m = u % MT, r = u / MT;
        const int t0 = (int)((int64_t)r * NT / R), t1 = (int)((int64_t)(r + 1) * NT / R);
        const int qrow = m * (2 * BM) + (int)crank * BM;
        for (int t = t0; t < t1; ++t) {
          const int crow = t * BN + (int)crank * BN_CTA;
          for (int kb = 0; kb < kblocks; ++kb) {
            ptx::mbar_wait(&bars->empty[stage], phase ^ 1);
            if (leader) ptx::mbar_arrive_expect_tx(&bars->full[stage], 2 * STAGE_BYTES);
            ptx::tma_load_2d_pair(&tmQ, sA + stage * A_BYTES, &bars->full[stage], kb * BK, qrow, ptx::kEvictLast);
            ptx::tma_load_2d_pair(&tmC, sB + stage * B_BYTES, &bars->full[stage], kb * BK, crow,
                                  ptx::kEvictNormal);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer (leader CTA) --------------------------------
    if (leader && ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < units; u += npairs) {
        const int r = u / MT;
        const int t0 = (int)((int64_t)r * NT / R), t1 = (int)((int64_t)(r + 1) * NT / R);
        for (int t = t0; t < t1; ++t) {
          ptx::mbar_wait(&bars->tempty[acc], acc_phase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < kblocks; ++kb) {
            ptx::mbar_wait(&bars->full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(sA + stage * A_BYTES);
            const uint32_t b0 = ptx::smem_u32(sB + stage * B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              ptx::umma_f16_ss_pair(d_tmem, ptx::sdesc_kmajor_sw128(a0 + kk * 32),
                                    ptx::sdesc_kmajor_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
            }
            ptx::umma_commit_pair(&bars->empty[stage], 0x3);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          ptx::umma_commit_pair(&bars->tfull[acc], 0x3);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------- epilogue (both CTAs) -----------------------------------
    const uint32_t q = warp & 3;              // TMEM lane quarter this warp may access
    const int row = (int)(q * 32 + lane);
    const uint32_t lane_addr = tmem_base + ((q * 32u) << 16);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < units; u += npairs) {
      const int m = u % MT, r = u / MT;
      const int t0 = (int)((int64_t)r * NT / R), t1 = (int)((int64_t)(r + 1) * NT / R);
      const int64_t prompt = (int64_t)m * (2 * BM) + crank * BM + row;
      float s[KMAX];
      int32_t g[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) { s[i] = -INFINITY; g[i] = -1; }
      for (int t = t0; t < t1; ++t) {
        ptx::mbar_wait(&bars->tfull[acc], acc_phase);
        ptx::tc_fence_after();
        const int64_t col_base = (int64_t)t * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(lane_addr + acc * BN + c * 32, v);
          ptx::tmem_wait_ld();
          const int64_t col0 = col_base + c * 32;
          if (DUMP) {
            if (prompt < N) {
              for (int j = 0; j < 32; ++j)
                if (col0 + j < M_local) dump[prompt * M_local + col0 + j] = __uint_as_float(v[j]);
            }
            continue;
          }
          if (col0 + 32 > M_local) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j >= M_local) v[j] = __float_as_uint(-INFINITY);
          }
          float mx = __uint_as_float(v[0]);
#pragma unroll
          for (int j = 1; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
          if (mx > s[KMAX - 1]) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float x = __uint_as_float(v[j]);
              if (x > s[KMAX - 1]) {
                s[KMAX - 1] = x;
                g[KMAX - 1] = (int32_t)((col0 + j) * G + rank);
#pragma unroll
                for (int i = KMAX - 1; i > 0; --i) {
                  if (s[i] > s[i - 1]) {
                    const float ts = s[i]; s[i] = s[i - 1]; s[i - 1] = ts;
                    const int32_t tg = g[i]; g[i] = g[i - 1]; g[i - 1] = tg;
                  }
                }
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(&bars->tempty[acc], 0);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (!DUMP && prompt < N) {
        Cand* dst = out + ((int64_t)r * N + prompt) * k;
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
          if (i < k) dst[i] = Cand{s[i], g[i]};
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

template <int KMAX, bool DUMP>
cudaError_t launch_variant(const SimTopkArgs& a, int MT, int NT, int grid, cudaStream_t st) {
  auto kern = k_simtopk<KMAX, DUMP>;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(*a.tmap_q, *a.tmap_c, a.N, a.M_local, a.d / BK, a.k, a.G, a.rank,
                                              a.R, MT, NT, a.out, a.dump);
  return cudaGetLastError();
}

}  // namespace

size_t simtopk_smem_bytes() { return SMEM_BYTES; }
int simtopk_prompt_rows() { return 2 * BM; }
int simtopk_box_q() { return BM; }
int simtopk_box_c() { return BN_CTA; }

// Opt the kernel variants into > 48 KB dynamic shared memory on the current device.
cudaError_t simtopk_init() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_simtopk<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES))) return e;
  if ((e = cudaFuncSetAttribute(k_simtopk<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES))) return e;
  return cudaFuncSetAttribute(k_simtopk<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

// Pick the number of cache ranges R so that (prompt pair-tiles x R) units fill the 74 CTA pairs with
// the smallest makespan: waves(R) * (tiles per unit + 1 tile of per-unit overhead).
int simtopk_choose_ranges(int64_t N, int64_t M_local) {
  const int64_t MT = (N + 2 * BM - 1) / (2 * BM);
  const int64_t NT = (M_local + BN - 1) / BN;
  if (NT <= 1 || MT <= 0) return 1;
  int best = 1;
  double best_cost = 1e300;
  const int64_t rmax = NT < 64 ? NT : 64;
  for (int64_t R = 1; R <= rmax; ++R) {
    if (R > 1 && MT * R > 8 * NUM_PAIRS) break;
    const int64_t waves = (MT * R + NUM_PAIRS - 1) / NUM_PAIRS;
    const double cost = (double)waves * (double)((NT + R - 1) / R + 1);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = (int)R; }
  }
  return best;
}

cudaError_t launch_simtopk(const SimTopkArgs& a, cudaStream_t st) {
  const int MT = (int)((a.N + 2 * BM - 1) / (2 * BM));
  const int NT = (int)((a.M_local + BN - 1) / BN);
  if (MT == 0 || NT == 0) return cudaSuccess;
  const int units = MT * a.R;
  const int pairs = units < NUM_PAIRS ? units : NUM_PAIRS;
  const int grid = 2 * pairs;
  if (a.dump) return launch_variant<8, true>(a, MT, NT, grid, st);
  if (a.k <= 8) return launch_variant<8, false>(a, MT, NT, grid, st);
  return launch_variant<16, false>(a, MT, NT, grid, st);
}

}  // namespace pas
