// pas_internal.cuh -- shared device/host definitions of libpas (sm_100a only).
//
// Nothing in here is imported by, or imports, the CPU oracle (oracle/).  See include/pas.h for the
// public C-ABI and DESIGN.md for the data layout and the roofline of every kernel.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include <utility>

#include "../../include/pas.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libpas is written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace pas {

// Programmatic dependent launch: every kernel of the batch pipeline is launched with
// programmatic stream serialization and starts with pdl_entry(), which lets the NEXT kernel be
// scheduled immediately (its launch latency hides behind this one) and then waits until the
// PREVIOUS kernel has completed and its writes are visible.  Outside PDL both are no-ops.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// zero up to three int32 buffers in one launch
cudaError_t launch_zero(int32_t* a, int64_t na, int32_t* b, int64_t nb, int32_t* c, int64_t nc, cudaStream_t st);

constexpr int kMaxLevels = PAS_MAX_LEVELS;
constexpr int kMaxInst = PAS_MAX_INSTANCES;
constexpr int kTTotal = PAS_T_TOTAL;
constexpr int kNumSMs = 148;

// Checked build (python -m paper_2502_06798_b200.build -DPAS_CHECKED=1 --out=...): device-side bounds
// and protocol checks on the indices the kernels compute (work units, parked-list slots, candidate,
// list and batch-list positions); a failed check prints its site and traps.  The product build compiles
// them out.  (compute-sanitizer is not available on this GPU pool.)
#ifndef PAS_CHECKED
#define PAS_CHECKED 0
#endif
#if PAS_CHECKED
#define PAS_CHECK(cond, what)                                                                             \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("PAS_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                            \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define PAS_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

// Candidate pair (score, global cache id); ordered by score desc, gid asc (R10).  Sentinel (-inf, -1).
struct __align__(8) Cand {
  float s;
  int32_t g;
};

__host__ __device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  return a.s > b.s || (a.s == b.s && (unsigned)a.g < (unsigned)b.g);
}

// f3 stateful dispatcher (R28-R32): per-instance queue state, kept on the device across
// batches, and the per-batch pick tables the prep kernel derives from it.
constexpr int kArrRing = 64;                         // arrival times kept per instance (b* <= 64, R30)
constexpr int64_t kNeverBusy = PAS_NEVER_BUSY;
struct DispState {
  int64_t Q[kMaxInst];                 // waiting prompts
  int64_t B[kMaxInst];                 // busy-until (us), kNeverBusy before the first batch
  int64_t E[kMaxInst];                 // prompts ever enqueued (arrival ring index)
  int64_t fired_prompts[kMaxInst], fired_batches[kMaxInst];
  int64_t svc[kMaxInst];               // batch service time (us)
  int64_t arr[kMaxInst][kArrRing];     // arrival time of enqueue number e at arr[w][e % 64]
};
struct DispPlan {
  int64_t Q0[kMaxInst];                // queue the batch found (after the events since the last batch)
  int64_t Q1[kMaxInst];                // queue after phase 1 (max(Q0, b*))
  int64_t Bp[kMaxInst];                // max(busy-until, now)
  int64_t svc[kMaxInst];
  double inv_svc[kMaxInst];
  int32_t p1_w[kMaxInst];              // phase-1 fill order, grouped by level: [p1_beg[j], p1_beg[j+1])
  int32_t p1_cum[kMaxInst];            // prompts of the level placed before this entry
  int32_t p1_beg[kMaxLevels + 1];
  int32_t p1_total[kMaxLevels];        // phase-1 capacity of the level
  int32_t cnt[kMaxInst];               // this batch's prompts per instance
};

// Per-batch parameters, passed BY VALUE to the kernels that need them (no upload, no host sync).
// Per-batch counters kept on the device so a batch's kernels need no per-call host state (CUDA-graph
// replay, pas_set_graph): the Philox batch sequence (R18), the f2 LRU tick of the next batch (R26), and
// the K2 launch epoch.  The last kernel of each batch advances batch_seq and lru_tick; K1 on the prompt
// path advances k2_epoch before the K2 that follows it.
struct BatchCounters {
  uint64_t batch_seq;
  uint32_t lru_tick;
  uint32_t k2_epoch;
};

struct RouteParams {
  int nK, W, bstar, mode, topk, G, rank, d;
  int64_t N, M_total;
  int64_t cand_stride;           // candidate rows between the S source blocks [S][stride][k] (0: N)
  uint64_t seed, batch_seq;
  int kb;                        // K6 bucket bits of kappa
  int bstar_shift;               // log2(bstar) if bstar is a power of two, else -1
  int grid[kMaxLevels];          // K values
  float thr[kMaxLevels];         // nK-1 thresholds
  double F[kMaxLevels];          // load fractions
  double c[kTTotal];             // degradation c(dK)
  int convex;                    // c convex: K5 takes the NW-corner closed form (R6, R7)
  int k6_force_fallback;         // tests: K6 takes its exact histogram path
  int64_t cI[kTTotal];           // non-convex c: round-half-even(c * 2^24), K5's exact integer costs (R37)
  int inst_level[kMaxInst];      // level index of each serving instance
  uint32_t* lru_stamp;           // f2: [global slots] last-use ticks (K4 stamps each usable top-1)
  uint32_t lru_tick;             // this batch's tick (when bc == nullptr)
  BatchCounters* bc;             // device counters (batch_seq, lru_tick override the fields above)
  // f3 stateful dispatcher (disp == 0: the stateless packing of R13 / R14)
  int disp;
  int bstar_prev;                // b* in force since the last batch (events in between, R28)
  int64_t now_us, timeout_us;
  DispState* dstate;
  DispPlan* dplan;
};

// K6 windows (k_redirect.cu): per class the distinct split ranks 0 < X < h of its plan row, each with
// the kappa window [lo, hi) its order statistic lies in with probability 1 - 1e-15 (mean +- 8 sd of the
// X-th of h uniforms); overlapping windows merged into zones.  At most nK - 1 splits exist (a basic
// plan has <= 2 nK - 1 nonzeros); more, a list overflow or a split outside its zone sets k6_fallback
// and the exact histogram path runs instead.
constexpr int kMaxZones = 32;
// K6's windowed split search serves batches of at least this many prompts (k_redirect.cu); below, the
// exact histogram path runs alone and K5 skips the windows.
constexpr int64_t kWindowMinN = 1 << 18;

// Device-side plan + counters of one batch (K5 writes, pas_plan_stats reads).
struct DevPlan {
  int h[kMaxLevels];
  int f[kMaxLevels];
  int x[kMaxLevels][kMaxLevels];
  int X[kMaxLevels][kMaxLevels];     // inclusive prefix sums of the rows of x
  int class_start[kMaxLevels + 1];   // exclusive prefix of h
  int n_inst[kMaxLevels];
  uint32_t n_inst_recip[kMaxLevels];   // ceil(2^32 / n_j) for n_j > 1, 0 for n_j <= 1: q div n_j ==
                                       // umulhi(q, recip) for q < 2^26 (the error < n_j times q stays < 2^32)
  alignas(16) int inst_list[kMaxLevels][kMaxInst];   // 16-byte aligned: K7 stages it with int4 copies
  int inst_pos[kMaxInst];              // position of instance i in inst_list[its level] (K7's closed form)
  int inst_base[kMaxLevels];           // #instances at levels < j: I_j's first entry in a level-ordered list
  double D_Q, D_Q_LP;
  int n_redirected, n_upgraded, n_downgraded;
  int n_invalid, n_near_top1, n_near_threshold;
  int inst_count[kMaxInst];
  int solver_iters;                  // non-convex K5: min-cost-flow augmentations (+ lex-max cycles); -1: cap hit
  // K6 windowed split search (written by K5, filled by the fused pass, resolved per zone)
  int k6_nz, k6_fallback;
  int cls_zone0[kMaxLevels], cls_nzone[kMaxLevels], cls_jtot[kMaxLevels], cls_slot0[kMaxLevels];
  int z_cls[kMaxZones], z_first[kMaxZones], z_nsplit[kMaxZones], z_jbelow[kMaxZones], z_cap[kMaxZones],
      z_base[kMaxZones], z_fill[kMaxZones];
  uint64_t z_lo[kMaxZones], z_hi[kMaxZones];
  int s_X[kMaxZones], s_mult[kMaxZones];
  int gapcnt[kMaxLevels + kMaxZones];   // class prompts per (class, gap) slot: slot cls_slot0[i] + g
  uint64_t s_thr_k[kMaxZones];          // each split's threshold entry (kappa, p): the prompt at rank X
  int s_thr_p[kMaxZones];
};
constexpr int kDegShift = 24;        // R37: non-convex c held as integers on a 2^-24 grid

// ------------------------------------------------------------------------------------------------
// launchers (each returns cudaGetLastError() of its launch)
// ------------------------------------------------------------------------------------------------
// K1: normalise + quantise rows; shard filter (first_gid + i) % G == rank -> local row (first_gid+i)/G
cudaError_t launch_normalize(const void* in, pas_dtype dtype, int64_t rows, int d, __nv_bfloat16* out,
                             uint8_t* flags, int64_t first_gid, int G, int rank, int* invalid_count,
                             cudaStream_t st, uint32_t* epoch_bump = nullptr, int64_t dup_rows = 0);
// dup_rows > 0: each row is also written dup_rows rows further down (K2's duplicated-row small-batch
// epilogue, SimTopkArgs::dup)

__device__ __forceinline__ uint64_t batch_seq_of(const RouteParams& P) {
  return P.bc ? P.bc->batch_seq : P.batch_seq;
}
__device__ __forceinline__ uint32_t lru_tick_of(const RouteParams& P) {
  return P.bc ? P.bc->lru_tick : P.lru_tick;
}
// The last kernel of a batch, one thread: the next batch's Philox sequence and LRU tick.
__device__ __forceinline__ void advance_batch_counters(const RouteParams& P) {
  if (P.bc && blockIdx.x == 0 && threadIdx.x == 0) {
    P.bc->batch_seq += 1;
    P.bc->lru_tick += 1;
  }
}

// K2 dynamic schedule (DESIGN.md 8 "K2 schedule"): units (chunk step, range, prompt tile) handed out
// in that order by a global counter; each (range, prompt tile) parks its two half top-k lists between
// chunks and publishes "chunks done" (epoch-tagged) for the unit that resumes them.
struct DynSched {
  int T = 0;                    // cache tiles per chunk
  int CS = 0;                   // chunk steps per range
  int MTg = 0;                  // prompt tiles per group (each group streams the cache once)
  float* st_s = nullptr;        // [R*MT][2][KMAX][128] parked scores
  int32_t* st_g = nullptr;      // [R*MT][2][KMAX][128] parked local rows
  uint64_t* done = nullptr;     // [R*MT] epoch << 32 | chunks done
  uint32_t* sched = nullptr;    // [2] unit counter, workers finished (zero between launches)
  int slots = 0;                // parked-list slots allocated (R * MT <= slots; checked builds)
};

// K2 schedule knobs for A/B experiments.  Read from the environment once per context at
// pas_create (K2Tuning::from_env), never on the routing path; defaults are the measured choices.
struct K2Tuning {
  bool force_static = false;   // PAS_K2_SCHED=static: the static ranges even where the dynamic schedule applies
  int ranges = 0;              // PAS_K2_RANGES: static-schedule ranges (0: chosen by the cost model)
  bool no_leash = false;       // PAS_K2_NOLEASH: static schedule without the progress leash
  int dyn_mb = 0;              // PAS_K2_DYN_MB: L2 budget (MB) for the chunks in flight
  int dyn_tmax = 0;            // PAS_K2_DYN_TMAX: longest chunk (tiles)
  int dyn_min_pairs = 0;       // PAS_K2_DYN_MIN_PAIRS: (range, prompt tile) pairs per group, in units of 148
  int dyn_min_steps = 0;       // PAS_K2_DYN_MIN_STEPS: fewest chunk steps for the dynamic schedule
  int dyn_amb = 0;             // PAS_K2_DYN_AMB: L2 budget (MB) for one group's prompt tiles
  static K2Tuning from_env();
};

// K2: similarity GEMM (tcgen05) + fused running top-k over cache ranges.
struct SimTopkArgs {
  const CUtensorMap* tmap_q;      // [rows_q x d] bf16, box 64 x simtopk_box_q(), SW128
  const CUtensorMap* tmap_c;      // [rows_c x d] bf16, box 64 x simtopk_box_c(), SW128
  const CUtensorMap* tmap_c_pair; // the same store, box 64 x simtopk_box_c_pair() (CTA-pair tile)
  int64_t N;                      // prompts
  int64_t M_local;                // valid store rows on this rank
  int d, k, G, rank, R;           // R cache ranges per prompt tile
  const __nv_bfloat16* qhat;      // [rows_q x d] (A-in-TMEM variant reads the prompt rows directly)
  Cand* out;                      // [R][N][k]
  float* dump;                    // test hook: [N x M_local] raw scores instead of top-k (or null)
  uint64_t* progress;             // [kNumSMs] leash words (epoch << 32 | tiles issued), or null: no leash
  uint32_t epoch;                 // this launch's epoch (never 0: zeroed words read as "not started")
  const uint32_t* epoch_dev;      // or, if set, read from here after the PDL wait (bumped by K1)
  DynSched dyn;                   // T > 0: the dynamic schedule (simtopk_plan_dynamic)
  int dup = 0;                    // 1: N <= 64 on the single-CTA static tile and K1 wrote every prompt
                                  // row again at row + 64, so the epilogue splits each row's columns
                                  // over all four TMEM lane quarters (simtopk_dup_rows)
};
// Batches of at most this many prompts take K2's duplicated-row epilogue (K1 writes row p also at
// p + 64); 0 for other shapes.
int64_t simtopk_dup_rows(int64_t N, int d);
// Small problems take a 128-row cache tile (simtopk_small); simtopk_tile_rows: 128 or 256.
bool simtopk_small(int64_t N, int64_t M_local, int d);
int simtopk_tile_rows(int64_t N, int64_t M_local, int d);
cudaError_t launch_simtopk(const SimTopkArgs& a, cudaStream_t st);
int simtopk_choose_ranges(int64_t N, int64_t M_local, int64_t cand_rows, int d);
// The dynamic schedule's ranges R and chunk T for this batch, or false when the static schedule
// serves it (CTA-pair tile, too few units, or more parked lists than `state_tiles` prompt tiles).
bool simtopk_plan_dynamic(int64_t N, int64_t M_local, int64_t cand_rows, int64_t state_tiles, int d,
                          const K2Tuning& tune, int* R, int* T, int* CS, int* MTg);
bool simtopk_pair(int64_t N, int d);   // the CTA-pair tile serves this batch size
cudaError_t simtopk_init();
int simtopk_prompt_rows();   // prompt rows per work unit (pair tile)
int simtopk_box_q();         // TMA box rows of the prompt map
int simtopk_box_c(int d);    // TMA box rows of the cache map
int simtopk_box_c_pair();    // TMA box rows of the cache map for the CTA-pair tile

// K3 (+K4 when final): merge [S][N][k] -> [N][k]
cudaError_t launch_merge(const Cand* in, int S, int64_t N, int k, Cand* out, cudaStream_t st);
struct SelectOut {
  int32_t* K;           // [N] (required)
  int32_t* topk_id;     // [N*k] optional
  float* topk_score;    // [N*k] optional
  uint8_t* flags;       // [N] optional
  uint8_t* level;       // [N] workspace
  Cand* cand_out;       // [N*k] optional (merged candidates)
  int* hist;            // [nK] workspace (zeroed by caller)
  DevPlan* plan;        // counters
};
cudaError_t launch_merge_select(const Cand* in, int S, const uint8_t* pflags, const RouteParams& p,
                                const SelectOut& o, cudaStream_t st);
// The latency path (k_small.cu): a4 .. a8 of a batch of N <= kSmallMax prompts in one CTA (stateless
// exact-plan modes), byte-identical to the multi-kernel chain it replaces.
constexpr int kSmallMax = 1024;
struct SmallOut {
  int32_t *K, *K_prime, *instance, *slot;
  int32_t* topk_id;          // optional
  float* topk_score;         // optional
  uint8_t* flags;            // optional
  int32_t *bucket_offsets, *bucket_prompts;   // optional
  uint8_t* level;            // workspace [N]
  DevPlan* plan;
};
cudaError_t launch_small_route(const Cand* in, int S, const uint8_t* pflags, const RouteParams& p, const SmallOut& o,
                               cudaStream_t st);

// Explicit-N2 mode (pas_set_collectives): the per-prompt results of every rank's prompt slice, gathered
// in prompt order (all_cand [N][k], all_K / all_level / all_flags [N]), copied into the outputs, with
// the LRU stamps of every usable top-1 (R26; the slice merges do not stamp).
cudaError_t launch_unpack_slices(const Cand* all_cand, const int32_t* all_K, const uint8_t* all_level,
                                 const uint8_t* all_flags, const RouteParams& p, const SelectOut& o,
                                 cudaStream_t st);

// K5 plan
cudaError_t launch_plan(const int* hist, const RouteParams& p, DevPlan* plan, cudaStream_t st);

// K6 redirection
struct __align__(16) KeyEntry {
  uint64_t key;           // kappa (60-bit Philox key)
  int32_t p;              // prompt index
  int32_t pad;
};
constexpr int kMaxK6Bits = 18;      // K6 buckets per class <= 2^18
struct K6Bounds {                   // per class i, split j: the bucket holding split rank X_i[j] (INT32_MAX:
  int32_t bucket[kMaxLevels][kMaxLevels];   // none), the split's rank inside it, its candidate list
  int32_t off[kMaxLevels][kMaxLevels];
  int32_t list[kMaxLevels][kMaxLevels];
};
struct K6List {                     // one bucket holding one or more splits of a class
  int32_t cls, bucket, cnt, base, fill, below;
};
struct RedirectWs {
  uint64_t* key;          // [N] kappa
  int32_t* hist;          // [kMaxLevels << kMaxK6Bits] (class, bucket) counts, zeroed per batch
  int32_t* used;          // [2] lists, candidate entries (zeroed per batch)
  int32_t* csum;          // [kMaxLevels * 256] chunk sums of the bucket counts
  K6Bounds* bnd;
  K6List* lists;          // [kMaxLevels * kMaxLevels]
  KeyEntry* cand;         // [N] entries of the split buckets
  uint8_t* cls7;          // [N] class for K7 (K' level in greedy, instance in uniform)
};
int redirect_kb(int64_t N);
// blk_counts / ntiles / nC: the K7 per-tile class counts, produced by the windowed pass (k_cls_count then
// only runs on the fallback, gated on plan->k6_fallback).
cudaError_t launch_redirect(const uint8_t* level, const RouteParams& p, DevPlan* plan,
                            const RedirectWs& w, int32_t* K_prime, int32_t* blk_counts, int ntiles, int nC,
                            cudaStream_t st, int* launches, bool* counts_ready);

// f1 forecast-driven mode (R21-R24): predictor ring buffer + fixed-point Route-Plan.
struct FcState {
  int32_t head, n;                  // ring write position, valid entries (<= window)
  int32_t cnt[kMaxLevels];          // level counts over the window (after the last batch)
  int32_t plan_cnt[kMaxLevels];     // the counts the held plan was built from
  int32_t plan_n;
  int32_t replanned;                // this batch rebuilt the plan
  uint64_t Hc[kMaxLevels + 1];      // cumulative forecast mass, units of 2^-32
  uint64_t Fc[kMaxLevels + 1];      // cumulative F, units of 2^-32
  double D_Q_plan, l2;
  int32_t n_unforecast;
  int32_t pad;
};
cudaError_t launch_fc_plan(const int* hist, const RouteParams& p, DevPlan* plan, FcState* fcs, bool replan,
                           cudaStream_t st);
cudaError_t launch_fc_sample(const uint8_t* level, const RouteParams& p, DevPlan* plan, FcState* fcs,
                             int32_t* K_prime, uint8_t* cls7, cudaStream_t st);
cudaError_t launch_fc_window(const uint8_t* level, const RouteParams& p, DevPlan* plan, FcState* fcs,
                             uint8_t* ring, int window, cudaStream_t st);

// f2 LRU maintenance of the store (R25-R27)
struct LruSel {
  uint32_t prefix, mask;   // radix-select state: the threshold stamp T after 4 passes
  int32_t k;               // rank still needed inside the current prefix (after: r entries of stamp T)
  int32_t pad;
  int32_t hist[256];
};
int lru_tiles(int64_t M);
cudaError_t launch_lru_victims(const uint32_t* stamps, int64_t M, int32_t n_evict, LruSel* sel, int32_t* counts,
                               int32_t* scanned, int32_t* scan_tmp, int32_t* victims, cudaStream_t st);
cudaError_t launch_store_rows(const __nv_bfloat16* staged, const int32_t* src, int64_t n, int64_t n_append,
                              int64_t first_new, const int32_t* victims, int d, int G, int rank,
                              __nv_bfloat16* store, uint32_t* stamps, uint32_t tick, int32_t* gids_out,
                              int32_t* gids_by_prompt, cudaStream_t st);
cudaError_t launch_fill_u32(uint32_t* a, int64_t n, uint32_t v, cudaStream_t st);
cudaError_t launch_vanilla_compact(const int32_t* K_prime, const uint8_t* pflags, int64_t N, int32_t* counts,
                                   int32_t* scanned, int32_t* scan_tmp, int32_t* idx, int32_t* count,
                                   int32_t* gids_by_prompt, cudaStream_t st);

// K7 route-and-batch
struct BatchWs {
  int32_t* blk_counts;   // [C * batch_tiles(N)], class-major (C <= 64 classes)
  int32_t* blk_off;      // [C * batch_tiles(N)]
  int32_t* offsets;      // [W+1]
  int32_t* scan_tmp;     // scan_tmp_ints(64 * batch_tiles(N))
};
int batch_tiles(int64_t N);
cudaError_t batch_init();   // kernel attributes (once per device)
// f3: events since the last batch, the pick tables, per-instance counts and the state after the batch
cudaError_t launch_disp_prep(const RouteParams& p, int ntiles, int nC, const int32_t* scanned, cudaStream_t st);
cudaError_t launch_route_and_batch(const RedirectWs& r, const RouteParams& p, DevPlan* plan, const int* count_gate,
                                   const BatchWs& w, int32_t* instance, int32_t* slot,
                                   int32_t* bucket_offsets, int32_t* bucket_prompts,
                                   cudaStream_t st, int* launches);

// f4 controller: exact assignment solver by enumeration (R33-R36)
struct AssignParams {
  int nK, W, bstar;
  double lam;                      // prompts / s
  int grid[kMaxLevels];
  int64_t service_us[kMaxLevels];  // batch service time at b*
  double H[kMaxLevels];            // forecast H_K (ignored when fc != nullptr)
  double c[kTTotal];               // degradation c(dK)
  const FcState* fc;               // f1 predictor window: H_i = cnt_i / n (uniform when empty)
};
struct AssignOut {
  int32_t n[kMaxLevels];
  double F[kMaxLevels], F_route[kMaxLevels], H[kMaxLevels];
  double served, quality;
  int32_t instance_level[kMaxInst];
};
int64_t assign_count(int W, int nK);
size_t assign_key_bytes();
cudaError_t launch_assign(const AssignParams& p, void* block_best, int max_blocks, AssignOut* out, cudaStream_t st);

cudaError_t launch_fill_sentinel(Cand* out, int64_t n, cudaStream_t st);

// device-wide exclusive scan of n int32 (tmp: scan_tmp_ints(n) ints)
int scan_tmp_ints(int64_t n);
cudaError_t launch_exclusive_scan(const int32_t* in, int32_t* out, int n, int32_t* tmp, cudaStream_t st,
                                  int* launches);

}  // namespace pas
