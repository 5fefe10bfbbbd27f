// pas_api.cu -- the C-ABI of libpas (include/pas.h): context, validation, workspace, the batch
// pipeline K1..K7 on the caller's stream, the cache store, and the NCCL all-gather for world > 1.
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: a no-op unless a tool (nsys) injects itself

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "pas_internal.cuh"


using namespace pas;

// ----------------------------------------------------------------------------------------------
// NCCL, loaded lazily (only world > 1 needs it; torch's bundled libnccl.so.2 is reused if loaded)
// ----------------------------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
bool nccl_load() {
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.CommAbort = (decltype(g_nccl.CommAbort))dlsym(h, "ncclCommAbort");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather && g_nccl.AllReduce &&
              g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.CommDestroy &&
              g_nccl.CommAbort && g_nccl.GetErrorString;
  return g_nccl.ok;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

thread_local std::string g_global_err;


}  // namespace

// ----------------------------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------------------------
struct pas_ctx {
  pas_config cfg{};
  std::string err;
  bool poisoned = false;
  int launches = 0;
  // state
  bool bands_set = false, fractions_set = false;
  int nK = 0, W = 0, bstar = 1, mode = 0;
  int grid[kMaxLevels]{};
  float thr[kMaxLevels]{};
  double F[kMaxLevels]{};
  double c[kTTotal]{};
  bool c_convex = true;        // R6: NW-corner plan; false: the exact integer solver (R37)
  int64_t cI[kTTotal]{};       // R37: round-half-even(c * 2^24)
  int inst_level[kMaxInst]{};
  uint64_t seed = 0, batch_seq = 0;
  int64_t M_total = 0, M_local = 0, cap_rows = 0, q_rows = 0, cand_cap = 0;
  int64_t last_local_N = -1;
  int64_t last_N = 0;
  // device memory
  __nv_bfloat16* store = nullptr;
  __nv_bfloat16* qhat = nullptr;
  uint8_t* pflags = nullptr;
  Cand* cand_local = nullptr;
  Cand* cand_rank = nullptr;
  Cand* cand_all = nullptr;
  uint64_t* k2_progress = nullptr;   // K2 leash words [kNumSMs]
  // K2 dynamic schedule: parked top-k lists, per-(range, prompt tile) chunk counters, unit counter
  float* k2_st_s = nullptr;
  int32_t* k2_st_g = nullptr;
  uint64_t* k2_done = nullptr;
  uint32_t* k2_sched = nullptr;
  int64_t k2_state_tiles = 0;
  int k2_last_R = 0, k2_last_T = 0, k2_last_CS = 0;   // schedule of the last K2 launch (pas_plan_stats)
  K2Tuning k2_tune;                                    // experiment knobs, read at pas_create
  int small_max = kSmallMax;   // the one-CTA latency path serves N <= small_max (PAS_SMALL_MAX; 0: off)
  bool k6_force_fallback = false;   // PAS_K6_FALLBACK=1: K6's exact histogram path for every batch (tests)
  // f1 forecast-driven mode (0 = exact per-batch plan)
  int fc_window = 0, fc_replan_every = 1;
  int64_t fc_tick = 0;
  bool fc_planned = false;
  double fc_F_planned[kMaxLevels] = {};
  uint8_t* fc_ring = nullptr;
  FcState* fc_state = nullptr;
  bool fc_stats_valid = false;
  uint32_t k2_epoch = 0;
  // f3 stateful dispatcher (R28-R32); off = the stateless packing R13 / R14
  bool disp_on = false, disp_stats_valid = false;
  int disp_W = 0, disp_bstar_prev = 1, load_mode = PAS_UNIFORM;
  int64_t disp_now = 0, disp_last = 0, disp_timeout = 0;
  int64_t disp_svc[kMaxInst] = {};
  DispState* dstate = nullptr;
  DispPlan* dplan = nullptr;
  // f4 controller solver workspace
  void* asg_keys = nullptr;
  AssignOut* asg_out = nullptr;
  // f2 LRU maintenance: stamps of every global slot (replicated on all ranks) + insert workspace
  uint32_t* stamps = nullptr;
  uint32_t lru_tick = 0;
  LruSel* lru_sel = nullptr;
  int32_t *lru_counts = nullptr, *lru_scanned = nullptr, *lru_scan_tmp = nullptr, *lru_victims = nullptr;
  int32_t *ins_idx = nullptr, *ins_count = nullptr;
  uint8_t* level = nullptr;
  BatchCounters* bc = nullptr;       // device: Philox batch_seq, next LRU tick, K2 epoch (graph-replayable)
  int* hist = nullptr;
  int* invalid_count = nullptr;
  DevPlan* plan = nullptr;
  RedirectWs rw{};
  BatchWs bw{};
  // host-API staging
  void* stage_emb = nullptr;
  int32_t *s_K = nullptr, *s_Kp = nullptr, *s_inst = nullptr, *s_slot = nullptr, *s_tid = nullptr,
          *s_boff = nullptr, *s_bpr = nullptr;
  float* s_tsc = nullptr;
  uint8_t* s_flags = nullptr;
  // pipelined host API (pas_route_batch_host_async): two staging slots (input + every output), an H2D
  // and a D2H copy stream, per slot: input copied / batch routed / outputs copied
  struct HostSlot {
    void* emb = nullptr;
    int32_t *K = nullptr, *Kp = nullptr, *inst = nullptr, *slot = nullptr, *tid = nullptr, *boff = nullptr,
            *bpr = nullptr;
    float* tsc = nullptr;
    uint8_t* flags = nullptr;
    cudaEvent_t h2d = nullptr, done = nullptr, d2h = nullptr;
    bool used = false;
  } hs[2];
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t h_join = nullptr;
  int64_t hseq = 0;
  // tensor maps
  CUtensorMap tm_q{}, tm_c{}, tm_c2{};
  // comm
  ncclComm_t comm = nullptr;
  int coll_mode = PAS_COLL_FOLDED;   // explicit: slice merge + N2 all-reduce of H_K + N3 all-gather
  Cand* x_cand = nullptr;            // explicit mode: [G * Ns][k] gathered slice results (prompt order)
  int32_t* x_K = nullptr;
  uint8_t *x_level = nullptr, *x_flags = nullptr;
  // timing
  cudaEvent_t ev[8]{};
  nvtxRangeId_t nvtx_range = 0;   // the open NVTX range of the stage being enqueued (0: none)
  cudaEvent_t ev_aux = nullptr;   // end event of pas_solve_assignment's timing
  // stage-timing ring (pas_stage_ring): the 7 stage boundaries of each of the last ring_n batches
  std::vector<cudaEvent_t> ring;
  int ring_n = 0;
  int64_t ring_pos = 0, ring_count = 0;
  // CUDA-graph replay of pas_route_batch (pas_set_graph): the batch is captured once per (emb, dtype,
  // N, outputs) and replayed; any setter or cache change invalidates it
  bool graph_on = false, graph_valid = false, capturing = false, stages_valid = false;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;
  const void* g_emb = nullptr;
  int g_dtype = -1, g_launches = 0;
  int64_t g_N = -1;
  pas_route_out g_out{};
  bool ev_valid = false;
  cudaStream_t last_stream = nullptr;
};

namespace {

pas_status fail(pas_ctx* ctx, pas_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) {
    ctx->err = buf;
    if (st == PAS_ERR_CUDA || st == PAS_ERR_NCCL) ctx->poisoned = true;
  } else {
    g_global_err = buf;
  }
  return st;
}

#define CUDA_TRY(ctx, expr)                                                                         \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess) return fail((ctx), PAS_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

template <typename T>
cudaError_t dmalloc(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T) + 16);
}

bool encode_map(CUtensorMap* m, void* base, int64_t rows, int d, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t local_rows_below(int64_t total, int G, int rank) {
  return total > rank ? (total - rank + G - 1) / G : 0;
}

// NVTX range names of the stages between boundaries i and i + 1 (tracing row).
constexpr const char* kStageNvtx[6] = {"pas K1 normalise",      "pas K2 similarity + top-k",
                                       "pas K3/K4 merge + optimal-K", "pas K5 plan",
                                       "pas K6 redirect",       "pas K7 route-and-batch"};

// Record stage boundary i (0..6) of the current batch: ev[i], and its slot of the timing ring.  The
// host-side enqueue of each stage is also an NVTX range (process-wide start/end ranges, so a batch
// enqueued from several threads stays well-formed; a range left open by an error closes at the next
// boundary), which nsys correlates with the stage's kernels.
cudaError_t rec_stage(pas_ctx* ctx, int i, cudaStream_t st) {
  if (ctx->nvtx_range) nvtxRangeEnd(ctx->nvtx_range);
  ctx->nvtx_range = i < 6 ? nvtxRangeStartA(kStageNvtx[i]) : 0;
  if (ctx->capturing) return cudaSuccess;   // a replayed graph is timed as a whole (pas_route_batch)
  cudaError_t e = cudaEventRecord(ctx->ev[i], st);
  if (e == cudaSuccess && ctx->ring_n > 0) e = cudaEventRecord(ctx->ring[(ctx->ring_pos % ctx->ring_n) * 7 + i], st);
  return e;
}

pas_status check_live(pas_ctx* ctx) {
  if (!ctx) return fail(nullptr, PAS_ERR_ARG, "null context");
  if (ctx->poisoned) return fail(ctx, PAS_ERR_STATE, "context poisoned by an earlier CUDA/NCCL error: %s",
                                 ctx->err.c_str());
  return PAS_OK;
}

RouteParams make_params(const pas_ctx* ctx, int64_t N) {
  RouteParams p{};
  p.nK = ctx->nK;
  p.W = ctx->W;
  p.bstar = ctx->bstar;
  p.bstar_shift = -1;
  for (int b = 0; b < 31; ++b)
    if (ctx->bstar == (1 << b)) p.bstar_shift = b;
  p.mode = ctx->mode;
  p.topk = ctx->cfg.topk;
  p.G = ctx->cfg.world;
  p.rank = ctx->cfg.rank;
  p.d = ctx->cfg.d;
  p.N = N;
  p.M_total = ctx->M_total;
  p.seed = ctx->seed;
  p.batch_seq = ctx->batch_seq;
  p.kb = redirect_kb(N);   // K6 buckets per class: 2^kb
  for (int i = 0; i < kMaxLevels; ++i) {
    p.grid[i] = ctx->grid[i];
    p.thr[i] = i + 1 < ctx->nK ? ctx->thr[i] : INFINITY;   // +inf padding: level by binary search
    p.F[i] = ctx->F[i];
  }
  for (int t = 0; t < kTTotal; ++t) p.c[t] = ctx->c[t];
  p.convex = ctx->c_convex ? 1 : 0;
  p.k6_force_fallback = ctx->k6_force_fallback ? 1 : 0;
  for (int t = 0; t < kTTotal; ++t) p.cI[t] = ctx->cI[t];
  for (int w = 0; w < kMaxInst; ++w) p.inst_level[w] = ctx->inst_level[w];
  p.lru_stamp = ctx->stamps;
  p.lru_tick = ctx->lru_tick;
  p.bc = ctx->bc;
  p.disp = ctx->disp_on ? 1 : 0;
  p.bstar_prev = ctx->disp_bstar_prev;
  p.now_us = ctx->disp_now;
  p.timeout_us = ctx->disp_timeout;
  p.dstate = ctx->dstate;
  p.dplan = ctx->dplan;
  return p;
}

pas_status validate_out(pas_ctx* ctx, const pas_route_out* out, bool device = true) {
  if (!out) return fail(ctx, PAS_ERR_ARG, "out is NULL");
  if (!out->K || !out->K_prime || !out->instance || !out->slot)
    return fail(ctx, PAS_ERR_ARG, "out->K, K_prime, instance and slot are required");
  if (device) {
    const void* ptrs[] = {out->K, out->K_prime, out->instance, out->slot, out->topk_id, out->topk_score,
                          out->flags, out->bucket_offsets, out->bucket_prompts};
    for (const void* q : ptrs)
      if (reinterpret_cast<uintptr_t>(q) & 15)
        return fail(ctx, PAS_ERR_ARG, "output arrays must be 16-byte aligned (vectorised stores)");
  }
  return PAS_OK;
}

// K1 reads rows with 128-bit (fp32) / 64-bit (bf16) vector loads: the base must be aligned to that
// (d is a multiple of 64, so every row then is).
pas_status validate_rows(pas_ctx* ctx, const void* rows, pas_dtype dt) {
  if (dt != PAS_F32 && dt != PAS_BF16) return fail(ctx, PAS_ERR_ARG, "dtype must be PAS_F32 or PAS_BF16");
  const uintptr_t a = reinterpret_cast<uintptr_t>(rows);
  if (a & (dt == PAS_F32 ? 15 : 7))
    return fail(ctx, PAS_ERR_ARG, "embedding rows must be %d-byte aligned (vector loads)", dt == PAS_F32 ? 16 : 8);
  return PAS_OK;
}

pas_status ready(pas_ctx* ctx, int64_t N) {
  if (!ctx->bands_set || !ctx->fractions_set)
    return fail(ctx, PAS_ERR_STATE, "pas_set_bands and pas_set_fractions must be called before routing");
  if (N < 0) return fail(ctx, PAS_ERR_ARG, "N < 0");
  if (N > ctx->cfg.max_batch)
    return fail(ctx, PAS_ERR_CAPACITY, "N = %lld exceeds max_batch = %lld", (long long)N,
                (long long)ctx->cfg.max_batch);
  return PAS_OK;
}

// K2 candidate and parked-list capacities for a context of max_batch prompts (pas_create).
int64_t k2_cand_cap(int64_t max_batch) {
  const int64_t qt = simtopk_prompt_rows();
  return 4 * max_batch > 592 * qt ? 4 * max_batch : 592 * qt;
}
int64_t k2_state_tiles(int64_t cand_cap) { return cand_cap / simtopk_box_q() + 8; }

// The K2 schedule of one batch: the dynamic schedule when simtopk_plan_dynamic takes it (dyn.T > 0),
// else the static ranges.  Returns R (the S of the merge).  Host only.
int k2_schedule(int64_t N, int64_t M_local, int d, int64_t cand_cap, const K2Tuning& tune, DynSched* dyn) {
  int R = 1;
  if (!tune.force_static &&
      simtopk_plan_dynamic(N, M_local, cand_cap, k2_state_tiles(cand_cap), d, tune, &R, &dyn->T, &dyn->CS, &dyn->MTg)) {
    return R;
  }
  dyn->T = dyn->CS = dyn->MTg = 0;
  R = simtopk_choose_ranges(N, M_local, cand_cap, d);
  if (tune.ranges >= 1 && (int64_t)tune.ranges * N <= cand_cap) R = tune.ranges;
  return R;
}

// Prompt-side workspace (Q_hat, validity flags, K2 candidates, NCCL buffers), allocated on the first
// call that runs a1 + a3, so a context used only through pas_route_from_candidates never holds it.
pas_status ensure_prompt_ws(pas_ctx* ctx) {
  if (ctx->qhat) return PAS_OK;
  const int64_t mb = ctx->cfg.max_batch, k = ctx->cfg.topk, d = ctx->cfg.d;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = dmalloc(&ctx->qhat, (size_t)(ctx->q_rows * d));
  if (e == cudaSuccess) e = dmalloc(&ctx->pflags, (size_t)mb);
  if (e == cudaSuccess) e = dmalloc(&ctx->k2_progress, (size_t)kNumSMs);
  if (e == cudaSuccess) e = cudaMemset(ctx->k2_progress, 0, sizeof(uint64_t) * kNumSMs);   // epoch 0 = none
  // parked lists of the K2 dynamic schedule: one slot per (range, prompt tile), R * MT <= cand_cap / 128 + 8
  ctx->k2_state_tiles = k2_state_tiles(ctx->cand_cap);
  const size_t st_elems = (size_t)ctx->k2_state_tiles * simtopk_box_q() * 2 * (k <= 8 ? 8 : 16);
  if (e == cudaSuccess) e = dmalloc(&ctx->k2_st_s, st_elems);
  if (e == cudaSuccess) e = dmalloc(&ctx->k2_st_g, st_elems);
  if (e == cudaSuccess) e = dmalloc(&ctx->k2_done, (size_t)ctx->k2_state_tiles);
  if (e == cudaSuccess) e = cudaMemset(ctx->k2_done, 0, sizeof(uint64_t) * (size_t)ctx->k2_state_tiles);
  if (e == cudaSuccess) e = dmalloc(&ctx->k2_sched, (size_t)2);
  if (e == cudaSuccess) e = cudaMemset(ctx->k2_sched, 0, sizeof(uint32_t) * 2);
  if (e == cudaSuccess) e = dmalloc(&ctx->cand_local, (size_t)(ctx->cand_cap * k));
  if (e == cudaSuccess) e = dmalloc(&ctx->cand_rank, (size_t)(mb * k));
  if (e == cudaSuccess && (ctx->cfg.world > 1 || ctx->comm))
    e = dmalloc(&ctx->cand_all, (size_t)((int64_t)ctx->cfg.world * mb * k));
  if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "prompt workspace allocation failed: %s", cudaGetErrorString(e));
  if (!encode_map(&ctx->tm_q, ctx->qhat, ctx->q_rows, (int)d, simtopk_box_q()))
    return fail(ctx, PAS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the prompt map");
  return PAS_OK;
}

// a1 + a3 (+ the intra-GPU part of a4 into `merged` if non-null).  Returns the candidate layout.
pas_status run_local(pas_ctx* ctx, const void* emb, pas_dtype dt, int64_t N, cudaStream_t st, const Cand** cand,
                     int* S, Cand* merged) {
  const int k = ctx->cfg.topk;
  if (pas_status s = ensure_prompt_ws(ctx)) return s;
  const int64_t dup = simtopk_dup_rows(N, (int)ctx->cfg.d);
  CUDA_TRY(ctx, launch_normalize(emb, dt, N, ctx->cfg.d, ctx->qhat, ctx->pflags, 0, 1, 0, nullptr, st,
                                 &ctx->bc->k2_epoch, dup));
  ctx->launches++;
  CUDA_TRY(ctx, rec_stage(ctx, 1, st));
  int R = 1;
  if (ctx->M_local > 0) {
    DynSched dyn;
    R = k2_schedule(N, ctx->M_local, ctx->cfg.d, ctx->cand_cap, ctx->k2_tune, &dyn);
    if (dyn.T > 0) {
      dyn.st_s = ctx->k2_st_s;
      dyn.st_g = ctx->k2_st_g;
      dyn.done = ctx->k2_done;
      dyn.slots = (int)ctx->k2_state_tiles;
      dyn.sched = ctx->k2_sched;
    }
    SimTopkArgs a{&ctx->tm_q, &ctx->tm_c, &ctx->tm_c2, N, ctx->M_local, ctx->cfg.d, k, ctx->cfg.world, ctx->cfg.rank, R,
                  ctx->qhat, ctx->cand_local, nullptr, ctx->k2_tune.no_leash ? nullptr : ctx->k2_progress,
                  0, &ctx->bc->k2_epoch, dyn};
    a.dup = dup > 0;
    CUDA_TRY(ctx, launch_simtopk(a, st));
    ctx->k2_last_R = R;
    ctx->k2_last_T = dyn.T;
    ctx->k2_last_CS = dyn.CS;
  } else {
    ctx->k2_last_R = 1;
    ctx->k2_last_T = ctx->k2_last_CS = 0;
    CUDA_TRY(ctx, launch_fill_sentinel(ctx->cand_local, N * k, st));
  }
  ctx->launches++;
  CUDA_TRY(ctx, rec_stage(ctx, 2, st));
  *cand = ctx->cand_local;
  *S = R;
  if (merged) {
    CUDA_TRY(ctx, launch_merge(ctx->cand_local, R, N, k, merged, st));
    ctx->launches++;
    *cand = merged;
    *S = 1;
  }
  ctx->last_local_N = N;
  return PAS_OK;
}

pas_status run_downstream(pas_ctx* ctx, RouteParams& p, int64_t N, const pas_route_out* out, cudaStream_t st);
pas_status finish_batch(pas_ctx* ctx, int64_t N, cudaStream_t st);

// a4 (final merge) .. a8 for all N prompts from S candidate blocks [S][N][k].
pas_status run_global(pas_ctx* ctx, const Cand* cand, int S, int64_t N, const pas_route_out* out, cudaStream_t st) {
  ctx->lru_tick++;   // f2 clock: one tick per routed batch (R26)
  RouteParams p = make_params(ctx, N);
  SelectOut so{out->K, out->topk_id, out->topk_score, out->flags, ctx->level, nullptr, ctx->hist, ctx->plan};
  // the validity flags of the pas_route_local / run_local that produced these candidates; consumed
  // here, so a later pas_route_from_candidates with the same N never reuses them (else: all valid)
  const uint8_t* pflags = ctx->last_local_N == N ? ctx->pflags : nullptr;
  ctx->last_local_N = -1;
  if (N <= ctx->small_max && S <= 128 && ctx->fc_window == 0 && !ctx->disp_on) {
    // the latency path: merge .. route-and-batch in one CTA (k_small.cu), no DevPlan zeroing launch
    SmallOut sm{out->K, out->K_prime, out->instance, out->slot, out->topk_id, out->topk_score, out->flags,
                out->bucket_offsets, out->bucket_prompts, ctx->level, ctx->plan};
    CUDA_TRY(ctx, launch_small_route(cand, S, pflags, p, sm, st));
    ctx->launches++;
    CUDA_TRY(ctx, rec_stage(ctx, 3, st));
    CUDA_TRY(ctx, rec_stage(ctx, 4, st));
    CUDA_TRY(ctx, rec_stage(ctx, 5, st));
    ctx->fc_stats_valid = false;
    return finish_batch(ctx, N, st);
  }
  static_assert(sizeof(DevPlan) % 4 == 0, "DevPlan zeroed as int32 words");
  CUDA_TRY(ctx, launch_zero(ctx->hist, kMaxLevels, reinterpret_cast<int32_t*>(ctx->plan), sizeof(DevPlan) / 4,
                            nullptr, 0, st));
  ctx->launches++;
  CUDA_TRY(ctx, launch_merge_select(cand, S, pflags, p, so, st));
  ctx->launches++;
  CUDA_TRY(ctx, rec_stage(ctx, 3, st));
  return run_downstream(ctx, p, N, out, st);
}

// The explicit form of SURVEY 8(e) (pas_set_collectives(PAS_COLL_EXPLICIT)): from the all-gathered
// [G][N][k] candidates each rank merges only its prompt slice [r Ns, r Ns + n_r) (Ns = ceil(N / G)),
// N2 all-reduces the slice H_K (and the flag counters) -- "an all-reduce of H_K precedes the route
// plan" (north_star) -- and N3 all-gathers the slice results (top-k, K, level, flags; one NCCL group),
// which every rank unpacks (stamping the top-1s, R26) before the redundant, deterministic K5..K7.
pas_status run_global_explicit(pas_ctx* ctx, const Cand* cand_all, int64_t N, const pas_route_out* out,
                               cudaStream_t st) {
  const int G = ctx->cfg.world, r = ctx->cfg.rank, k = ctx->cfg.topk;
  const int64_t Ns = (N + G - 1) / G, lo = (int64_t)r * Ns;
  const int64_t n_r = N - lo < 0 ? 0 : (N - lo < Ns ? N - lo : Ns);
  if (!ctx->x_cand) {
    const int64_t cap = ((ctx->cfg.max_batch + G - 1) / G) * G;
    cudaError_t e = dmalloc(&ctx->x_cand, (size_t)(cap * k));
    if (e == cudaSuccess) e = dmalloc(&ctx->x_K, (size_t)cap);
    if (e == cudaSuccess) e = dmalloc(&ctx->x_level, (size_t)cap);
    if (e == cudaSuccess) e = dmalloc(&ctx->x_flags, (size_t)cap);
    if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "explicit-collective workspace: %s", cudaGetErrorString(e));
  }
  ctx->lru_tick++;   // f2 clock (R26)
  RouteParams p = make_params(ctx, N);
  CUDA_TRY(ctx, launch_zero(ctx->hist, kMaxLevels, reinterpret_cast<int32_t*>(ctx->plan), sizeof(DevPlan) / 4,
                            nullptr, 0, st));
  ctx->launches++;
  const uint8_t* pflags = ctx->last_local_N == N ? ctx->pflags : nullptr;
  ctx->last_local_N = -1;
  if (n_r > 0) {   // slice merge + select straight into this rank's segment of the gather buffers
    RouteParams ps = p;
    ps.N = n_r;
    ps.cand_stride = N;
    ps.lru_stamp = nullptr;   // stamped for all N after the gather
    SelectOut so{ctx->x_K + lo, nullptr, nullptr, ctx->x_flags + lo, ctx->x_level + lo, ctx->x_cand + lo * k,
                 ctx->hist, ctx->plan};
    CUDA_TRY(ctx, launch_merge_select(cand_all + lo * k, G, pflags ? pflags + lo : nullptr, ps, so, st));
    ctx->launches++;
  }
  ncclResult_t nr = g_nccl.GroupStart();
  if (nr == ncclSuccess)   // N2: H_K and the three flag counters (contiguous in DevPlan)
    nr = g_nccl.AllReduce(ctx->hist, ctx->hist, (size_t)ctx->nK, ncclInt32, ncclSum, ctx->comm, st);
  if (nr == ncclSuccess)
    nr = g_nccl.AllReduce(&ctx->plan->n_invalid, &ctx->plan->n_invalid, 3, ncclInt32, ncclSum, ctx->comm, st);
  // N3 (in place: rank r's segment already sits at r * Ns)
  if (nr == ncclSuccess)
    nr = g_nccl.AllGather(ctx->x_cand + lo * k, ctx->x_cand, (size_t)Ns * k * 2, ncclInt32, ctx->comm, st);
  if (nr == ncclSuccess) nr = g_nccl.AllGather(ctx->x_K + lo, ctx->x_K, (size_t)Ns, ncclInt32, ctx->comm, st);
  if (nr == ncclSuccess) nr = g_nccl.AllGather(ctx->x_level + lo, ctx->x_level, (size_t)Ns, ncclUint8, ctx->comm, st);
  if (nr == ncclSuccess) nr = g_nccl.AllGather(ctx->x_flags + lo, ctx->x_flags, (size_t)Ns, ncclUint8, ctx->comm, st);
  const ncclResult_t ne = g_nccl.GroupEnd();
  if (nr != ncclSuccess || ne != ncclSuccess)
    return fail(ctx, PAS_ERR_NCCL, "explicit collectives: %s", g_nccl.GetErrorString(nr != ncclSuccess ? nr : ne));
  SelectOut so{out->K, out->topk_id, out->topk_score, out->flags, ctx->level, nullptr, ctx->hist, ctx->plan};
  CUDA_TRY(ctx, launch_unpack_slices(ctx->x_cand, ctx->x_K, ctx->x_level, ctx->x_flags, p, so, st));
  ctx->launches++;
  CUDA_TRY(ctx, rec_stage(ctx, 3, st));
  return run_downstream(ctx, p, N, out, st);
}

// a6 .. a8 (plan, redirection, route-and-batch) after the merge stage has written level / hist / plan.
pas_status run_downstream(pas_ctx* ctx, RouteParams& p, int64_t N, const pas_route_out* out, cudaStream_t st) {
  bool counts_ready = false;
  if (ctx->fc_window > 0) {
    // f1: plan from the forecast (held between rebuilds, R24), i.i.d. K' (R23), window update (R21)
    bool replan = !ctx->fc_planned || ctx->fc_tick % ctx->fc_replan_every == 0;
    for (int j = 0; j < ctx->nK; ++j) replan = replan || ctx->F[j] != ctx->fc_F_planned[j];
    if (replan) {
      for (int j = 0; j < kMaxLevels; ++j) ctx->fc_F_planned[j] = ctx->F[j];
      ctx->fc_planned = true;
    }
    ctx->fc_tick++;
    CUDA_TRY(ctx, launch_fc_plan(ctx->hist, p, ctx->plan, ctx->fc_state, replan, st));
    CUDA_TRY(ctx, rec_stage(ctx, 4, st));
    CUDA_TRY(ctx, launch_fc_sample(ctx->level, p, ctx->plan, ctx->fc_state, out->K_prime, ctx->rw.cls7, st));
    CUDA_TRY(ctx, launch_fc_window(ctx->level, p, ctx->plan, ctx->fc_state, ctx->fc_ring, ctx->fc_window, st));
    ctx->launches += 3;
    ctx->fc_stats_valid = true;
  } else {
    CUDA_TRY(ctx, launch_plan(ctx->hist, p, ctx->plan, st));
    ctx->launches++;
    CUDA_TRY(ctx, rec_stage(ctx, 4, st));
    CUDA_TRY(ctx, launch_redirect(ctx->level, p, ctx->plan, ctx->rw, out->K_prime, ctx->bw.blk_counts,
                                  batch_tiles(N), p.mode == PAS_UNIFORM ? p.W : p.nK, st, &ctx->launches,
                                  &counts_ready));
    ctx->fc_stats_valid = false;
  }
  CUDA_TRY(ctx, rec_stage(ctx, 5, st));
  // K6's windowed pass wrote K7's tile counts (k_cls_count then only on its fallback)
  CUDA_TRY(ctx, launch_route_and_batch(ctx->rw, p, ctx->plan, counts_ready ? &ctx->plan->k6_fallback : nullptr,
                                       ctx->bw, out->instance, out->slot, out->bucket_offsets, out->bucket_prompts, st,
                                       &ctx->launches));
  return finish_batch(ctx, N, st);
}

// The batch's last stage boundary and the host-side bookkeeping of a routed batch.
pas_status finish_batch(pas_ctx* ctx, int64_t N, cudaStream_t st) {
  CUDA_TRY(ctx, rec_stage(ctx, 6, st));
  ctx->ev_valid = true;
  ctx->stages_valid = !ctx->capturing;
  ctx->last_stream = st;
  ctx->last_N = N;
  ctx->batch_seq++;
  if (ctx->ring_n > 0 && !ctx->capturing) {   // a capture records no stage events
    ctx->ring_pos++;
    ctx->ring_count = ctx->ring_count < ctx->ring_n ? ctx->ring_count + 1 : ctx->ring_n;
  }
  ctx->disp_stats_valid = ctx->disp_on;
  if (ctx->disp_on) {   // R28: the events until the next batch follow this batch's policy
    ctx->disp_bstar_prev = ctx->bstar;
    ctx->disp_last = ctx->disp_now;
  }
  return PAS_OK;
}

}  // namespace

// ----------------------------------------------------------------------------------------------
// C-ABI
// ----------------------------------------------------------------------------------------------
extern "C" {

const char* pas_version(void) {
  return "libpas 0.6 (sm_100a; K2 tcgen05 cta_group::1 128x256 on a dynamic chunked schedule, cta_group::2 256x256 for even tile counts <= 4, 128x128 for one prompt tile vs small caches)";
}

const char* pas_last_error(const pas_ctx* ctx) { return ctx ? ctx->err.c_str() : g_global_err.c_str(); }

int pas_last_launch_count(const pas_ctx* ctx) { return ctx ? ctx->launches : 0; }

pas_status pas_nccl_unique_id(unsigned char* out) {
  if (!out) return fail(nullptr, PAS_ERR_ARG, "out is NULL");
  if (!nccl_load()) return fail(nullptr, PAS_ERR_NCCL, "cannot load libnccl.so.2");
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, PAS_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  memcpy(out, id.internal, PAS_NCCL_ID_BYTES);
  return PAS_OK;
}

pas_status pas_destroy(pas_ctx* ctx) {
  if (!ctx) return PAS_OK;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  if (ctx->comm) {
    if (ctx->poisoned) g_nccl.CommAbort(ctx->comm);
    else g_nccl.CommDestroy(ctx->comm);
  }
  void* ptrs[] = {ctx->store,   ctx->qhat,      ctx->pflags,     ctx->cand_local,   ctx->cand_rank, ctx->cand_all, ctx->k2_progress, ctx->fc_ring, ctx->fc_state,
                  ctx->k2_st_s, ctx->k2_st_g, ctx->k2_done, ctx->k2_sched,
                  ctx->dstate, ctx->dplan, ctx->asg_keys, ctx->asg_out,
                  ctx->stamps, ctx->lru_sel, ctx->lru_counts, ctx->lru_scanned, ctx->lru_scan_tmp, ctx->lru_victims,
                  ctx->ins_idx, ctx->ins_count,
                  ctx->level,   ctx->bc, ctx->hist,      ctx->invalid_count, ctx->plan,      ctx->rw.key,    ctx->rw.hist,
                  ctx->rw.used, ctx->rw.csum, ctx->rw.bnd, ctx->rw.lists,  ctx->rw.cand,    ctx->rw.cls7,
                  ctx->bw.blk_counts, ctx->bw.blk_off, ctx->bw.offsets, ctx->bw.scan_tmp,
                  ctx->stage_emb, ctx->s_K, ctx->s_Kp,
                  ctx->s_inst,  ctx->s_slot,    ctx->s_tid,      ctx->s_boff,       ctx->s_bpr,     ctx->s_tsc,
                  ctx->s_flags, ctx->x_cand, ctx->x_K, ctx->x_level, ctx->x_flags};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& h : ctx->hs) {
    void* hp[] = {h.emb, h.K, h.Kp, h.inst, h.slot, h.tid, h.boff, h.bpr, h.tsc, h.flags};
    for (void* p : hp)
      if (p) cudaFree(p);
    for (cudaEvent_t e : {h.h2d, h.done, h.d2h})
      if (e) cudaEventDestroy(e);
  }
  if (ctx->h_join) cudaEventDestroy(ctx->h_join);
  if (ctx->h2d_stream) cudaStreamDestroy(ctx->h2d_stream);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_aux) cudaEventDestroy(ctx->ev_aux);
  for (auto e : ctx->ring) cudaEventDestroy(e);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  delete ctx;
  return PAS_OK;
}

pas_status pas_create(pas_ctx** out_ctx, const pas_config* cfg) {
  if (!out_ctx || !cfg) return fail(nullptr, PAS_ERR_ARG, "null argument");
  *out_ctx = nullptr;
  if (cfg->d < 64 || cfg->d > 4096 || cfg->d % 64)
    return fail(nullptr, PAS_ERR_ARG, "d = %d must be a multiple of 64 in [64, 4096]", cfg->d);
  if (cfg->topk < 1 || cfg->topk > PAS_MAX_TOPK)
    return fail(nullptr, PAS_ERR_ARG, "topk = %d outside [1, %d]", cfg->topk, PAS_MAX_TOPK);
  if (cfg->max_batch < 1 || cfg->max_batch > (1LL << 26))
    return fail(nullptr, PAS_ERR_ARG, "max_batch outside [1, 2^26]");
  if (cfg->max_rows_per_rank < 0 || cfg->max_rows_per_rank > (1LL << 31) / 2)
    return fail(nullptr, PAS_ERR_ARG, "max_rows_per_rank outside [0, 2^30]");
  if (cfg->world < 1 || cfg->world > 128 || cfg->rank < 0 || cfg->rank >= cfg->world)
    return fail(nullptr, PAS_ERR_ARG, "rank/world invalid (1 <= world <= 128, 0 <= rank < world)");
  if ((int64_t)cfg->max_rows_per_rank * cfg->world >= (1LL << 31))
    return fail(nullptr, PAS_ERR_ARG, "global ids must fit int32 (max_rows_per_rank * world < 2^31)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
    return fail(nullptr, PAS_ERR_ARG, "CUDA device %d not available", cfg->device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10 || prop.minor != 0)
    return fail(nullptr, PAS_ERR_ARG, "libpas needs an sm_100 device (B200); device %d is sm_%d%d", cfg->device,
                prop.major, prop.minor);
  if (cudaSetDevice(cfg->device) != cudaSuccess) return fail(nullptr, PAS_ERR_CUDA, "cudaSetDevice failed");

  pas_ctx* ctx = new pas_ctx();
  ctx->cfg = *cfg;
  ctx->cfg.nccl_id = nullptr;
  ctx->seed = cfg->seed;
  for (int t = 0; t < kTTotal; ++t) ctx->c[t] = 0.006 * t;   // SPEC S:49 default, R6
  const int64_t mb = cfg->max_batch, d = cfg->d;
  const int64_t qt = simtopk_prompt_rows();
  ctx->q_rows = (mb + qt - 1) / qt * qt;
  ctx->cap_rows = cfg->max_rows_per_rank;
  // K2 writes [R][N][k] with R * N <= cand_cap (simtopk_choose_ranges)
  ctx->cand_cap = k2_cand_cap(mb);
  ctx->k2_tune = K2Tuning::from_env();
  ctx->k6_force_fallback = getenv("PAS_K6_FALLBACK") && atoi(getenv("PAS_K6_FALLBACK")) != 0;   // tests
  if (const char* v = getenv("PAS_SMALL_MAX")) {   // A/B and tests: force the multi-kernel chain
    const int m = atoi(v);
    ctx->small_max = m < 0 ? 0 : (m > kSmallMax ? kSmallMax : m);
  }
  const int64_t nb = (int64_t)kMaxLevels << redirect_kb(mb);
  const int64_t ncls = 64 * (int64_t)batch_tiles(mb);
  cudaError_t e = cudaSuccess;
#define ALLOC(ptr, n) \
  if (e == cudaSuccess) e = dmalloc(&(ptr), (size_t)(n))
  ALLOC(ctx->store, (ctx->cap_rows > 0 ? ctx->cap_rows : 1) * d);
  ALLOC(ctx->stamps, (int64_t)cfg->world * (ctx->cap_rows > 0 ? ctx->cap_rows : 1));
  if (e == cudaSuccess)
    e = cudaMemset(ctx->stamps, 0, sizeof(uint32_t) * (size_t)cfg->world * (ctx->cap_rows > 0 ? ctx->cap_rows : 1));
  ALLOC(ctx->level, mb);
  ALLOC(ctx->bc, 1);
  ALLOC(ctx->hist, kMaxLevels);
  ALLOC(ctx->invalid_count, 1);
  ALLOC(ctx->plan, 1);
  ALLOC(ctx->rw.key, mb);
  ALLOC(ctx->rw.hist, nb);
  ALLOC(ctx->rw.used, 2);
  ALLOC(ctx->rw.csum, kMaxLevels * 256);
  ALLOC(ctx->rw.bnd, 1);
  ALLOC(ctx->rw.lists, kMaxLevels * kMaxLevels);
  ALLOC(ctx->rw.cand, mb);
  ALLOC(ctx->rw.cls7, mb);
  ALLOC(ctx->bw.blk_counts, ncls);
  ALLOC(ctx->bw.blk_off, ncls);
  ALLOC(ctx->bw.offsets, kMaxInst + 1);
  ALLOC(ctx->bw.scan_tmp, scan_tmp_ints(ncls));
#undef ALLOC
  if (e != cudaSuccess) {
    pas_destroy(ctx);
    return fail(nullptr, PAS_ERR_CUDA, "device allocation failed: %s", cudaGetErrorString(e));
  }
  for (auto& ev : ctx->ev)
    if (cudaEventCreate(&ev) != cudaSuccess) {
      pas_destroy(ctx);
      return fail(nullptr, PAS_ERR_CUDA, "cudaEventCreate failed");
    }
  if (cudaEventCreate(&ctx->ev_aux) != cudaSuccess) {
    pas_destroy(ctx);
    return fail(nullptr, PAS_ERR_CUDA, "cudaEventCreate failed");
  }
  {
    const BatchCounters b0{0, 1, 0};   // batch 0, next LRU tick 1 (host tick 0), K2 epoch 0 = none yet
    if (cudaMemcpy(ctx->bc, &b0, sizeof b0, cudaMemcpyHostToDevice) != cudaSuccess) {
      pas_destroy(ctx);
      return fail(nullptr, PAS_ERR_CUDA, "batch counter initialisation failed");
    }
  }
  if (!encode_map(&ctx->tm_c, ctx->store, ctx->cap_rows > 0 ? ctx->cap_rows : 1, (int)d, simtopk_box_c((int)d)) ||
      !encode_map(&ctx->tm_c2, ctx->store, ctx->cap_rows > 0 ? ctx->cap_rows : 1, (int)d, simtopk_box_c_pair())) {
    pas_destroy(ctx);
    return fail(nullptr, PAS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable or failed");
  }
  if ((e = simtopk_init()) != cudaSuccess || (e = batch_init()) != cudaSuccess) {
    pas_destroy(ctx);
    return fail(nullptr, PAS_ERR_CUDA, "kernel attribute setup failed: %s", cudaGetErrorString(e));
  }
  if (cfg->nccl_id) {   // world == 1 with an id: a 1-rank communicator (exercises the collective path)
    if (!nccl_load()) {
      pas_destroy(ctx);
      return fail(nullptr, PAS_ERR_NCCL, "cannot load libnccl.so.2");
    }
    ncclUniqueId id;
    memcpy(id.internal, cfg->nccl_id, PAS_NCCL_ID_BYTES);
    ncclResult_t r = g_nccl.CommInitRank(&ctx->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      pas_destroy(ctx);
      return fail(nullptr, PAS_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    }
  }
  *out_ctx = ctx;
  return PAS_OK;
}

pas_status pas_cache_clear(pas_ctx* ctx) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  ctx->M_total = 0;
  ctx->M_local = 0;
  return PAS_OK;
}

pas_status pas_cache_size(const pas_ctx* ctx, int64_t* global_rows, int64_t* local_rows) {
  if (!ctx) return PAS_ERR_ARG;
  if (global_rows) *global_rows = ctx->M_total;
  if (local_rows) *local_rows = ctx->M_local;
  return PAS_OK;
}

pas_status pas_cache_load(pas_ctx* ctx, const void* rows, pas_dtype dtype, int64_t M, int64_t* first_gid,
                          pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (M < 0 || (M > 0 && !rows)) return fail(ctx, PAS_ERR_ARG, "bad rows / M");
  if ((s = validate_rows(ctx, rows, dtype))) return s;
  const int G = ctx->cfg.world, rank = ctx->cfg.rank;
  const int64_t new_total = ctx->M_total + M;
  if (new_total >= (1LL << 31)) return fail(ctx, PAS_ERR_CAPACITY, "global ids must stay below 2^31");
  const int64_t new_local = local_rows_below(new_total, G, rank);
  if (new_local > ctx->cap_rows)
    return fail(ctx, PAS_ERR_CAPACITY, "shard capacity %lld rows exceeded (need %lld)", (long long)ctx->cap_rows,
                (long long)new_local);
  if (first_gid) *first_gid = ctx->M_total;
  if (M == 0) return PAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->invalid_count, 0, sizeof(int), st));
  // rows are written at local row (first_gid + i) / G of the store
  CUDA_TRY(ctx, launch_normalize(rows, dtype, M, ctx->cfg.d, ctx->store, nullptr, ctx->M_total, G, rank,
                                 ctx->invalid_count, st));
  int bad = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&bad, ctx->invalid_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (bad) return fail(ctx, PAS_ERR_INVALID_ROWS, "%d of the rows are non-finite or have zero norm", bad);
  ctx->lru_tick++;
  CUDA_TRY(ctx, launch_fill_u32(ctx->stamps + ctx->M_total, M, ctx->lru_tick, st));
  CUDA_TRY(ctx, launch_fill_u32(&ctx->bc->lru_tick, 1, ctx->lru_tick + 1, st));   // the next batch's tick
  ctx->M_total = new_total;
  ctx->M_local = new_local;
  return PAS_OK;
}

namespace {

pas_status ensure_lru_ws(pas_ctx* ctx) {
  if (ctx->lru_sel) return PAS_OK;
  const int64_t cap = (int64_t)ctx->cfg.world * ctx->cap_rows;
  const int64_t span = cap > ctx->cfg.max_batch ? cap : ctx->cfg.max_batch;
  const int64_t tiles = 2 * (int64_t)lru_tiles(span);
  cudaError_t e = dmalloc(&ctx->lru_sel, 1);
  if (e == cudaSuccess) e = dmalloc(&ctx->lru_counts, (size_t)tiles);
  if (e == cudaSuccess) e = dmalloc(&ctx->lru_scanned, (size_t)tiles);
  if (e == cudaSuccess) e = dmalloc(&ctx->lru_scan_tmp, (size_t)scan_tmp_ints(tiles));
  if (e == cudaSuccess) e = dmalloc(&ctx->lru_victims, (size_t)ctx->cfg.max_batch);
  if (e == cudaSuccess) e = dmalloc(&ctx->ins_idx, (size_t)ctx->cfg.max_batch);
  if (e == cudaSuccess) e = dmalloc(&ctx->ins_count, 1);
  if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "LRU workspace allocation failed: %s", cudaGetErrorString(e));
  return PAS_OK;
}

// Rows already normalised in ctx->qhat (staged); src = staged row of insert i (nullptr: i).  R26/R27:
// append at the free end first, then take the n_evict LRU slots in ascending gid order.
pas_status insert_staged(pas_ctx* ctx, const int32_t* src, int64_t n, int32_t* gids_out, int32_t* gids_by_prompt,
                         cudaStream_t st) {
  const int G = ctx->cfg.world, rank = ctx->cfg.rank;
  const int64_t cap = (int64_t)G * ctx->cap_rows;
  if (n > cap) return fail(ctx, PAS_ERR_CAPACITY, "%lld rows exceed the store capacity %lld", (long long)n,
                           (long long)cap);
  ctx->lru_tick++;
  const int64_t n_append = n < cap - ctx->M_total ? n : cap - ctx->M_total;
  const int64_t n_evict = n - n_append;
  if (n_evict > 0)
    CUDA_TRY(ctx, launch_lru_victims(ctx->stamps, ctx->M_total, (int32_t)n_evict, ctx->lru_sel, ctx->lru_counts,
                                     ctx->lru_scanned, ctx->lru_scan_tmp, ctx->lru_victims, st));
  CUDA_TRY(ctx, launch_store_rows(ctx->qhat, src, n, n_append, ctx->M_total, ctx->lru_victims, ctx->cfg.d, G, rank,
                                  ctx->store, ctx->stamps, ctx->lru_tick, gids_out, gids_by_prompt, st));
  CUDA_TRY(ctx, launch_fill_u32(&ctx->bc->lru_tick, 1, ctx->lru_tick + 1, st));   // the next batch's tick
  ctx->M_total += n_append;
  ctx->M_local = local_rows_below(ctx->M_total, G, rank);
  ctx->last_local_N = -1;   // the staging buffers no longer hold the last routed batch
  return PAS_OK;
}

}  // namespace

pas_status pas_cache_insert(pas_ctx* ctx, const void* rows, pas_dtype dtype, int64_t n, int32_t* gids_out,
                            pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (n < 0 || (n > 0 && !rows)) return fail(ctx, PAS_ERR_ARG, "bad rows / n");
  if ((s = validate_rows(ctx, rows, dtype))) return s;
  if (n > ctx->cfg.max_batch) return fail(ctx, PAS_ERR_CAPACITY, "n > max_batch (rows are staged like a batch)");
  if (n == 0) return PAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_prompt_ws(ctx))) return s;
  if ((s = ensure_lru_ws(ctx))) return s;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->invalid_count, 0, sizeof(int), st));
  CUDA_TRY(ctx, launch_normalize(rows, dtype, n, ctx->cfg.d, ctx->qhat, nullptr, 0, 1, 0, ctx->invalid_count, st));
  int bad = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&bad, ctx->invalid_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (bad) return fail(ctx, PAS_ERR_INVALID_ROWS, "%d of the rows are non-finite or have zero norm", bad);
  if ((s = insert_staged(ctx, nullptr, n, gids_out, nullptr, st))) return s;
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return PAS_OK;
}

pas_status pas_cache_insert_vanilla(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N,
                                    const int32_t* K_prime, int32_t* gids_by_prompt, int64_t* n_inserted,
                                    pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (n_inserted) *n_inserted = 0;
  if (N < 0 || (N > 0 && (!emb || !K_prime))) return fail(ctx, PAS_ERR_ARG, "bad emb / K_prime / N");
  if ((s = validate_rows(ctx, emb, dtype))) return s;
  if (N > ctx->cfg.max_batch) return fail(ctx, PAS_ERR_CAPACITY, "N > max_batch");
  if (N == 0) return PAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_prompt_ws(ctx))) return s;
  if ((s = ensure_lru_ws(ctx))) return s;
  // stage all N (validity flags; invalid prompts are skipped, R25), then compact K' == 0 in order
  CUDA_TRY(ctx, launch_normalize(emb, dtype, N, ctx->cfg.d, ctx->qhat, ctx->pflags, 0, 1, 0, nullptr, st));
  CUDA_TRY(ctx, launch_vanilla_compact(K_prime, ctx->pflags, N, ctx->lru_counts, ctx->lru_scanned,
                                       ctx->lru_scan_tmp, ctx->ins_idx, ctx->ins_count, gids_by_prompt, st));
  int n = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&n, ctx->ins_count, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (n > 0 && (s = insert_staged(ctx, ctx->ins_idx, n, nullptr, gids_by_prompt, st))) return s;
  ctx->last_local_N = -1;
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (n_inserted) *n_inserted = n;
  return PAS_OK;
}

pas_status pas_cache_stamps(pas_ctx* ctx, uint32_t* stamps_dev, int64_t n, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!stamps_dev || n < 0 || n > (int64_t)ctx->cfg.world * ctx->cap_rows)
    return fail(ctx, PAS_ERR_ARG, "bad stamps buffer / n");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaMemcpyAsync(stamps_dev, ctx->stamps, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream));
  return PAS_OK;
}

pas_status pas_set_bands(pas_ctx* ctx, const int32_t* K_levels, int nK, const float* thresholds) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (!K_levels || nK < 1 || nK > kMaxLevels || (nK > 1 && !thresholds))
    return fail(ctx, PAS_ERR_BANDS, "need 1 <= nK <= %d levels and nK-1 thresholds", kMaxLevels);
  if (K_levels[0] != 0) return fail(ctx, PAS_ERR_BANDS, "level 0 required (K_levels[0] == 0, S:29)");
  for (int i = 0; i < nK; ++i) {
    if (K_levels[i] < 0 || K_levels[i] >= kTTotal) return fail(ctx, PAS_ERR_BANDS, "K must be in [0, %d)", kTTotal);
    if (i && K_levels[i] <= K_levels[i - 1]) return fail(ctx, PAS_ERR_BANDS, "K levels must be strictly increasing");
  }
  for (int m = 0; m + 1 < nK; ++m) {
    if (!std::isfinite(thresholds[m])) return fail(ctx, PAS_ERR_BANDS, "thresholds must be finite");
    if (m && !(thresholds[m] > thresholds[m - 1]))
      return fail(ctx, PAS_ERR_BANDS, "thresholds must be strictly increasing (S:150)");
  }
  ctx->nK = nK;
  for (int i = 0; i < kMaxLevels; ++i) {
    ctx->grid[i] = i < nK ? K_levels[i] : 0;
    ctx->thr[i] = i + 1 < nK ? thresholds[i] : 0.f;
  }
  ctx->bands_set = true;
  ctx->fractions_set = false;
  if (ctx->fc_window > 0) {   // the window holds level indices of the old bands: start afresh
    CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
    CUDA_TRY(ctx, cudaDeviceSynchronize());   // no batch in flight may still read or write the window
    CUDA_TRY(ctx, cudaMemset(ctx->fc_state, 0, sizeof(FcState)));
    ctx->fc_tick = 0;
    ctx->fc_planned = false;
  }
  return PAS_OK;
}

pas_status pas_set_forecast(pas_ctx* ctx, int window, int replan_every) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (window < 0 || window > PAS_MAX_FORECAST_WINDOW)
    return fail(ctx, PAS_ERR_ARG, "window must be in [0, %d]", PAS_MAX_FORECAST_WINDOW);
  if (replan_every < 1) return fail(ctx, PAS_ERR_ARG, "replan_every must be >= 1");
  if (window > 0 && !ctx->bands_set) return fail(ctx, PAS_ERR_STATE, "pas_set_bands must precede pas_set_forecast");
  if (window > 0 && !ctx->c_convex)
    return fail(ctx, PAS_ERR_DEGRADATION, "the forecast-driven mode's coupling plan needs a convex c (R22)");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaDeviceSynchronize());   // no batch in flight may still read the old window
  if (window > 0) {
    if (window > ctx->fc_window) {
      if (ctx->fc_ring) cudaFree(ctx->fc_ring);
      ctx->fc_ring = nullptr;
      cudaError_t e = dmalloc(&ctx->fc_ring, (size_t)window);
      if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "forecast window allocation failed");
    }
    if (!ctx->fc_state) {
      cudaError_t e = dmalloc(&ctx->fc_state, 1);
      if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "forecast state allocation failed");
    }
    CUDA_TRY(ctx, cudaMemset(ctx->fc_state, 0, sizeof(FcState)));
  }
  ctx->fc_window = window;
  ctx->fc_replan_every = replan_every;
  ctx->fc_tick = 0;
  ctx->fc_planned = false;
  ctx->fc_stats_valid = false;
  return PAS_OK;
}

pas_status pas_set_degradation(pas_ctx* ctx, const double* c, int len) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (!c || len != kTTotal) return fail(ctx, PAS_ERR_DEGRADATION, "c must have PAS_T_TOTAL = %d entries", kTTotal);
  if (c[0] != 0.0) return fail(ctx, PAS_ERR_DEGRADATION, "c[0] must be 0");
  for (int t = 0; t < len; ++t)
    if (!std::isfinite(c[t])) return fail(ctx, PAS_ERR_DEGRADATION, "c must be finite");
  for (int t = 1; t < len; ++t)
    if (c[t] < c[t - 1]) return fail(ctx, PAS_ERR_DEGRADATION, "c must be non-decreasing");
  bool convex = true;
  for (int t = 1; t + 1 < len; ++t) {
    const double sec = c[t + 1] - 2 * c[t] + c[t - 1];
    if (sec < -1e-12 * (1.0 + std::fabs(c[t]))) convex = false;
  }
  if (!convex) {   // R37: exact integer costs for the min-cost solver; D_int = sum x cI < 2^50 needs c <= 1
    if (c[len - 1] > 1.0)
      return fail(ctx, PAS_ERR_DEGRADATION, "a non-convex c must stay in [0, 1] (quality loss, S:74)");
    if (ctx->fc_window > 0)
      return fail(ctx, PAS_ERR_DEGRADATION, "the forecast-driven mode's coupling plan needs a convex c (R22)");
  }
  for (int t = 0; t < kTTotal; ++t) {
    ctx->c[t] = c[t];
    ctx->cI[t] = convex ? 0 : (int64_t)std::nearbyint(std::ldexp(c[t], kDegShift));   // exact scaling, RNE
  }
  ctx->c_convex = convex;
  return PAS_OK;
}

pas_status pas_set_fractions(pas_ctx* ctx, const double* F, const int32_t* instance_level, int W, int bstar,
                             pas_mode mode) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (!ctx->bands_set) return fail(ctx, PAS_ERR_STATE, "pas_set_bands must precede pas_set_fractions");
  if (!F || !instance_level) return fail(ctx, PAS_ERR_ARG, "null argument");
  if (W < 1 || W > kMaxInst) return fail(ctx, PAS_ERR_ARG, "W must be in [1, %d]", kMaxInst);
  if (bstar < 1) return fail(ctx, PAS_ERR_ARG, "bstar must be >= 1");
  if (mode != PAS_GREEDY && mode != PAS_UNIFORM) return fail(ctx, PAS_ERR_ARG, "unknown mode");
  if (mode == PAS_UNIFORM && bstar != 1) return fail(ctx, PAS_ERR_ARG, "uniform routing uses batch size 1 (P:104)");
  double sum = 0.0;
  for (int j = 0; j < ctx->nK; ++j) {
    if (!std::isfinite(F[j]) || F[j] < 0.0) return fail(ctx, PAS_ERR_FRACTIONS, "F must be finite and >= 0");
    sum += F[j];
  }
  if (std::fabs(sum - 1.0) > 1e-9) return fail(ctx, PAS_ERR_FRACTIONS, "sum F = %.12g != 1 (S:35)", sum);
  bool has[kMaxLevels] = {false};
  for (int w = 0; w < W; ++w) {
    if (instance_level[w] < 0 || instance_level[w] >= ctx->nK)
      return fail(ctx, PAS_ERR_ARG, "instance_level[%d] = %d outside [0, nK)", w, instance_level[w]);
    has[instance_level[w]] = true;
  }
  for (int j = 0; j < ctx->nK; ++j)
    if (F[j] > 0.0 && !has[j])
      return fail(ctx, PAS_ERR_NO_INSTANCE, "F[%d] > 0 but no instance runs level %d (S:309)", j, j);
  if (ctx->disp_on && (W != ctx->disp_W || bstar > kArrRing))
    return fail(ctx, PAS_ERR_ARG, "the stateful dispatcher needs W = %d (as set) and bstar <= %d", ctx->disp_W,
                kArrRing);
  for (int j = 0; j < kMaxLevels; ++j) ctx->F[j] = j < ctx->nK ? F[j] : 0.0;
  for (int w = 0; w < kMaxInst; ++w) ctx->inst_level[w] = w < W ? instance_level[w] : 0;
  ctx->W = W;
  ctx->bstar = bstar;
  ctx->mode = mode;
  ctx->load_mode = mode;
  ctx->fractions_set = true;
  return PAS_OK;
}

pas_status pas_stage_ring(pas_ctx* ctx, int slots) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (slots < 0 || slots > PAS_MAX_RING) return fail(ctx, PAS_ERR_ARG, "slots outside [0, %d]", PAS_MAX_RING);
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  for (auto e : ctx->ring) cudaEventDestroy(e);
  ctx->ring.assign((size_t)slots * 7, nullptr);
  for (auto& e : ctx->ring) CUDA_TRY(ctx, cudaEventCreate(&e));
  ctx->ring_n = slots;
  ctx->ring_pos = ctx->ring_count = 0;
  return PAS_OK;
}

pas_status pas_stage_ring_read(pas_ctx* ctx, int n, float* ms, int* n_out) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!ms || !n_out || n < 0) return fail(ctx, PAS_ERR_ARG, "bad arguments");
  *n_out = 0;
  const int64_t have = ctx->ring_count < n ? ctx->ring_count : n;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  for (int64_t b = 0; b < have; ++b) {   // oldest first
    const int64_t slot = (ctx->ring_pos - have + b) % ctx->ring_n;
    cudaEvent_t* e = &ctx->ring[slot * 7];
    CUDA_TRY(ctx, cudaEventSynchronize(e[6]));
    for (int i = 0; i < 6; ++i) CUDA_TRY(ctx, cudaEventElapsedTime(&ms[b * 7 + i], e[i], e[i + 1]));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms[b * 7 + 6], e[0], e[6]));
  }
  *n_out = (int)have;
  return PAS_OK;
}

pas_status pas_set_collectives(pas_ctx* ctx, int mode) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (mode != PAS_COLL_FOLDED && mode != PAS_COLL_EXPLICIT) return fail(ctx, PAS_ERR_ARG, "unknown collective mode");
  ctx->coll_mode = mode;
  return PAS_OK;
}

pas_status pas_set_seed(pas_ctx* ctx, uint64_t seed, uint64_t batch_seq) {
  pas_status s = check_live(ctx);
  if (s) return s;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaDeviceSynchronize());   // batches in flight keep the sequence they were enqueued with
  CUDA_TRY(ctx, cudaMemcpy(&ctx->bc->batch_seq, &batch_seq, sizeof batch_seq, cudaMemcpyHostToDevice));
  ctx->seed = seed;
  ctx->batch_seq = batch_seq;
  ctx->graph_valid = false;
  return PAS_OK;
}

pas_status pas_set_dispatcher(pas_ctx* ctx, const int64_t* service_us, int W, int64_t timeout_us) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (!service_us) {   // back to the stateless packing
    ctx->disp_on = false;
    ctx->disp_stats_valid = false;
    return PAS_OK;
  }
  if (!ctx->fractions_set) return fail(ctx, PAS_ERR_STATE, "pas_set_fractions must precede pas_set_dispatcher");
  if (W != ctx->W) return fail(ctx, PAS_ERR_ARG, "W = %d differs from the W = %d of pas_set_fractions", W, ctx->W);
  if (ctx->bstar > kArrRing) return fail(ctx, PAS_ERR_ARG, "the stateful dispatcher needs bstar <= %d", kArrRing);
  if (timeout_us < 0 || timeout_us > PAS_MAX_TIME_US) return fail(ctx, PAS_ERR_ARG, "timeout_us outside [0, 2^52]");
  for (int w = 0; w < W; ++w)
    if (service_us[w] < 1 || service_us[w] > PAS_MAX_SERVICE_US)
      return fail(ctx, PAS_ERR_ARG, "service_us[%d] outside [1, 2^26]", w);
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if (!ctx->dstate) {
    cudaError_t e = dmalloc(&ctx->dstate, 1);
    if (e == cudaSuccess) e = dmalloc(&ctx->dplan, 1);
    CUDA_TRY(ctx, e);
  }
  DispState* h = new DispState();   // ~40 KB: not on the stack
  for (int w = 0; w < kMaxInst; ++w) {
    h->B[w] = kNeverBusy;
    h->svc[w] = w < W ? service_us[w] : 1;
  }
  cudaError_t e = cudaMemcpy(ctx->dstate, h, sizeof(DispState), cudaMemcpyHostToDevice);
  delete h;
  CUDA_TRY(ctx, e);
  for (int w = 0; w < kMaxInst; ++w) ctx->disp_svc[w] = w < W ? service_us[w] : 0;
  ctx->disp_on = true;
  ctx->disp_stats_valid = false;
  ctx->disp_W = W;
  ctx->disp_timeout = timeout_us;
  ctx->disp_now = ctx->disp_last = 0;
  ctx->disp_bstar_prev = ctx->bstar;
  return PAS_OK;
}

pas_status pas_set_clock(pas_ctx* ctx, int64_t now_us) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!ctx->disp_on) return fail(ctx, PAS_ERR_STATE, "pas_set_clock needs pas_set_dispatcher");
  if (now_us < ctx->disp_last || now_us > PAS_MAX_TIME_US)
    return fail(ctx, PAS_ERR_ARG, "now_us = %lld must be in [last batch = %lld, 2^52]", (long long)now_us,
                (long long)ctx->disp_last);
  ctx->disp_now = now_us;
  return PAS_OK;
}

pas_status pas_set_load(pas_ctx* ctx, double lambda_rps, int bstar_high, pas_mode* mode_out) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_valid = false;   // a captured batch bakes this state in
  if (!ctx->disp_on) return fail(ctx, PAS_ERR_STATE, "pas_set_load needs pas_set_dispatcher (service times)");
  if (!(lambda_rps >= 0.0) || !std::isfinite(lambda_rps)) return fail(ctx, PAS_ERR_ARG, "lambda must be finite, >= 0");
  if (bstar_high < 1 || bstar_high > kArrRing) return fail(ctx, PAS_ERR_ARG, "bstar_high outside [1, %d]", kArrRing);
  // R32: capacity at the optimal batch size; low -> high above 0.8, high -> low below 0.7
  double cap = 0.0;
  for (int w = 0; w < ctx->W; ++w) cap += (double)bstar_high / ((double)ctx->disp_svc[w] * 1e-6);
  const double u = lambda_rps / cap;
  int mode = ctx->load_mode;
  if (mode == PAS_UNIFORM) mode = u > 0.8 ? PAS_GREEDY : PAS_UNIFORM;
  else mode = u < 0.8 - 0.1 ? PAS_UNIFORM : PAS_GREEDY;
  ctx->load_mode = mode;
  ctx->mode = mode;
  ctx->bstar = mode == PAS_GREEDY ? bstar_high : 1;
  if (mode_out) *mode_out = (pas_mode)mode;
  return PAS_OK;
}

pas_status pas_dispatcher_state(pas_ctx* ctx, int64_t* queue_len, int64_t* busy_until_us, int64_t* fired_prompts,
                                int64_t* fired_batches) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!ctx->disp_on) return fail(ctx, PAS_ERR_STATE, "the stateful dispatcher is off");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  DispState* h = new DispState();
  cudaError_t e = cudaMemcpy(h, ctx->dstate, sizeof(DispState), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    for (int w = 0; w < ctx->disp_W; ++w) {
      if (queue_len) queue_len[w] = h->Q[w];
      if (busy_until_us) busy_until_us[w] = h->B[w];
      if (fired_prompts) fired_prompts[w] = h->fired_prompts[w];
      if (fired_batches) fired_batches[w] = h->fired_batches[w];
    }
  delete h;
  CUDA_TRY(ctx, e);
  return PAS_OK;
}

pas_status pas_solve_assignment(pas_ctx* ctx, int W, double lambda_rps, const double* H,
                                const int64_t* service_us, int bstar, pas_assignment* out) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!ctx->bands_set) return fail(ctx, PAS_ERR_STATE, "pas_set_bands must precede pas_solve_assignment");
  if (!service_us || !out) return fail(ctx, PAS_ERR_ARG, "null argument");
  if (W < 1 || W > kMaxInst) return fail(ctx, PAS_ERR_ARG, "W must be in [1, %d]", kMaxInst);
  if (bstar < 1) return fail(ctx, PAS_ERR_ARG, "bstar must be >= 1");
  if (!(lambda_rps >= 0.0) || !std::isfinite(lambda_rps)) return fail(ctx, PAS_ERR_ARG, "lambda must be finite, >= 0");
  if (!H && ctx->fc_window == 0)
    return fail(ctx, PAS_ERR_STATE, "H == NULL takes the forecast window: pas_set_forecast first");
  AssignParams p{};
  p.nK = ctx->nK;
  p.W = W;
  p.bstar = bstar;
  p.lam = lambda_rps;
  const int64_t total = assign_count(W, ctx->nK);
  if (total > PAS_MAX_ASSIGNMENTS)
    return fail(ctx, PAS_ERR_ARG, "C(W + nK - 1, nK - 1) = %lld assignments exceed %lld", (long long)total,
                (long long)PAS_MAX_ASSIGNMENTS);
  for (int k = 0; k < ctx->nK; ++k) {
    if (service_us[k] < 1 || service_us[k] > PAS_MAX_SERVICE_US)
      return fail(ctx, PAS_ERR_ARG, "service_us[%d] outside [1, 2^26]", k);
    if (H && (!std::isfinite(H[k]) || H[k] < 0.0)) return fail(ctx, PAS_ERR_ARG, "H must be finite and >= 0");
    p.grid[k] = ctx->grid[k];
    p.service_us[k] = service_us[k];
    p.H[k] = H ? H[k] : 0.0;
  }
  if (H) {   // a_K = 1 - sum_i H_i c(K - K_i) is SPEC's expected quality only for a distribution
    double hs = 0.0;
    for (int k = 0; k < ctx->nK; ++k) hs += H[k];
    if (std::fabs(hs - 1.0) > 1e-9) return fail(ctx, PAS_ERR_ARG, "sum H = %.12g != 1 (S:35)", hs);
  }
  for (int t = 0; t < kTTotal; ++t) p.c[t] = ctx->c[t];
  p.fc = H ? nullptr : ctx->fc_state;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  constexpr int kMaxBlocks = kNumSMs * 8;
  if (!ctx->asg_keys) {
    cudaError_t e = cudaMalloc(&ctx->asg_keys, assign_key_bytes() * kMaxBlocks);
    if (e == cudaSuccess) e = dmalloc(&ctx->asg_out, 1);
    CUDA_TRY(ctx, e);
  }
  cudaStream_t st = ctx->last_stream;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev[7], st));
  CUDA_TRY(ctx, launch_assign(p, ctx->asg_keys, kMaxBlocks, ctx->asg_out, st));
  cudaEvent_t done = ctx->ev_aux;
  CUDA_TRY(ctx, cudaEventRecord(done, st));
  AssignOut h;
  CUDA_TRY(ctx, cudaMemcpyAsync(&h, ctx->asg_out, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[7], done);
  memset(out, 0, sizeof(*out));
  out->nK = ctx->nK;
  out->W = W;
  for (int k = 0; k < ctx->nK; ++k) {
    out->n[k] = h.n[k];
    out->F[k] = h.F[k];
    out->F_route[k] = h.F_route[k];
    out->H[k] = h.H[k];
  }
  for (int w = 0; w < W; ++w) out->instance_level[w] = h.instance_level[w];
  out->served = h.served;
  out->quality = h.quality;
  out->candidates = total;
  out->solve_ms = ms;
  return PAS_OK;
}

pas_status pas_route_local(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N, void* cand_dev,
                           pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (N < 0 || N > ctx->cfg.max_batch) return fail(ctx, PAS_ERR_CAPACITY, "N outside [0, max_batch]");
  if ((s = validate_rows(ctx, emb, dtype))) return s;
  if (N > 0 && (!emb || !cand_dev)) return fail(ctx, PAS_ERR_ARG, "null emb / cand");
  ctx->launches = 0;
  if (N == 0) return PAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_prompt_ws(ctx))) return s;
  CUDA_TRY(ctx, rec_stage(ctx, 0, st));
  const Cand* cand;
  int S;
  return run_local(ctx, emb, dtype, N, st, &cand, &S, static_cast<Cand*>(cand_dev));
}

pas_status pas_route_from_candidates(pas_ctx* ctx, const void* cand_dev, int S, int64_t N, const pas_route_out* out,
                                     pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if ((s = ready(ctx, N))) return s;
  if (S < 1 || S > 128) return fail(ctx, PAS_ERR_ARG, "S must be in [1, 128]");
  if (N == 0) return PAS_OK;
  if ((s = validate_out(ctx, out))) return s;
  if (!cand_dev) return fail(ctx, PAS_ERR_ARG, "null candidates");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, rec_stage(ctx, 0, st));
  CUDA_TRY(ctx, rec_stage(ctx, 1, st));
  CUDA_TRY(ctx, rec_stage(ctx, 2, st));
  return run_global(ctx, static_cast<const Cand*>(cand_dev), S, N, out, st);
}

namespace {
// The whole batch enqueued on st (eager, or into a graph being captured).
pas_status route_enqueue(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N, const pas_route_out* out,
                         cudaStream_t st) {
  pas_status s;
  const int G = ctx->cfg.world;
  CUDA_TRY(ctx, rec_stage(ctx, 0, st));
  const Cand* cand;
  int S;
  if (!ctx->comm) {
    if ((s = run_local(ctx, emb, dtype, N, st, &cand, &S, nullptr))) return s;
  } else {
    if ((s = run_local(ctx, emb, dtype, N, st, &cand, &S, ctx->cand_rank))) return s;
    const size_t count = (size_t)N * ctx->cfg.topk * 2;   // (score, gid) as 2 x 32-bit words
    ncclResult_t r = g_nccl.AllGather(ctx->cand_rank, ctx->cand_all, count, ncclInt32, ctx->comm, st);
    if (r != ncclSuccess) return fail(ctx, PAS_ERR_NCCL, "ncclAllGather: %s", g_nccl.GetErrorString(r));
    // ncclAllGather places rank r's N*k pairs at offset r*N*k: the layout is [G][N][k]
    cand = ctx->cand_all;
    S = G;
    if (ctx->coll_mode == PAS_COLL_EXPLICIT) return run_global_explicit(ctx, cand, N, out, st);
  }
  return run_global(ctx, cand, S, N, out, st);
}

bool same_out(const pas_route_out& a, const pas_route_out& b) { return memcmp(&a, &b, sizeof a) == 0; }

// Capture the batch into ctx->gexec (the host-side counters the capture advanced are restored: the
// graph has not run yet).
pas_status capture_graph(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N, const pas_route_out* out) {
  if (!ctx->cap_stream) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  if (ctx->gexec) {
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  const uint64_t bseq = ctx->batch_seq;
  const uint32_t tick = ctx->lru_tick;
  CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
  ctx->capturing = true;
  ctx->launches = 0;
  pas_status s = route_enqueue(ctx, emb, dtype, N, out, ctx->cap_stream);
  ctx->capturing = false;
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
  ctx->batch_seq = bseq;
  ctx->lru_tick = tick;
  if (s != PAS_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  if (e != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(e));
  const cudaError_t ei = cudaGraphInstantiate(&ctx->gexec, g, 0);
  cudaGraphDestroy(g);
  if (ei != cudaSuccess) return fail(ctx, PAS_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ei));
  ctx->g_emb = emb;
  ctx->g_dtype = dtype;
  ctx->g_N = N;
  ctx->g_out = *out;
  ctx->g_launches = ctx->launches;
  ctx->graph_valid = true;
  return PAS_OK;
}
}  // namespace

pas_status pas_set_graph(pas_ctx* ctx, int on) {
  pas_status s = check_live(ctx);
  if (s) return s;
  ctx->graph_on = on != 0;
  ctx->graph_valid = false;
  return PAS_OK;
}

pas_status pas_route_batch(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N, const pas_route_out* out,
                           pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if ((s = ready(ctx, N))) return s;
  if ((s = validate_rows(ctx, emb, dtype))) return s;
  ctx->launches = 0;
  if (N == 0) return PAS_OK;
  if ((s = validate_out(ctx, out))) return s;
  if (!emb) return fail(ctx, PAS_ERR_ARG, "emb is NULL");
  const int G = ctx->cfg.world;
  if (G > 1 && !ctx->comm)
    return fail(ctx, PAS_ERR_STATE, "world > 1 without an NCCL communicator: use the split calls");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_prompt_ws(ctx))) return s;   // first call only: outside the timed stages
  // graph replay: the stateless exact-plan path (the forecast / dispatcher modes carry host-side state
  // per batch and run eagerly)
  if (ctx->graph_on && !ctx->disp_on && ctx->fc_window == 0) {
    if (!ctx->graph_valid || ctx->g_emb != emb || ctx->g_dtype != (int)dtype || ctx->g_N != N ||
        !same_out(ctx->g_out, *out))
      if ((s = capture_graph(ctx, emb, dtype, N, out))) return s;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[0], st));
    CUDA_TRY(ctx, cudaGraphLaunch(ctx->gexec, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev[6], st));
    ctx->launches = ctx->g_launches;
    ctx->lru_tick++;   // the host mirrors of what the replayed batch advanced on the device
    ctx->batch_seq++;
    ctx->last_local_N = -1;
    ctx->ev_valid = true;
    ctx->stages_valid = false;
    ctx->last_stream = st;
    ctx->last_N = N;
    ctx->fc_stats_valid = false;
    ctx->disp_stats_valid = false;
    return PAS_OK;
  }
  return route_enqueue(ctx, emb, dtype, N, out, st);
}

namespace {
// The device→host copies of one routed batch (every non-NULL array of oh) on stream st.
pas_status copy_out(pas_ctx* ctx, const pas_route_out& od, const pas_route_out* oh, int64_t N, cudaStream_t st) {
  const int64_t k = ctx->cfg.topk;
  const int W = ctx->W;
  CUDA_TRY(ctx, cudaMemcpyAsync(oh->K, od.K, N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(oh->K_prime, od.K_prime, N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(oh->instance, od.instance, N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(oh->slot, od.slot, N * 4, cudaMemcpyDeviceToHost, st));
  if (oh->topk_id) CUDA_TRY(ctx, cudaMemcpyAsync(oh->topk_id, od.topk_id, N * k * 4, cudaMemcpyDeviceToHost, st));
  if (oh->topk_score)
    CUDA_TRY(ctx, cudaMemcpyAsync(oh->topk_score, od.topk_score, N * k * 4, cudaMemcpyDeviceToHost, st));
  if (oh->flags) CUDA_TRY(ctx, cudaMemcpyAsync(oh->flags, od.flags, N, cudaMemcpyDeviceToHost, st));
  if (oh->bucket_offsets)
    CUDA_TRY(ctx, cudaMemcpyAsync(oh->bucket_offsets, od.bucket_offsets, (W + 1) * 4, cudaMemcpyDeviceToHost, st));
  if (oh->bucket_prompts)
    CUDA_TRY(ctx, cudaMemcpyAsync(oh->bucket_prompts, od.bucket_prompts, N * 4, cudaMemcpyDeviceToHost, st));
  return PAS_OK;
}
}  // namespace

pas_status pas_route_batch_host(pas_ctx* ctx, const void* emb_host, pas_dtype dtype, int64_t N,
                                const pas_route_out* oh, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if ((s = ready(ctx, N))) return s;
  if (dtype != PAS_F32 && dtype != PAS_BF16) return fail(ctx, PAS_ERR_ARG, "bad dtype");
  if (N == 0) return PAS_OK;
  if ((s = validate_out(ctx, oh, false))) return s;
  if (!emb_host) return fail(ctx, PAS_ERR_ARG, "emb_host is NULL");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  const int64_t mb = ctx->cfg.max_batch, k = ctx->cfg.topk;
  cudaError_t e = cudaSuccess;
  if (!ctx->stage_emb) {
    e = cudaMalloc(&ctx->stage_emb, (size_t)mb * ctx->cfg.d * 4);
    if (!e) e = dmalloc(&ctx->s_K, mb);
    if (!e) e = dmalloc(&ctx->s_Kp, mb);
    if (!e) e = dmalloc(&ctx->s_inst, mb);
    if (!e) e = dmalloc(&ctx->s_slot, mb);
    if (!e) e = dmalloc(&ctx->s_tid, mb * k);
    if (!e) e = dmalloc(&ctx->s_tsc, mb * k);
    if (!e) e = dmalloc(&ctx->s_flags, mb);
    if (!e) e = dmalloc(&ctx->s_boff, kMaxInst + 1);
    if (!e) e = dmalloc(&ctx->s_bpr, mb);
    CUDA_TRY(ctx, e);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t esz = dtype == PAS_F32 ? 4 : 2;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->stage_emb, emb_host, (size_t)N * ctx->cfg.d * esz, cudaMemcpyHostToDevice, st));
  pas_route_out od{ctx->s_K,   ctx->s_Kp,
                   ctx->s_inst, ctx->s_slot,
                   oh->topk_id ? ctx->s_tid : nullptr,
                   oh->topk_score ? ctx->s_tsc : nullptr,
                   oh->flags ? ctx->s_flags : nullptr,
                   oh->bucket_offsets ? ctx->s_boff : nullptr,
                   oh->bucket_prompts ? ctx->s_bpr : nullptr};
  if ((s = pas_route_batch(ctx, ctx->stage_emb, dtype, N, &od, stream))) return s;
  if ((s = copy_out(ctx, od, oh, N, st))) return s;
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return PAS_OK;
}


namespace {
// The pipelined host API's copy streams and fence event (created on first use).
pas_status ensure_host_streams(pas_ctx* ctx) {
  if (ctx->h2d_stream) return PAS_OK;
  CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
  CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->h_join, cudaEventDisableTiming));
  return PAS_OK;
}
}  // namespace

pas_status pas_route_batch_host_async(pas_ctx* ctx, const void* emb_host, pas_dtype dtype, int64_t N,
                                      const pas_route_out* oh, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if ((s = ready(ctx, N))) return s;
  if (dtype != PAS_F32 && dtype != PAS_BF16) return fail(ctx, PAS_ERR_ARG, "bad dtype");
  if (N == 0) return PAS_OK;
  if ((s = validate_out(ctx, oh, false))) return s;
  if (!emb_host) return fail(ctx, PAS_ERR_ARG, "emb_host is NULL");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  const int64_t mb = ctx->cfg.max_batch, k = ctx->cfg.topk;
  if ((s = ensure_host_streams(ctx))) return s;
  pas_ctx::HostSlot& S = ctx->hs[ctx->hseq & 1];
  if (!S.emb) {
    cudaError_t e = cudaMalloc(&S.emb, (size_t)mb * ctx->cfg.d * 4);
    if (!e) e = dmalloc(&S.K, mb);
    if (!e) e = dmalloc(&S.Kp, mb);
    if (!e) e = dmalloc(&S.inst, mb);
    if (!e) e = dmalloc(&S.slot, mb);
    if (!e) e = dmalloc(&S.tid, mb * k);
    if (!e) e = dmalloc(&S.tsc, mb * k);
    if (!e) e = dmalloc(&S.flags, mb);
    if (!e) e = dmalloc(&S.boff, kMaxInst + 1);
    if (!e) e = dmalloc(&S.bpr, mb);
    for (cudaEvent_t* ev : {&S.h2d, &S.done, &S.d2h})
      if (!e) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    CUDA_TRY(ctx, e);
  }
  // at most two batches in flight: this slot's previous batch must have delivered its outputs (its
  // input buffer was consumed before those copies started)
  if (S.used) CUDA_TRY(ctx, cudaEventSynchronize(S.d2h));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t esz = dtype == PAS_F32 ? 4 : 2;
  CUDA_TRY(ctx, cudaMemcpyAsync(S.emb, emb_host, (size_t)N * ctx->cfg.d * esz, cudaMemcpyHostToDevice, ctx->h2d_stream));
  CUDA_TRY(ctx, cudaEventRecord(S.h2d, ctx->h2d_stream));
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, S.h2d, 0));
  pas_route_out od{S.K, S.Kp, S.inst, S.slot,
                   oh->topk_id ? S.tid : nullptr,
                   oh->topk_score ? S.tsc : nullptr,
                   oh->flags ? S.flags : nullptr,
                   oh->bucket_offsets ? S.boff : nullptr,
                   oh->bucket_prompts ? S.bpr : nullptr};
  if ((s = pas_route_batch(ctx, S.emb, dtype, N, &od, stream))) return s;
  CUDA_TRY(ctx, cudaEventRecord(S.done, st));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->d2h_stream, S.done, 0));
  if ((s = copy_out(ctx, od, oh, N, ctx->d2h_stream))) return s;
  CUDA_TRY(ctx, cudaEventRecord(S.d2h, ctx->d2h_stream));
  S.used = true;
  ctx->hseq++;
  return PAS_OK;
}

pas_status pas_route_host_begin(pas_ctx* ctx, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_host_streams(ctx))) return s;
  CUDA_TRY(ctx, cudaEventRecord(ctx->h_join, (cudaStream_t)stream));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->h2d_stream, ctx->h_join, 0));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->d2h_stream, ctx->h_join, 0));
  return PAS_OK;
}

pas_status pas_route_host_end(pas_ctx* ctx, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  for (auto& S : ctx->hs)
    if (S.used) CUDA_TRY(ctx, cudaStreamWaitEvent((cudaStream_t)stream, S.d2h, 0));
  return PAS_OK;
}

pas_status pas_plan_stats(pas_ctx* ctx, pas_stats* out) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!out) return fail(ctx, PAS_ERR_ARG, "out is NULL");
  memset(out, 0, sizeof(*out));
  out->nK = ctx->nK;
  out->W = ctx->W;
  if (!ctx->ev_valid) return PAS_OK;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev[6]));
  DevPlan p;
  CUDA_TRY(ctx, cudaMemcpy(&p, ctx->plan, sizeof p, cudaMemcpyDeviceToHost));
  out->N = ctx->last_N;
  for (int i = 0; i < ctx->nK; ++i) {
    out->h[i] = p.h[i];
    out->f[i] = p.f[i];
    for (int j = 0; j < ctx->nK; ++j) out->x[i][j] = p.x[i][j];
  }
  out->D_Q = p.D_Q;
  out->D_Q_LP = p.D_Q_LP;
  out->plan_solver_iters = p.solver_iters;
  out->k6_fallback = p.k6_fallback;
  out->n_redirected = p.n_redirected;
  out->n_upgraded = p.n_upgraded;
  out->n_downgraded = p.n_downgraded;
  out->n_invalid = p.n_invalid;
  out->n_near_top1 = p.n_near_top1;
  out->n_near_threshold = p.n_near_threshold;
  for (int w = 0; w < ctx->W; ++w) out->bucket_count[w] = p.inst_count[w];
  out->k2_ranges = ctx->k2_last_R;
  out->k2_chunk_tiles = ctx->k2_last_T;
  out->k2_chunk_steps = ctx->k2_last_CS;
  if (ctx->fc_stats_valid) {
    FcState f;
    CUDA_TRY(ctx, cudaMemcpy(&f, ctx->fc_state, sizeof f, cudaMemcpyDeviceToHost));
    out->forecast = 1;
    out->fc_replanned = f.replanned;
    out->fc_plan_n = f.plan_n;
    for (int i = 0; i < ctx->nK; ++i) out->fc_plan_counts[i] = f.plan_cnt[i];
    out->fc_window_n = f.n;
    out->fc_l2_error = f.l2;
    out->n_unforecast = f.n_unforecast;
    for (int i = 0; i <= ctx->nK; ++i) {
      out->fc_Hc[i] = f.Hc[i];
      out->fc_Fc[i] = f.Fc[i];
    }
  }
  if (ctx->disp_stats_valid) {
    out->dispatcher = 1;
    out->now_us = ctx->disp_last;
    if ((s = pas_dispatcher_state(ctx, out->queue_len, out->busy_until_us, out->fired_prompts,
                                  out->fired_batches)))
      return s;
  }
  for (int i = 0; i < 6 && ctx->stages_valid; ++i) {   // a replayed graph: only the total
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]) == cudaSuccess) out->stage_ms[i] = ms;
  }
  float tot = 0.f;
  if (cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[6]) == cudaSuccess) out->stage_ms[6] = tot;
  cudaGetLastError();
  return PAS_OK;
}

// Test hooks: the bf16 rows K1 wrote -- the prompt-side Q_hat of the last a1 (R11) and this rank's store.
pas_status pas_debug_qhat(pas_ctx* ctx, void* out_dev, int64_t N, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!out_dev || N < 0 || N > ctx->cfg.max_batch) return fail(ctx, PAS_ERR_ARG, "bad out / N");
  if (N == 0) return PAS_OK;
  if (!ctx->qhat) return fail(ctx, PAS_ERR_STATE, "no prompt has been normalised yet");
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaMemcpyAsync(out_dev, ctx->qhat, (size_t)N * ctx->cfg.d * 2, cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream));
  return PAS_OK;
}

pas_status pas_debug_store_rows(pas_ctx* ctx, int64_t first_local_row, int64_t n, void* out_dev, pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (!out_dev || first_local_row < 0 || n < 0 || first_local_row + n > ctx->M_local)
    return fail(ctx, PAS_ERR_ARG, "rows [%lld, %lld) outside this rank's %lld", (long long)first_local_row,
                (long long)(first_local_row + n), (long long)ctx->M_local);
  if (n == 0) return PAS_OK;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(ctx, cudaMemcpyAsync(out_dev, ctx->store + first_local_row * ctx->cfg.d, (size_t)n * ctx->cfg.d * 2,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return PAS_OK;
}

// Test hook: K1 + K2 with the epilogue writing every raw score (no top-k); scores_dev [N x M_local].
pas_status pas_debug_k2_schedule(int64_t N, int64_t M_local, int d, int64_t max_batch, int* out) {
  if (!out || N < 0 || M_local < 0 || d <= 0 || max_batch < N) return PAS_ERR_ARG;
  DynSched dyn;
  const int64_t cap = k2_cand_cap(max_batch);
  out[0] = k2_schedule(N, M_local, d, cap, K2Tuning::from_env(), &dyn);
  out[1] = dyn.T;
  out[2] = dyn.CS;
  out[3] = dyn.MTg;
  out[4] = simtopk_pair(N, d) ? 1 : 0;
  out[5] = (int)((N + simtopk_box_q() - 1) / simtopk_box_q());
  const int tr = simtopk_tile_rows(N, M_local, d);
  out[6] = (int)((M_local + tr - 1) / tr);
  out[7] = (int)(cap > INT32_MAX ? INT32_MAX : cap);
  out[8] = tr;
  return PAS_OK;
}

pas_status pas_debug_scores(pas_ctx* ctx, const void* emb, pas_dtype dtype, int64_t N, float* scores_dev,
                            pas_stream stream) {
  pas_status s = check_live(ctx);
  if (s) return s;
  if (N < 1 || N > ctx->cfg.max_batch || !emb || !scores_dev) return fail(ctx, PAS_ERR_ARG, "bad arguments");
  if ((s = validate_rows(ctx, emb, dtype))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(ctx, cudaSetDevice(ctx->cfg.device));
  if ((s = ensure_prompt_ws(ctx))) return s;
  CUDA_TRY(ctx, launch_normalize(emb, dtype, N, ctx->cfg.d, ctx->qhat, ctx->pflags, 0, 1, 0, nullptr, st));
  SimTopkArgs a{&ctx->tm_q, &ctx->tm_c, &ctx->tm_c2, N, ctx->M_local, ctx->cfg.d, 1, ctx->cfg.world, ctx->cfg.rank, 1,
                ctx->qhat, ctx->cand_local, scores_dev, nullptr, 0, nullptr};
  CUDA_TRY(ctx, launch_simtopk(a, st));
  return PAS_OK;
}

}  // extern "C"
