/*
 * pas.h -- C-ABI of libpas, the B200-native prompt-routing hot path of
 *          "Prompt-Aware Scheduling for Efficient Text-to-Image Inferencing System"
 *          (arxiv 2502.06798; /root/reference/PAPER.md, cited as P:<line>).
 *
 * One call, pas_route_batch, runs the paper's per-batch Query Dispatcher path for N prompts:
 *   a1 normalise + quantise the prompt embeddings            ("closeness")
 *   a3 cosine similarity vs the approximate-cache store with a fused running top-k
 *                                                            ("retrieves the nearest cache")
 *   a4 merge of per-range / per-GPU candidates
 *   a5 best similarity -> optimal-K, H_K histogram
 *   a6 targets f from F(K), Eq. 1 K->K' route plan, D_Q      (P:88-P:96, Eq. 1)
 *   a7 redirection sampling (Philox, reproducible)           ("K-to-K' Router")
 *   a8 route-and-batch (greedy / uniform) into per-instance FIFO batches
 * Readings of silent or garbled passages are R1..R20 in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Every function returns pas_status; nothing throws across the ABI.  Arguments are
 *     validated before anything is enqueued, so a validation error writes nothing.
 *     pas_last_error(ctx) returns a per-context message for the last failure.
 *   - A CUDA or NCCL failure is sticky: the context is poisoned (every later call returns
 *     PAS_ERR_STATE) and must be destroyed.
 *   - Pointers named *_dev are device pointers on cfg.device; *_host are host pointers.
 *     Device work is enqueued on the caller's stream (stream-ordered, no host sync) unless
 *     the function says it synchronises.
 *   - One context per stream; calls on one context are not re-entrant.
 *   - Sizes are element counts unless stated.  Layouts are row-major, C order.
 */
#ifndef PAS_H_
#define PAS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pas_ctx pas_ctx;          /* opaque, library-owned */
typedef struct CUstream_st* pas_stream;  /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
  PAS_OK = 0,
  PAS_ERR_ARG = -1,          /* bad pointer / size / value */
  PAS_ERR_STATE = -2,        /* call order violated, or context poisoned */
  PAS_ERR_FRACTIONS = -3,    /* F(K) invalid (F >= 0, sum F = 1 +- 1e-9) */
  PAS_ERR_NO_INSTANCE = -4,  /* F_j > 0 but no serving instance at level j */
  PAS_ERR_BANDS = -5,        /* K grid / thresholds invalid */
  PAS_ERR_DEGRADATION = -6,  /* c(dK) not c[0]=0, finite, non-decreasing; non-convex c > 1 (R6, R37) */
  PAS_ERR_CAPACITY = -7,     /* store or batch capacity exceeded */
  PAS_ERR_CUDA = -8,
  PAS_ERR_NCCL = -9,
  PAS_ERR_INVALID_ROWS = -10 /* pas_cache_load: a row is non-finite or has zero norm (R16) */
} pas_status;

typedef enum { PAS_F32 = 0, PAS_BF16 = 1 } pas_dtype;
typedef enum { PAS_GREEDY = 0, PAS_UNIFORM = 1 } pas_mode;  /* P:104 high / low load */

#define PAS_MAX_LEVELS 16        /* nK <= 16 (configs use 6 and 10) */
#define PAS_MAX_INSTANCES 64     /* W <= 64 serving instances */
#define PAS_T_TOTAL 50           /* total denoising steps */
#define PAS_MAX_FORECAST_WINDOW (1 << 22)   /* f1 predictor window (paper: 1000) */
#define PAS_MAX_TOPK 16
#define PAS_NEVER_BUSY (-(INT64_C(1) << 62))  /* f3: busy-until of an instance that never fired */
#define PAS_MAX_TIME_US (INT64_C(1) << 52)    /* f3: clock and timeout range (us) */
#define PAS_MAX_SERVICE_US (INT64_C(1) << 26) /* f3: batch service time range (us, ~67 s) */
#define PAS_NCCL_ID_BYTES 128

/* Flags per prompt (pas_route_out.flags), informational; the oracle grades with its own. */
#define PAS_FLAG_INVALID 1        /* non-finite or zero-norm embedding -> treated as cold (R16) */
#define PAS_FLAG_COLD 2           /* empty cache -> K = 0 */
#define PAS_FLAG_NEAR_TOP1 4      /* GPU s1 - s2 < 2e-2 (north_star near-tie margin); needs topk >= 2 */
#define PAS_FLAG_NEAR_THRESHOLD 8 /* GPU |s1 - t_m| < 2e-2 for some threshold t_m */

typedef struct {
  int d;                       /* embedding width; multiple of 64, 64..4096 (configs: 768) */
  int topk;                    /* k, 1..PAS_MAX_TOPK (default 8) */
  int64_t max_batch;           /* largest N accepted by pas_route_batch */
  int64_t max_rows_per_rank;   /* store capacity of THIS rank's shard, rows */
  int device;                  /* CUDA device ordinal */
  int rank, world;             /* router GPUs: 0 <= rank < world; cache gid g lives on rank g % world */
  const unsigned char* nccl_id;/* PAS_NCCL_ID_BYTES from pas_nccl_unique_id on rank 0, broadcast by the
                                  caller; required iff world > 1 and pas_route_batch is to be used.
                                  NULL with world > 1 = "external transport": only the split calls
                                  pas_route_local / pas_route_from_candidates are available.
                                  Non-NULL with world == 1: a 1-rank communicator, pas_route_batch
                                  takes the all-gather path (transport self-test). */
  uint64_t seed;               /* Philox key of the redirection / uniform-routing streams (R18) */
} pas_config;

/* Per-prompt outputs, caller-owned DEVICE arrays (SoA), each 16-byte aligned (PAS_ERR_ARG otherwise).
 * Required arrays must be non-NULL. */
typedef struct {
  int32_t* K;               /* [N] optimal-K value (grid value, not index)                 required */
  int32_t* K_prime;         /* [N] K' the prompt is served at                              required */
  int32_t* instance;        /* [N] serving instance id in [0, W) ("gpu" of the north star, R12) required */
  int32_t* slot;            /* [N] FIFO position within that instance; batch = slot / bstar  required */
  int32_t* topk_id;         /* [N*topk] global cache ids of the k nearest, -1 padded         optional */
  float* topk_score;        /* [N*topk] their cosine similarities, -inf padded              optional */
  uint8_t* flags;           /* [N] PAS_FLAG_* bits                                          optional */
  int32_t* bucket_offsets;  /* [W+1] exclusive scan of per-instance counts                  optional */
  int32_t* bucket_prompts;  /* [N] prompt ids grouped by instance, FIFO (slot) order         optional */
} pas_route_out;

/* Host-side view of the last batch's plan (pas_plan_stats). */
typedef struct {
  int nK, W;
  int64_t N;
  int64_t h[PAS_MAX_LEVELS];                    /* H_K counts (R4) */
  int64_t f[PAS_MAX_LEVELS];                    /* integer targets from F (R3) */
  int64_t x[PAS_MAX_LEVELS][PAS_MAX_LEVELS];    /* route plan: x[i][j] prompts with optimal level i served at j */
  double D_Q;                                   /* Eq. 1 on the integer plan, sum_{K_j>K_i} x_ij D_ij / N */
  double D_Q_LP;                                /* Eq. 1 optimum on unrounded (h/N, F), context only (NaN:
                                                   non-convex c) */
  int plan_solver_iters;                        /* non-convex c: solver augmentations (-1: iteration cap hit,
                                                   the plan is feasible but not canonical); 0 otherwise */
  int64_t n_redirected, n_upgraded, n_downgraded;   /* K'!=K, K'<K (slower/better), K'>K */
  int64_t n_invalid, n_near_top1, n_near_threshold;
  int64_t bucket_count[PAS_MAX_INSTANCES];      /* prompts per instance */
  float stage_ms[8];    /* device ms per stage of the last batch: [0] normalise, [1] similarity+top-k,
                           [2] merge + collective + optimal-K/H_K, [3] plan, [4] redirect,
                           [5] route-and-batch, [6] total, [7] unused */
  /* forecast-driven mode (pas_set_forecast; all zero in the exact mode).  There, f and x are the
   * REALISED K' counts and moves, D_Q the realised sum_p D(K'_p, K_p) / N, and D_Q_LP the Eq. 1 value
   * of the fixed-point plan the batch was routed with (R22). */
  int forecast;                                 /* 1 if the last batch ran in forecast mode */
  int fc_replanned;                             /* the plan was rebuilt for this batch (R24) */
  int64_t fc_plan_n;                            /* window length the plan was built from (0: uniform) */
  int64_t fc_plan_counts[PAS_MAX_LEVELS];       /* window level counts the plan was built from */
  int64_t fc_window_n;                          /* window length after this batch */
  double fc_l2_error;                           /* |forecast H_K - realised h/N|_2 */
  int64_t n_unforecast;                         /* prompts of a level the forecast gave no mass (R23) */
  uint64_t fc_Hc[PAS_MAX_LEVELS + 1];           /* cumulative forecast mass, units of 2^-32 */
  uint64_t fc_Fc[PAS_MAX_LEVELS + 1];           /* cumulative F, units of 2^-32 */
  /* stateful dispatcher (pas_set_dispatcher; all zero when off): the state AFTER the last batch */
  int dispatcher;                               /* 1 if the last batch went through the stateful dispatcher */
  int64_t now_us;                               /* its arrival time */
  int64_t queue_len[PAS_MAX_INSTANCES];         /* prompts waiting per instance */
  int64_t busy_until_us[PAS_MAX_INSTANCES];     /* PAS_NEVER_BUSY if the instance never fired */
  int64_t fired_prompts[PAS_MAX_INSTANCES];     /* cumulative since pas_set_dispatcher */
  int64_t fired_batches[PAS_MAX_INSTANCES];
  /* K2 schedule of the last batch: cache ranges per prompt tile (the S of the merge),
   * and for the dynamic schedule the cache tiles per chunk and the chunk steps per range (0, 0: the
   * static schedule, one unit per (prompt tile, range)) */
  int k2_ranges, k2_chunk_tiles, k2_chunk_steps;
  /* K6 (a7): 1 if the windowed split search fell back to the exact histogram path for this batch (a split
   * rank outside its kappa window -- probability ~1e-15 --, a list overflow, > 32 splits, or forced) */
  int k6_fallback;
} pas_stats;

/* Library and build identification ("sm_100a", version). Never fails. */
const char* pas_version(void);

/* Create a context: allocates the store (max_rows_per_rank x d bf16), the per-batch workspace
 * (the prompt-side part -- max_batch x d bf16 and the candidate buffers -- on the first routing call
 * that needs it) and, if world > 1 and nccl_id != NULL, the NCCL communicator (collective over all
 * ranks).
 * Defaults after create: no bands (pas_set_bands required), c(dK) = 0.006 dK (R6),
 * batch_seq = 0.  Errors: PAS_ERR_ARG (bad cfg), PAS_ERR_CUDA (allocation), PAS_ERR_NCCL. */
pas_status pas_create(pas_ctx** ctx, const pas_config* cfg);

/* Destroy a context (also poisoned ones); frees everything it owns.  NULL is a no-op. */
pas_status pas_destroy(pas_ctx* ctx);

/* NCCL unique id for the world>1 bootstrap (rank 0 calls it, the caller broadcasts the bytes).
 * out: PAS_NCCL_ID_BYTES host bytes.  Errors: PAS_ERR_NCCL if NCCL cannot be loaded. */
pas_status pas_nccl_unique_id(unsigned char* out);

/* Append M cache rows (the approximate-cache store).  Every rank passes the SAME rows;
 * global id g = (rows already loaded) + i; this rank keeps rows with g % world == rank at local row
 * g / world, normalised and rounded to bf16 at insert (a2: v / |v|_2, norm in fp64, fp32 RN, bf16 RNE).
 * rows_dev: device [M x d] of dtype.  first_gid (optional, host): receives the first gid.
 * Synchronises the stream (validity check).  Errors: PAS_ERR_CAPACITY (shard full, nothing appended),
 * PAS_ERR_INVALID_ROWS (some row non-finite / zero-norm; nothing appended), PAS_ERR_ARG. */
pas_status pas_cache_load(pas_ctx* ctx, const void* rows_dev, pas_dtype dtype, int64_t M,
                          int64_t* first_gid, pas_stream stream);

/* NEXT f2, cache maintenance (
 * DESIGN.md R25-R27).  The store has G x max_rows_per_rank global slots; gid g lives on rank g % G.
 * A logical clock ticks once per routed batch, per insert call and per pas_cache_load; an entry's
 * stamp is the tick of its insertion or of the last batch that used it as a prompt's top-1 (every
 * routed batch stamps the top-1 of each valid prompt, on every rank).
 *
 * pas_cache_insert: n rows (device [n x d] of dtype, the SAME rows on every rank, n <= max_batch and
 * <= the global capacity).  Free slots at the end are used first (ascending gids); when they run
 * out, the entries smallest in (stamp, gid) are evicted -- exactly as many as needed -- and their
 * slots reused in ascending gid order.  gids_out (optional, device int32 [n]) receives the gid of
 * each row.  Rows are normalised and rounded like pas_cache_load (a2).  Synchronises the stream.
 * Errors: PAS_ERR_INVALID_ROWS (a row non-finite or zero-norm: nothing inserted, nothing evicted),
 * PAS_ERR_CAPACITY, PAS_ERR_ARG. */
pas_status pas_cache_insert(pas_ctx* ctx, const void* rows_dev, pas_dtype dtype, int64_t n,
                            int32_t* gids_out_dev, pas_stream stream);

/* The warm-up policy: insert the prompts of a routed batch that were served by vanilla
 * diffusion (K'_dev[p] == 0, device int32 [N], e.g. pas_route_out.K_prime) once their generations
 * complete, in prompt order, skipping invalid embeddings; emb_dev: the batch's embeddings [N x d].
 * gids_by_prompt_dev (optional, device int32 [N]): the new gid of each inserted prompt, -1 for the
 * others.  n_inserted (optional, host): how many.  Same eviction rule as pas_cache_insert.
 * Synchronises the stream.  Errors: PAS_ERR_CAPACITY, PAS_ERR_ARG. */
pas_status pas_cache_insert_vanilla(pas_ctx* ctx, const void* emb_dev, pas_dtype dtype, int64_t N,
                                    const int32_t* K_prime_dev, int32_t* gids_by_prompt_dev,
                                    int64_t* n_inserted, pas_stream stream);

/* Test hook: copy the first n LRU stamps (uint32, one per global slot) to stamps_dev. */
pas_status pas_cache_stamps(pas_ctx* ctx, uint32_t* stamps_dev, int64_t n, pas_stream stream);

/* Drop every cached row (global count back to 0).  Stream-ordered. */
pas_status pas_cache_clear(pas_ctx* ctx);

/* Rows in the store: global total (all ranks) and this rank's shard. */
pas_status pas_cache_size(const pas_ctx* ctx, int64_t* global_rows, int64_t* local_rows);

/* The optimal-K Selector's similarity bands (R8): K_levels[0..nK) strictly increasing,
 * K_levels[0] == 0, each < PAS_T_TOTAL; thresholds[0..nK-1) strictly increasing and finite.
 * A prompt with best similarity s1 gets level #{m : s1 >= thresholds[m]} (bands closed below).
 * Invalidates previously set fractions.  Errors: PAS_ERR_BANDS. */
pas_status pas_set_bands(pas_ctx* ctx, const int32_t* K_levels, int nK, const float* thresholds);

/* Degradation c(dK) for dK = 0..len-1 (Eq. 1's D(K',K) = c(K'-K) for K' > K, 0 otherwise; P:89 leaves
 * D's form open; R5, R6).  len must be PAS_T_TOTAL; c[0] == 0, finite, non-decreasing.
 *   - convex c (second differences >= -1e-12 (1 + |c|)): the route plan (a6) is the NW-corner
 *     coupling, the exact optimum under R7 (ties within 1e-9 relative -> min sum x dK^2);
 *   - any other c (NEXT f4, R37) must stay in [0, 1] (a quality loss): it is held as integers
 *     cI = round-half-even(c * 2^24) and the plan is the exact optimum of the integer transportation
 *     problem under (sum x cI, sum x dK^2) lexicographically, and among those the lexicographically
 *     greatest x in row-major order (one CTA, min-cost flow; pas_stats.plan_solver_iters).  D_Q is
 *     still Eq. 1 in fp64 on the real c; D_Q_LP is NaN (not computed).  Not with the forecast mode
 *     (its coupling plan is the optimum only for convex c).
 * Errors: PAS_ERR_DEGRADATION. */
pas_status pas_set_degradation(pas_ctx* ctx, const double* c_of_dK, int len);

/* Controller outputs for the next batches: F[nK] per-level load fractions (sum 1 +- 1e-9,
 * F >= 0), instance_level[W] the level index each serving instance runs at (1 <= W <= 64),
 * bstar >= 1 the optimal batch size ("2-4"), mode greedy (high load) / uniform (low load,
 * requires bstar == 1, "batch size of 1").  Requires pas_set_bands.
 * Errors: PAS_ERR_STATE, PAS_ERR_FRACTIONS, PAS_ERR_NO_INSTANCE, PAS_ERR_ARG. */
pas_status pas_set_fractions(pas_ctx* ctx, const double* F, const int32_t* instance_level, int W,
                             int bstar, pas_mode mode);

/* NEXT f1, forecast-driven streaming mode (R21-R24).
 * window > 0: from the next batch on, the Optimal-K Predictor is a ring buffer of the last `window`
 * optimal-K levels (fed with every routed batch, prompt order; empty = uniform forecast), the Route-
 * Plan P(K'|K) is the Eq. 1 optimum (monotone coupling, 2^-32 fixed point) of that forecast and F,
 * rebuilt every `replan_every`-th batch and whenever F changed, and every prompt draws its K' i.i.d.
 * from its plan row (Philox stream 3) instead of the exact per-batch integer plan.  Route-and-batch,
 * outputs and buckets are unchanged.  window == 0 returns to the exact mode.  Resets the window
 * (also reset by pas_set_bands).  Synchronises the device.  Requires pas_set_bands for window > 0.
 * Errors: PAS_ERR_ARG (window outside [0, PAS_MAX_FORECAST_WINDOW], replan_every < 1), PAS_ERR_STATE,
 * PAS_ERR_CUDA. */
pas_status pas_set_forecast(pas_ctx* ctx, int window, int replan_every);

/* NEXT f3, the stateful load-aware dispatcher (
 * DESIGN.md R28-R32).  service_us != NULL switches route-and-batch (a8) from the stateless packing
 * (R13 / R14) to per-instance queues kept on the device across batches: waiting prompts Q_w,
 * busy-until B_w, service time s_w per batch (service_us[w], 1..PAS_MAX_SERVICE_US), batch timeout
 * timeout_us (Delta, 0..PAS_MAX_TIME_US; SPEC's default 250000).  Time is integer microseconds.
 * Each routed batch arrives at the clock set by pas_set_clock (R28) and is dispatched atomically:
 *   - the form_batch events since the previous batch happen first (R30: an idle instance fires
 *     min(Q, b*) prompts when Q >= b* or its oldest prompt has waited Delta; busy for s_w);
 *   - greedy (R29): the longest queue below b* (ties: lowest id), else the instance whose next batch
 *     starts soonest, max(B_w, now) + floor(Q_w / b*) s_w (ties: lowest id); uniform: as R14;
 *   - slot (pas_route_out.slot) = the prompt's position in its instance's queue, counting the prompts
 *     still waiting from earlier batches (R31); batch lists: this batch's prompts per instance;
 *   - then idle instances fire at `now`.
 * W must equal pas_set_fractions' W and b* <= 64 while the dispatcher is on.  Resets the state
 * (empty queues, never busy, clock 0).  service_us == NULL turns it off.  Synchronous.
 * Errors: PAS_ERR_STATE (no fractions), PAS_ERR_ARG, PAS_ERR_CUDA. */
pas_status pas_set_dispatcher(pas_ctx* ctx, const int64_t* service_us, int W, int64_t timeout_us);

/* Arrival time (us) of the next routed batch: >= the previous batch's, <= PAS_MAX_TIME_US.  Batches
 * routed without a new pas_set_clock arrive at the same instant as the previous one.
 * Errors: PAS_ERR_STATE (dispatcher off), PAS_ERR_ARG. */
pas_status pas_set_clock(pas_ctx* ctx, int64_t now_us);

/* Load-mode switch (R32): utilisation u = lambda_rps / capacity with capacity =
 * sum_w bstar_high / s_w; uniform -> greedy when u > 0.8, greedy -> uniform when u < 0.7.  Sets the
 * mode and b* (bstar_high or 1) for the next batches; F and the instance levels are kept.
 * mode_out (optional) receives the mode.  Errors: PAS_ERR_STATE (dispatcher off), PAS_ERR_ARG. */
pas_status pas_set_load(pas_ctx* ctx, double lambda_rps, int bstar_high, pas_mode* mode_out);

/* Current dispatcher state (host arrays of W entries, each optional).  Synchronises the device.
 * Errors: PAS_ERR_STATE (dispatcher off), PAS_ERR_CUDA. */
pas_status pas_dispatcher_state(pas_ctx* ctx, int64_t* queue_len, int64_t* busy_until_us, int64_t* fired_prompts,
                                int64_t* fired_batches);

/* NEXT f4, the Resource Controller's Model Cache Assigner + Query Fraction Solver (PAPER.md P:88, P:207,
 * P:223; R33-R36), solved exactly on the GPU by enumerating all
 * C(W + nK - 1, nK - 1) assignments of W instances to the nK levels of pas_set_bands (11.2M for
 * W = 64, 6 levels; at most PAS_MAX_ASSIGNMENTS).  Inputs: lambda_rps arrival rate (>= 0), H[nK] the
 * forecast H_K (fractions; NULL = the f1 predictor window, which needs pas_set_forecast), service_us[nK]
 * the batch service time of a level-k instance at batch size bstar (us).  rate_k = bstar 1e6 / s_k;
 * a_k = 1 - sum_{K_i < K_k} H_i c(K_k - K_i) (the degradation of pas_set_degradation).  For each
 * assignment: served S = min(1, sum n_k rate_k / lambda), F = greedy fill of S by a_k descending,
 * quality q = sum F_k a_k; the optimum maximises (S, q) lexicographically (2^-40 grid), then prefers
 * the lexicographically largest n (instances at the slower, better levels).  out: host struct.  Uses the
 * context's last stream; synchronises.  Errors: PAS_ERR_STATE (no bands / no forecast for H == NULL),
 * PAS_ERR_ARG. */
#define PAS_MAX_ASSIGNMENTS (INT64_C(1) << 34)
typedef struct {
  int nK, W;
  int32_t n[PAS_MAX_LEVELS];                    /* instances per level */
  double F[PAS_MAX_LEVELS];                     /* load fractions, sum = served */
  double F_route[PAS_MAX_LEVELS];               /* F / served: the input of pas_set_fractions */
  double H[PAS_MAX_LEVELS];                     /* the forecast used */
  double served, quality;                       /* S and q of the optimum (R34) */
  int32_t instance_level[PAS_MAX_INSTANCES];    /* level of instance w (levels ascending) */
  int64_t candidates;                           /* assignments enumerated */
  float solve_ms;                               /* device time of the solve */
} pas_assignment;
pas_status pas_solve_assignment(pas_ctx* ctx, int W, double lambda_rps, const double* H, const int64_t* service_us,
                                int bstar, pas_assignment* out);

/* How pas_route_batch combines the ranks when world > 1:
 *   PAS_COLL_FOLDED (default): N1 ncclAllGather of every rank's [N x k] candidates, then every rank
 *     merges all N prompts and builds the full H_K itself -- the north_star's all-reduce of H_K is
 *     folded into the redundant merge (one collective per batch);
 *   PAS_COLL_EXPLICIT: N1, then each rank merges only its slice of ceil(N / G) prompts, N2
 *     ncclAllReduce of the slice H_K (+ flag counters), N3 ncclAllGather of the slice results (top-k,
 *     K, level, flags) in one NCCL group, then the same redundant K5..K7.
 * Outputs are byte-identical either way (R18, R19).  Errors: PAS_ERR_ARG. */
#define PAS_COLL_FOLDED 0
#define PAS_COLL_EXPLICIT 1
pas_status pas_set_collectives(pas_ctx* ctx, int mode);

/* Reset the Philox key and the batch sequence number (R18). */
pas_status pas_set_seed(pas_ctx* ctx, uint64_t seed, uint64_t batch_seq);

/* Route one batch (the hot path).  emb_dev: device [N x d] of dtype (16-byte aligned rows), the SAME
 * prompts on every rank.
 * out: device arrays, written in full on every rank.  N == 0 is a no-op; N > max_batch ->
 * PAS_ERR_CAPACITY.  Requires bands and fractions (PAS_ERR_STATE).  Enqueue-only (no host sync);
 * batch_seq increments on success.  world > 1 needs the NCCL communicator.  One batch in flight per
 * context (its workspace is reused).  The batch-varying state lives in device memory, so the whole
 * call can be replayed as a CUDA graph (pas_set_graph). */
pas_status pas_route_batch(pas_ctx* ctx, const void* emb_dev, pas_dtype dtype, int64_t N,
                           const pas_route_out* out, pas_stream stream);

/* CUDA-graph replay of pas_route_batch.  on != 0: the next pas_route_batch captures the
 * whole batch (K1 .. K7, and the NCCL collectives for world > 1) into a graph owned by the context and
 * every later call with the same (emb_dev, dtype, N, out pointers) replays it with one cudaGraphLaunch
 * -- one host call per batch instead of ~14 launches.  The batch-varying state (Philox batch_seq, the
 * LRU tick, the K2 epoch) lives in device memory and is advanced by the batch's own kernels, so a
 * replay is exactly the batch an eager call would run.  Any setter, cache load / insert / clear, or a
 * different pointer / N re-captures (the next call).  The forecast (f1) and dispatcher (f3) modes keep
 * per-batch host state and always run eagerly.  In graph mode pas_stats.stage_ms holds only the total
 * [6].  on == 0: eager launches (default).  Errors: PAS_ERR_STATE (poisoned). */
pas_status pas_set_graph(pas_ctx* ctx, int on);

/* Same, from HOST buffers: copies emb_host (should be pinned) to the device, routes, copies every
 * non-NULL array of out_host (host pointers, same shapes as pas_route_out) back, and synchronises.
 * This is the end-to-end public path (bench.py "e2e"). */
pas_status pas_route_batch_host(pas_ctx* ctx, const void* emb_host, pas_dtype dtype, int64_t N,
                                const pas_route_out* out_host, pas_stream stream);

/* Pipelined form of pas_route_batch_host for a stream of batches: enqueues the host→device copy of
 * emb_host on the context's H2D copy stream, the batch on `stream` (after that copy), and the copies of
 * every non-NULL array of out_host on the context's D2H copy stream (after the batch), and returns
 * without waiting, so the copies of one batch overlap the routing of its neighbours.  Two staging slots
 * (inputs and outputs on the device): a call blocks the host only until the batch issued two calls
 * earlier has delivered its outputs.  emb_host and out_host must stay valid (pinned for speed) until
 * that batch is done; the outputs are complete once `stream` has passed pas_route_host_end.
 * pas_route_host_begin(ctx, stream): the copy streams wait for all work enqueued on `stream` so far (a
 * timing or ordering fence before a pipelined run).  pas_route_host_end(ctx, stream): `stream` waits
 * for every batch issued so far, outputs included (does not block the host).  Same arguments and
 * errors as pas_route_batch_host; graph mode re-captures for each slot's buffers. */
pas_status pas_route_batch_host_async(pas_ctx* ctx, const void* emb_host, pas_dtype dtype, int64_t N,
                                      const pas_route_out* out_host, pas_stream stream);
pas_status pas_route_host_begin(pas_ctx* ctx, pas_stream stream);
pas_status pas_route_host_end(pas_ctx* ctx, pas_stream stream);

/* Split form of pas_route_batch for callers with their own transport (and for single-GPU tests of
 * the sharded path).  pas_route_local runs a1+a3+the intra-GPU part of a4 on this rank's shard and
 * writes cand_dev: device [N x topk] pairs {float score; int32 gid} (8 bytes each, score desc, gid asc,
 * padded (-inf, -1)).  pas_route_from_candidates takes S such blocks laid out [S][N][topk]
 * (e.g. the all-gather over ranks, S == world), merges them and runs a5..a8 for all N prompts,
 * using the validity flags of this context's last pas_route_local when it had the same N (otherwise
 * every prompt is valid; a caller marks an invalid prompt with an all-sentinel list, which yields
 * K = 0).  batch_seq increments here.  1 <= S <= 128. */
pas_status pas_route_local(pas_ctx* ctx, const void* emb_dev, pas_dtype dtype, int64_t N,
                           void* cand_dev, pas_stream stream);
pas_status pas_route_from_candidates(pas_ctx* ctx, const void* cand_dev, int S, int64_t N,
                                     const pas_route_out* out, pas_stream stream);

/* Plan and counters of the last routed batch (host struct).  Synchronises the context's last stream. */
pas_status pas_plan_stats(pas_ctx* ctx, pas_stats* out);

/* Stage-timing ring (bench.py): with slots > 0 every routed batch also records its 7 stage boundaries
 * into slot (batch index % slots), so per-batch device times of many back-to-back batches can be read
 * after the fact without a host sync per batch.  slots == 0 turns it off.  Synchronises the device.
 * pas_stage_ring_read: the last min(n, batches recorded, slots) batches, oldest first, as rows of 7
 * floats (ms): stages [0..5] as pas_stats.stage_ms, [6] total; *n_out receives the row count.
 * Synchronises on those batches.  Errors: PAS_ERR_ARG. */
#define PAS_MAX_RING 4096
pas_status pas_stage_ring(pas_ctx* ctx, int slots);
pas_status pas_stage_ring_read(pas_ctx* ctx, int n, float* ms, int* n_out);

/* Last error message of this context ("" if none).  ctx may be NULL (global errors, e.g. create). */
const char* pas_last_error(const pas_ctx* ctx);

/* Kernel launches the last pas_route_batch / pas_route_batch_host enqueued (for bench.py's
 * gpu_launches count). */
int pas_last_launch_count(const pas_ctx* ctx);

/* ---- test hooks (not part of the routing path) ---------------------------------------------- */
/* Runs a1 and the a3 GEMM with an epilogue that writes every raw score instead of the top-k:
 * scores_dev: device [N x local_rows] fp32 (local_rows = this rank's shard size).  For the GEMM's
 * element-wise parity test on small inputs only. */
pas_status pas_debug_scores(pas_ctx* ctx, const void* emb_dev, pas_dtype dtype, int64_t N, float* scores_dev,
                            pas_stream stream);

/* The bf16 rows K1 produced (a1 / a2, R11), for bit-exact checks against the oracle's quantisation:
 * pas_debug_qhat copies the first N rows of the prompt-side Q_hat written by the last pas_route_batch /
 * pas_route_local (device [N x d] bf16, out_dev caller-owned); pas_debug_store_rows copies this rank's
 * store rows [first_local_row, first_local_row + n) (local row r holds gid r * world + rank).
 * Stream-ordered copies.  Errors: PAS_ERR_ARG (range), PAS_ERR_STATE (no prompt normalised yet). */
pas_status pas_debug_qhat(pas_ctx* ctx, void* out_dev, int64_t N, pas_stream stream);
pas_status pas_debug_store_rows(pas_ctx* ctx, int64_t first_local_row, int64_t n, void* out_dev, pas_stream stream);

/* The K2 work schedule a batch of N prompts against M_local rows of width d would get in a context of
 * max_batch prompts (host logic only, no device; DESIGN.md 8 "K2 schedule").  out[9] receives:
 * R (cache ranges per prompt tile = sources of the merge), T (cache tiles per chunk; 0 = static
 * schedule), CS (chunk steps per range), MTg (prompt tiles per group), pair (1 = CTA-pair tile),
 * MT (prompt tiles of 128), NT (cache tiles), cand_cap (candidate rows: R * N <= cand_cap), and the
 * cache tile's rows (256, or 128 for the small-problem tile).
 * The PAS_K2_* experiment variables are read at each call here; a context reads them
 * once, at pas_create.  Errors: PAS_ERR_ARG. */
pas_status pas_debug_k2_schedule(int64_t N, int64_t M_local, int d, int64_t max_batch, int* out);

#ifdef __cplusplus
}
#endif
#endif /* PAS_H_ */
