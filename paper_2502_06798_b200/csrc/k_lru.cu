// f2 -- LRU maintenance of the approximate-cache store (R25-R27).
//
// Paper: the cache holds prior generations' states reused by prompt closeness (PAPER.md P:57,
// P:102); new entries come from vanilla generations; the store evicts LRU
// (SPEC S:144-147).  Every rank keeps the full stamp array (uint32 per global slot): routed
// batches touch the top-1 entry of every usable prompt (K4 writes stamp[g1] = tick, R26) and every
// rank sees all N merged lists, so the arrays stay identical without communication.
//
// Victims of an insert that finds n_evict fewer free slots than rows: the n_evict smallest
// (stamp, gid).  Radix select on the 32-bit stamp (4 passes of 8 bits: per-CTA shared histograms,
// one global atomic per non-zero bin, one warp picks the digit) gives the threshold stamp T and how
// many entries r of stamp T are needed; then a gid-ordered compaction (per-tile counts of "below"
// and "equal", a device-wide scan, per-tile emit) writes the victims in ascending gid order.
// Finally k_store_rows copies the staged (K1-normalised) bf16 rows into their slots on the rank that
// owns them and stamps them.  O(M) per insert call, off the routing path.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int HIST_THREADS = 256;
constexpr int CT_THREADS = 256;
constexpr int CT_PER = 16;
constexpr int CT_TILE = CT_THREADS * CT_PER;   // gids per compaction tile

__global__ void k_lru_init(LruSel* sel, int32_t k) {
  pdl_entry();
  if (threadIdx.x == 0) {
    sel->prefix = 0;
    sel->mask = 0;
    sel->k = k;
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sel->hist[i] = 0;
}

__global__ void __launch_bounds__(HIST_THREADS) k_lru_hist(const uint32_t* __restrict__ stamps, int64_t M,
                                                           int shift, LruSel* __restrict__ sel) {
  pdl_entry();
  __shared__ int32_t h[256];
  for (int i = threadIdx.x; i < 256; i += HIST_THREADS) h[i] = 0;
  __syncthreads();
  const uint32_t prefix = sel->prefix, mask = sel->mask;
  const int64_t stride = (int64_t)gridDim.x * HIST_THREADS;
  for (int64_t g = (int64_t)blockIdx.x * HIST_THREADS + threadIdx.x; g < M; g += stride) {
    const uint32_t s = stamps[g];
    if ((s & mask) == prefix) atomicAdd(&h[(s >> shift) & 0xFFu], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += HIST_THREADS)
    if (h[i]) atomicAdd(&sel->hist[i], h[i]);
}

// One warp: the digit whose cumulative count reaches k; k becomes the rank inside that digit.
__global__ void __launch_bounds__(32) k_lru_find(LruSel* __restrict__ sel, int shift) {
  pdl_entry();
  const int lane = threadIdx.x;
  const int32_t k = sel->k;
  int32_t c[8], sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = sel->hist[lane * 8 + i];
    sum += c[i];
  }
  int32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int32_t before = incl - sum;
  int digit = -1, kk = 0;
  if (before < k && k <= incl) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (digit < 0 && k <= before + c[i]) {
        digit = lane * 8 + i;
        kk = k - before;
      }
      before += c[i];
    }
  }
  const unsigned who = __ballot_sync(0xffffffffu, digit >= 0);
  const int src = __ffs(who) - 1;
  digit = __shfl_sync(0xffffffffu, digit, src);
  kk = __shfl_sync(0xffffffffu, kk, src);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) sel->hist[lane * 8 + i] = 0;
  if (lane == 0) {
    sel->prefix |= (uint32_t)digit << shift;
    sel->mask |= 0xFFu << shift;
    sel->k = kk;
  }
}

// Per tile of gids: how many have stamp < T and stamp == T (T = sel->prefix after 4 passes).
__global__ void __launch_bounds__(CT_THREADS) k_lru_tile_count(const uint32_t* __restrict__ stamps, int64_t M,
                                                               const LruSel* __restrict__ sel, int ntiles,
                                                               int32_t* __restrict__ counts /*[2][ntiles]*/) {
  pdl_entry();
  __shared__ int32_t red[2][CT_THREADS / 32];
  const uint32_t T = sel->prefix;
  const int64_t g0 = (int64_t)blockIdx.x * CT_TILE + (int64_t)threadIdx.x * CT_PER;
  int below = 0, equal = 0;
#pragma unroll
  for (int e = 0; e < CT_PER; ++e) {
    if (g0 + e < M) {
      const uint32_t s = stamps[g0 + e];
      below += s < T;
      equal += s == T;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    below += __shfl_xor_sync(0xffffffffu, below, o);
    equal += __shfl_xor_sync(0xffffffffu, equal, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = below;
    red[1][w] = equal;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = 0, q = 0;
    for (int i = 0; i < CT_THREADS / 32; ++i) {
      b += red[0][i];
      q += red[1][i];
    }
    counts[blockIdx.x] = b;
    counts[ntiles + blockIdx.x] = q;
  }
}

// Victim position of gid g = #{g' < g : stamp < T} + min(#{g' < g : stamp == T}, r).
__global__ void __launch_bounds__(CT_THREADS) k_lru_emit(const uint32_t* __restrict__ stamps, int64_t M,
                                                         const LruSel* __restrict__ sel, int ntiles,
                                                         const int32_t* __restrict__ scanned,
                                                         int32_t* __restrict__ victims) {
  pdl_entry();
  __shared__ uint32_t wsum[CT_THREADS / 32];
  const uint32_t T = sel->prefix;
  const int32_t r = sel->k;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t g0 = (int64_t)blockIdx.x * CT_TILE + (int64_t)threadIdx.x * CT_PER;
  uint32_t s[CT_PER];
  uint32_t mine = 0;   // below in bits 0..15, equal in bits 16..31 (<= 4096 each)
#pragma unroll
  for (int e = 0; e < CT_PER; ++e) {
    s[e] = g0 + e < M ? stamps[g0 + e] : 0xFFFFFFFFu;
    mine += (g0 + e < M) ? ((s[e] < T) ? 1u : (s[e] == T ? 0x10000u : 0u)) : 0u;
  }
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (int i = 0; i < w; ++i) wpre += wsum[i];
  uint32_t run = wpre + incl - mine;
  int32_t below = scanned[blockIdx.x] + (int32_t)(run & 0xFFFFu);
  int32_t equal = scanned[ntiles + blockIdx.x] - scanned[ntiles] + (int32_t)(run >> 16);
#pragma unroll
  for (int e = 0; e < CT_PER; ++e) {
    if (g0 + e >= M) break;
    if (s[e] < T) {
      victims[below + min(equal, r)] = (int32_t)(g0 + e);
      ++below;
    } else if (s[e] == T) {
      if (equal < r) victims[below + equal] = (int32_t)(g0 + e);
      ++equal;
    }
  }
}

// gids[i]: the first n_append rows append at gid first_new + i, the rest take victims[i - n_append].
// This rank copies staged row src[i] (or i) into its local slot gid / G; every rank stamps the gid.
__global__ void k_store_rows(const __nv_bfloat16* __restrict__ staged, const int32_t* __restrict__ src, int64_t n,
                             int64_t n_append, int64_t first_new, const int32_t* __restrict__ victims, int d, int G,
                             int rank, __nv_bfloat16* __restrict__ store, uint32_t* __restrict__ stamps, uint32_t tick,
                             int32_t* __restrict__ gids_out, int32_t* __restrict__ gids_by_prompt) {
  pdl_entry();
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int32_t g = i < n_append ? (int32_t)(first_new + i) : victims[i - n_append];
  const int64_t row = src ? src[i] : i;
  if (threadIdx.x == 0) {
    stamps[g] = tick;
    if (gids_out) gids_out[i] = g;
    if (gids_by_prompt) gids_by_prompt[row] = g;
  }
  if (g % G != rank) return;
  const uint4* a = reinterpret_cast<const uint4*>(staged + row * d);
  uint4* b = reinterpret_cast<uint4*>(store + (int64_t)(g / G) * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) b[c] = a[c];
}

__global__ void k_fill_u32(uint32_t* __restrict__ a, int64_t n, uint32_t v) {
  pdl_entry();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

// Compaction of the prompts to insert (R25): take[p] = valid && K'[p] == 0, in prompt order.
__global__ void __launch_bounds__(CT_THREADS) k_vanilla_count(const int32_t* __restrict__ K_prime,
                                                              const uint8_t* __restrict__ pflags, int64_t N,
                                                              int32_t* __restrict__ counts) {
  pdl_entry();
  __shared__ int32_t red[CT_THREADS / 32];
  const int64_t p0 = (int64_t)blockIdx.x * CT_TILE + (int64_t)threadIdx.x * CT_PER;
  int c = 0;
#pragma unroll
  for (int e = 0; e < CT_PER; ++e)
    if (p0 + e < N) c += (K_prime[p0 + e] == 0 && !(pflags[p0 + e] & PAS_FLAG_INVALID));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < CT_THREADS / 32; ++i) t += red[i];
    counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(CT_THREADS) k_vanilla_emit(const int32_t* __restrict__ K_prime,
                                                             const uint8_t* __restrict__ pflags, int64_t N,
                                                             const int32_t* __restrict__ scanned, int ntiles,
                                                             int32_t* __restrict__ idx, int32_t* __restrict__ count,
                                                             int32_t* __restrict__ gids_by_prompt) {
  pdl_entry();
  __shared__ int32_t wsum[CT_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t p0 = (int64_t)blockIdx.x * CT_TILE + (int64_t)threadIdx.x * CT_PER;
  bool take[CT_PER];
  int mine = 0;
#pragma unroll
  for (int e = 0; e < CT_PER; ++e) {
    take[e] = p0 + e < N && K_prime[p0 + e] == 0 && !(pflags[p0 + e] & PAS_FLAG_INVALID);
    mine += take[e];
    if (p0 + e < N && gids_by_prompt) gids_by_prompt[p0 + e] = -1;
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int pos = scanned[blockIdx.x] + incl - mine;
  for (int i = 0; i < w; ++i) pos += wsum[i];
#pragma unroll
  for (int e = 0; e < CT_PER; ++e)
    if (take[e]) idx[pos++] = (int32_t)(p0 + e);
  if (blockIdx.x == ntiles - 1 && threadIdx.x == CT_THREADS - 1) *count = pos;   // last thread: total
}

}  // namespace

int lru_tiles(int64_t M) { return (int)((M + CT_TILE - 1) / CT_TILE); }

cudaError_t launch_lru_victims(const uint32_t* stamps, int64_t M, int32_t n_evict, LruSel* sel, int32_t* counts,
                               int32_t* scanned, int32_t* scan_tmp, int32_t* victims, cudaStream_t st) {
  launch_pdl(k_lru_init, 1, 256, 0, st, sel, n_evict);
  int64_t blocks = (M + HIST_THREADS - 1) / HIST_THREADS;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  for (int shift = 24; shift >= 0; shift -= 8) {
    launch_pdl(k_lru_hist, (unsigned)blocks, HIST_THREADS, 0, st, stamps, M, shift, sel);
    launch_pdl(k_lru_find, 1, 32, 0, st, sel, shift);
  }
  const int ntiles = lru_tiles(M);
  launch_pdl(k_lru_tile_count, ntiles, CT_THREADS, 0, st, stamps, M, (const LruSel*)sel, ntiles, counts);
  int launches = 0;
  cudaError_t e = launch_exclusive_scan(counts, scanned, 2 * ntiles, scan_tmp, st, &launches);
  if (e != cudaSuccess) return e;
  launch_pdl(k_lru_emit, ntiles, CT_THREADS, 0, st, stamps, M, (const LruSel*)sel, ntiles, (const int32_t*)scanned,
             victims);
  return cudaGetLastError();
}

cudaError_t launch_store_rows(const __nv_bfloat16* staged, const int32_t* src, int64_t n, int64_t n_append,
                              int64_t first_new, const int32_t* victims, int d, int G, int rank,
                              __nv_bfloat16* store, uint32_t* stamps, uint32_t tick, int32_t* gids_out,
                              int32_t* gids_by_prompt, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  launch_pdl(k_store_rows, (unsigned)n, 96, 0, st, staged, src, n, n_append, first_new, victims, d, G, rank, store,
             stamps, tick, gids_out, gids_by_prompt);
  return cudaGetLastError();
}

cudaError_t launch_fill_u32(uint32_t* a, int64_t n, uint32_t v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  launch_pdl(k_fill_u32, (unsigned)blocks, 256, 0, st, a, n, v);
  return cudaGetLastError();
}

cudaError_t launch_vanilla_compact(const int32_t* K_prime, const uint8_t* pflags, int64_t N, int32_t* counts,
                                   int32_t* scanned, int32_t* scan_tmp, int32_t* idx, int32_t* count,
                                   int32_t* gids_by_prompt, cudaStream_t st) {
  const int ntiles = lru_tiles(N);
  launch_pdl(k_vanilla_count, ntiles, CT_THREADS, 0, st, K_prime, pflags, N, counts);
  int launches = 0;
  cudaError_t e = launch_exclusive_scan(counts, scanned, ntiles, scan_tmp, st, &launches);
  if (e != cudaSuccess) return e;
  launch_pdl(k_vanilla_emit, ntiles, CT_THREADS, 0, st, K_prime, pflags, N, (const int32_t*)scanned, ntiles, idx,
             count, gids_by_prompt);
  return cudaGetLastError();
}

}  // namespace pas
