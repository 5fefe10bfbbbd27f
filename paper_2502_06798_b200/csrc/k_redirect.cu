// K6 -- redirection sampling: every prompt gets its K' from the Route-Plan.
//
// Exact-count form (R3): within optimal-K class i, prompts are ordered by a 60-bit Philox
// key kappa_p (ties by prompt index); the prompt of class rank r is served at K'_j for
// X_i[j-1] <= r < X_i[j] (X_i = inclusive prefix of row i of the plan x), so exactly x_ij prompts of
// class i go to level j and the ranks are a uniformly random permutation of the class (R18: kappa
// depends only on seed, batch_seq, p -- not on the router GPU count).
//
// Selection instead of sorting: K'_p only depends on how many of the class's nK - 1 split ranks
// X_i[j] lie at or below rank_p, so only the split elements have to be located -- order statistics,
// not a sort.  Two levels:
//   k6_hist    kappa = Philox(p) (stored, 8 B), histogram of (class, top kb bits of kappa) in global
//              atomics (kb = ceil(log2 N) - 6, <= 18: on average <= 64 prompts per bucket of a full
//              class);
//   k6_chunks + k6_bounds  per class: chunk sums of the bucket counts (many CTAs, coalesced), then
//              the bucket holding each split rank and the split's rank inside it (a warp scan over
//              one chunk); each distinct split bucket gets a candidate list;
//   k6_assign  every prompt counts the split buckets below its own bucket -- that IS its K' -- unless
//              its bucket holds a split, then it appends (kappa, p) to that bucket's list;
//   k6_resolve one CTA per split bucket ranks its few entries exactly by (kappa, p) in shared memory.
// Per prompt: level 1 B read twice, kappa 8 B written + read, K' 4 B + K7 class 1 B written; plus one
// L2 atomic.  The previous full counting-sort ranking (scatter + in-bucket rank of all N entries)
// moved 53 B per prompt through scattered accesses (8.8 ms at 64M prompts).
//
// Windowed split search (the default since round 2; the histogram path above is its exact fallback):
// kappa is uniform, so the kappa of the prompt at class rank X lies, with probability 1 - 1e-15, in a
// window of +- 8 sd around the X-th order statistic of h uniforms (K5 computes the windows, merged into
// zones: pas_internal.cuh DevPlan).  A prompt whose kappa falls OUTSIDE every zone of its class has its
// K' fixed by the zones below it alone -- every split in them has a smaller kappa -- so
//   k6_fused   one streaming pass, 4,096 prompts per CTA (K7's tiles): Philox, zone test, K' and the K7
//              class for the outside prompts, (kappa, p) appended to the zone's list for the inside ones
//              (~8 sqrt(h) per split: 0.1 % at 64M prompts), per-(class, gap) counts, and K7's per-tile
//              class counts (so k_cls_count only runs on the fallback);
//   k6_zone    one CTA per zone: the zone's class prompts below it (gap counts + lower zones), each
//              split's rank inside the zone located through a 2,048-bucket histogram and an exact
//              (kappa, p) selection in its bucket, then every entry's K', class and tile count.
// If a split rank falls outside its zone (or a list overflows, or there are > 32 splits) the
// flag DevPlan::k6_fallback is set and the histogram path below (gated kernels, no-ops otherwise)
// recomputes every K' exactly.  Per prompt: level 1 B read, K' 4 B + class 1 B written: 6 B.
#include "pas_internal.cuh"
#include "philox.cuh"

namespace pas {
namespace {

constexpr int RT = 256;
#ifndef PAS_K6_GRIDCAP
#define PAS_K6_GRIDCAP 1   // k6_assign: grid capped at 8 CTAs per SM (grid-stride); 0: uncapped
#endif
constexpr int kSmemList = 2048;   // k6_resolve: entries staged in shared memory (else read from L2)
// The windowed split search serves N >= kWindowMinN; below, its fixed launch cost (fused pass, zone
// kernels, gated fallback launches) exceeds what it saves, and the exact histogram path runs alone.

__device__ __forceinline__ bool entry_less(uint64_t ka, int32_t pa, uint64_t kb, int32_t pb) {
  return ka < kb || (ka == kb && pa < pb);
}

__device__ __forceinline__ uint32_t top_bits(uint64_t kappa, int kb) {
  return kb ? (uint32_t)(kappa >> (60 - kb)) : 0u;
}

// K' level j of prompt p: K' value and the route-and-batch class (K' level in greedy mode, the
// instance I_j[(u n_j) >> 32] in uniform mode)
__device__ __forceinline__ void emit(const RouteParams& P, const int* grid, const DevPlan* __restrict__ plan,
                                     int64_t p, int j, int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7) {
  K_prime[p] = grid[j];
  if (P.mode == PAS_UNIFORM) {
    const uint4 w = philox_stream(P.seed, batch_seq_of(P), (uint32_t)p, kStreamUniform);
    const uint32_t nj = (uint32_t)plan->n_inst[j];
    cls7[p] = (uint8_t)plan->inst_list[j][(uint32_t)(((uint64_t)w.x * nj) >> 32)];
  } else {
    cls7[p] = (uint8_t)j;
  }
}

// Fallback gate: the histogram kernels run only when the windowed pass could not decide every prompt.
__device__ __forceinline__ bool gated_off(const int* gate) {
  return gate && *reinterpret_cast<const volatile int*>(gate) == 0;
}

__global__ void __launch_bounds__(RT) k6_zero(const int* __restrict__ gate, int32_t* __restrict__ a, int64_t n,
                                              int32_t* __restrict__ b, int nb) {
  pdl_entry();
  if (gated_off(gate)) return;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT) a[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < nb) b[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(RT) k6_hist(const uint8_t* __restrict__ level, const __grid_constant__ RouteParams P,
                                              const int* __restrict__ gate, uint64_t* __restrict__ key,
                                              int32_t* __restrict__ hist) {
  pdl_entry();
  if (gated_off(gate)) return;   // a capped grid (grid-stride): a gated-off launch costs ~a microsecond
  const uint64_t bseq = batch_seq_of(P);
  for (int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x; p < P.N; p += (int64_t)gridDim.x * RT) {
    const uint4 w = philox_stream(P.seed, bseq, (uint32_t)p, kStreamRedirect);
    const uint64_t kappa = (((uint64_t)w.y << 32) | w.x) >> 4;
    key[p] = kappa;
    atomicAdd(&hist[((uint32_t)level[p] << P.kb) | top_bits(kappa, P.kb)], 1);
  }
}

// Per (class, chunk of kChunks) sums of the bucket counts, coalesced, many CTAs.
constexpr int kChunks = 256;
__global__ void __launch_bounds__(RT) k6_chunks(const __grid_constant__ RouteParams P, const int* __restrict__ gate,
                                                const int32_t* __restrict__ hist, int32_t* __restrict__ csum) {
  pdl_entry();
  if (gated_off(gate)) return;
  __shared__ int32_t ws[RT / 32];
  const int i = blockIdx.x / kChunks, c = blockIdx.x % kChunks;
  const int nb = 1 << P.kb, len = (nb + kChunks - 1) / kChunks;
  const int c0 = c * len, c1 = c0 + len < nb ? c0 + len : nb;
  const int32_t* hc = hist + ((int64_t)i << P.kb);
  int s = 0;
  for (int b = c0 + threadIdx.x; b < c1; b += RT) s += hc[b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < RT / 32; ++w) t += ws[w];
    csum[blockIdx.x] = t;
  }
}

// One CTA per class: the chunk holding each split rank (scan of the chunk sums), then one warp per
// split walks that chunk 32 buckets at a time (warp scan) to the bucket and the split's rank in it.
__global__ void __launch_bounds__(RT) k6_bounds(const __grid_constant__ RouteParams P, const DevPlan* __restrict__ plan,
                                                const int32_t* __restrict__ hist, const int32_t* __restrict__ csum,
                                                K6Bounds* __restrict__ bnd, K6List* __restrict__ lists,
                                                int32_t* __restrict__ used, const int* __restrict__ gate) {
  pdl_entry();
  if (gated_off(gate)) return;
  __shared__ int32_t cex[kChunks + 1];
  __shared__ int32_t sb[kMaxLevels], so[kMaxLevels];
  const int i = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int nb = 1 << P.kb, len = (nb + kChunks - 1) / kChunks;
  const int32_t* hc = hist + ((int64_t)i << P.kb);
  {   // exclusive scan of the class's kChunks chunk sums (one per thread: warp scans + warp totals)
    static_assert(kChunks == RT, "one chunk sum per thread");
    __shared__ int32_t wtot[RT / 32];
    const int v = csum[i * kChunks + t];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wtot[w] = incl;
    __syncthreads();
    int before = 0;
    for (int q = 0; q < w; ++q) before += wtot[q];
    cex[t] = before + incl - v;
    if (t == RT - 1) cex[kChunks] = before + incl;
  }
  if (t < kMaxLevels) sb[t] = INT32_MAX;
  __syncthreads();
  const int h = plan->h[i];
  for (int j = w; j + 1 < P.nK; j += RT / 32) {   // split rank X_i[j]: the first prompt of group j + 1
    const int X = plan->X[i][j];
    if (X >= h) continue;                          // no such prompt
    int c = 0;   // the chunk holding rank X: the last c with cex[c] <= X (binary search, cex ascending)
    for (int step = kChunks / 2; step > 0; step >>= 1)
      if (c + step < kChunks && cex[c + step] <= X) c += step;
    const int c0 = c * len, c1 = c0 + len < nb ? c0 + len : nb;
    int run = cex[c];
    for (int base = c0; base < c1; base += 32) {   // 32 buckets at a time, warp scan
      const int v = base + lane < c1 ? hc[base + lane] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (run + tot > X) {
        const unsigned hit = __ballot_sync(0xffffffffu, run + incl > X);
        const int L = __ffs(hit) - 1;
        if (lane == L) {
          sb[j] = base + L;
          so[j] = X - (run + incl - v);
        }
        break;
      }
      run += tot;
    }
  }
  __syncthreads();
  if (t == 0) {
    int last_bucket = -1, id = -1;
    for (int j = 0; j + 1 < P.nK; ++j) {
      const int b = sb[j];
      bnd->bucket[i][j] = b;
      bnd->off[i][j] = so[j];
      if (b == INT32_MAX) {
        bnd->list[i][j] = -1;
        continue;
      }
      if (b != last_bucket) {   // one candidate list per distinct split bucket (splits are sorted)
        const int cnt = hc[b];
        id = atomicAdd(&used[0], 1);
        K6List L;
        L.cls = i;
        L.bucket = b;
        L.cnt = cnt;
        L.base = atomicAdd(&used[1], cnt);
        L.fill = 0;
        L.below = j;             // splits in lower buckets of the class
        lists[id] = L;
        last_bucket = b;
      }
      bnd->list[i][j] = id;
    }
  }
}

__global__ void __launch_bounds__(RT) k6_assign(const uint8_t* __restrict__ level, const uint64_t* __restrict__ key,
                                                const __grid_constant__ RouteParams P, const DevPlan* __restrict__ plan,
                                                const K6Bounds* __restrict__ bnd, K6List* __restrict__ lists,
                                                KeyEntry* __restrict__ cand, int32_t* __restrict__ K_prime,
                                                uint8_t* __restrict__ cls7, const int* __restrict__ gate) {
  pdl_entry();
  if (gated_off(gate)) return;
  __shared__ int32_t sb[kMaxLevels][kMaxLevels], sl[kMaxLevels][kMaxLevels];
  __shared__ int grid_s[kMaxLevels];
  if (threadIdx.x < kMaxLevels) grid_s[threadIdx.x] = P.grid[threadIdx.x];
  for (int e = threadIdx.x; e < P.nK * kMaxLevels; e += RT) {   // once per (persistent) CTA
    const int i = e / kMaxLevels, j = e % kMaxLevels;
    sb[i][j] = j + 1 < P.nK ? bnd->bucket[i][j] : INT32_MAX;
    sl[i][j] = j + 1 < P.nK ? bnd->list[i][j] : -1;
  }
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x; p < P.N; p += (int64_t)gridDim.x * RT) {
    const int i = level[p];
    const uint64_t kappa = key[p];
    const int b = (int)top_bits(kappa, P.kb);
    int below = 0, list = -1;
    for (int j = 0; j + 1 < P.nK; ++j) {
      below += sb[i][j] < b;
      if (sb[i][j] == b) list = sl[i][j];
    }
    if (list < 0) {
      emit(P, grid_s, plan, p, below, K_prime, cls7);
      continue;
    }
    K6List* L = lists + list;
    const int slot = atomicAdd(&L->fill, 1);
    cand[L->base + slot] = KeyEntry{kappa, (int32_t)p, 0};
  }
}

__global__ void __launch_bounds__(RT) k6_resolve(const __grid_constant__ RouteParams P, const DevPlan* __restrict__ plan,
                                                 const K6Bounds* __restrict__ bnd, const K6List* __restrict__ lists,
                                                 const int32_t* __restrict__ used, const KeyEntry* __restrict__ cand,
                                                 int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7,
                                                 const int* __restrict__ gate) {
  pdl_entry();
  if (gated_off(gate)) return;
  __shared__ uint64_t sk[kSmemList];
  __shared__ int32_t sp[kSmemList];
  __shared__ int grid_s[kMaxLevels];
  if (threadIdx.x < kMaxLevels) grid_s[threadIdx.x] = P.grid[threadIdx.x];
  if ((int)blockIdx.x >= used[0]) return;
  const K6List L = lists[blockIdx.x];
  const KeyEntry* E = cand + L.base;
  const bool staged = L.cnt <= kSmemList;
  if (staged)
    for (int e = threadIdx.x; e < L.cnt; e += RT) {
      sk[e] = E[e].key;
      sp[e] = E[e].p;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < L.cnt; e += RT) {
    const uint64_t k = staged ? sk[e] : E[e].key;
    const int32_t p = staged ? sp[e] : E[e].p;
    int r = 0;   // rank inside the bucket by (kappa, p)
    for (int f = 0; f < L.cnt; ++f)
      r += staged ? entry_less(sk[f], sp[f], k, p) : entry_less(E[f].key, E[f].p, k, p);
    int j = L.below;
    for (int q = 0; q + 1 < P.nK; ++q)
      j += (bnd->bucket[L.cls][q] == L.bucket && r >= bnd->off[L.cls][q]) ? 1 : 0;
    emit(P, grid_s, plan, p, j, K_prime, cls7);
  }
}

// ---- windowed split search -----------------------------------------------------------------------
constexpr int FT = 256;                 // k6_fused threads; 16 consecutive prompts each = one K7 tile
constexpr int FPER = 16;
constexpr int kSlots = kMaxLevels + kMaxZones;   // (class, gap) slots

// Per prompt: Philox, then the (class, gap) slot.  A coarse table per class (256 buckets of the top 8
// kappa bits) gives the gap of every bucket no zone touches (zones cover ~0.1 % of kappa space), so
// almost every prompt resolves its slot with one shared load; the rest walk the class's zones.  Per
// slot: K' and (greedy) the K7 class are table look-ups.  Counters: private byte columns in shared
// memory (the column is the thread: no atomics, no conflicts); greedy class counts are the slot sums.
constexpr int kCoarseBits = 8;
template <int NCLS>
__global__ void __launch_bounds__(FT) k6_fused(const uint8_t* __restrict__ level, const __grid_constant__ RouteParams P,
                                               DevPlan* __restrict__ plan, KeyEntry* __restrict__ cand,
                                               int32_t* __restrict__ K_prime, uint8_t* __restrict__ cls7,
                                               int32_t* __restrict__ blk_counts, int ntiles) {
  constexpr bool UNIFORM = NCLS > kMaxLevels;
  pdl_entry();
  __shared__ uint64_t zlo[kMaxZones], zhi[kMaxZones];
  __shared__ int zcap[kMaxZones], zbase[kMaxZones];
  __shared__ int cinfo[kMaxLevels];                    // zone0 | nzone << 8 | slot0 << 16
  __shared__ int slotK[kSlots];                        // K' value of a prompt in the slot
  __shared__ uint8_t slotJ[kSlots];                    // its K' level (the greedy K7 class)
  __shared__ uint8_t coarse[kMaxLevels][1 << kCoarseBits];   // gap of a zone-free bucket, else 0xFF
  __shared__ uint8_t gcol[kSlots][FT];                 // (class, gap) counts per thread (<= 16 each)
  __shared__ uint8_t ccol[UNIFORM ? NCLS : 1][FT];     // uniform: K7 class (instance) counts per thread
  __shared__ int csum[NCLS];
  const int t = threadIdx.x;
  const int nK = P.nK;
  if (t < kMaxZones) {
    zlo[t] = plan->z_lo[t];
    zhi[t] = plan->z_hi[t];
    zcap[t] = plan->z_cap[t];
    zbase[t] = plan->z_base[t];
  }
  if (t < nK) {
    const int i = t, z0 = plan->cls_zone0[i], nz = plan->cls_nzone[i], s0 = plan->cls_slot0[i];
    cinfo[i] = z0 | (nz << 8) | (s0 << 16);
    for (int g = 0; g <= nz; ++g) {   // gap g: below zone g (or above all zones)
      const int j = g < nz ? plan->z_jbelow[z0 + g] : plan->cls_jtot[i];
      slotK[s0 + g] = P.grid[j];
      slotJ[s0 + g] = (uint8_t)j;
    }
  }
  for (int q = 0; q < kSlots; ++q) gcol[q][t] = 0;
  if (UNIFORM)
    for (int q = 0; q < NCLS; ++q) ccol[q][t] = 0;
  if (t < NCLS) csum[t] = 0;
  __syncthreads();
  for (int e = t; e < nK << kCoarseBits; e += FT) {   // coarse buckets: gap, or 0xFF if a zone touches it
    const int i = e >> kCoarseBits, b = e & ((1 << kCoarseBits) - 1);
    const uint64_t blo = (uint64_t)b << (60 - kCoarseBits), bhi = blo + (1ull << (60 - kCoarseBits));
    const int ci = cinfo[i], z0 = ci & 0xFF, nz = (ci >> 8) & 0xFF;
    int g = 0;
    bool touched = false;
    for (int z = z0; z < z0 + nz; ++z) {
      if (zhi[z] <= blo) ++g;
      else if (zlo[z] < bhi) touched = true;
    }
    coarse[i][b] = touched ? 0xFF : (uint8_t)g;
  }
  __syncthreads();
  const uint64_t bseq = batch_seq_of(P);
  // the tile's prompts in warp-coalesced order: p = tile base + e * 256 + t
  const int64_t p0 = (int64_t)blockIdx.x * (FT * FPER) + t;
  bool overflow = false;
  auto one = [&](int64_t p) {
    const int i = __ldg(level + p);
    const uint4 w = philox_stream(P.seed, bseq, (uint32_t)p, kStreamRedirect);
    const uint64_t kappa = (((uint64_t)w.y << 32) | w.x) >> 4;
    const int ci = cinfo[i];
    int g = coarse[i][(int)(kappa >> (60 - kCoarseBits))];
    if (g == 0xFF) {   // a bucket a zone touches: walk the class's zones
      const int z0 = ci & 0xFF, nz = (ci >> 8) & 0xFF;
      int z = -1;
      for (g = 0; g < nz; ++g) {
        if (kappa < zlo[z0 + g]) break;
        if (kappa < zhi[z0 + g]) {
          z = z0 + g;
          break;
        }
      }
      if (z >= 0) {
        const int slot = atomicAdd(&plan->z_fill[z], 1);
        PAS_CHECK(zbase[z] + zcap[z] <= P.N, "K6 zone list beyond N");
        if (slot < zcap[z]) cand[zbase[z] + slot] = KeyEntry{kappa, (int32_t)p, 0};
        else overflow = true;
        return;
      }
    }
    const int slot = (ci >> 16) + g;
    PAS_CHECK(i < nK && slot < kSlots, "K6 gap slot");
    ++gcol[slot][t];
    K_prime[p] = slotK[slot];
    if (UNIFORM) {   // the instance I_j[(u n_j) >> 32]
      const int j = slotJ[slot];
      const uint4 u = philox_stream(P.seed, bseq, (uint32_t)p, kStreamUniform);
      const int c = plan->inst_list[j][(uint32_t)(((uint64_t)u.x * (uint32_t)plan->n_inst[j]) >> 32)];
      cls7[p] = (uint8_t)c;
      ++ccol[c][t];
    } else {
      cls7[p] = slotJ[slot];
    }
  };
  if ((int64_t)(blockIdx.x + 1) * (FT * FPER) <= P.N) {   // a full tile: no bounds checks
#pragma unroll 4
    for (int e = 0; e < FPER; ++e) one(p0 + (int64_t)e * FT);
  } else {
    for (int e = 0; e < FPER && p0 + (int64_t)e * FT < P.N; ++e) one(p0 + (int64_t)e * FT);
  }
  if (overflow) plan->k6_fallback = 1;
  __syncthreads();
  // column sums: one warp per counter row; (class, gap) totals to the plan, class totals to K7's tile
  const int lane = t & 31, wp = t >> 5;
  const int nslots = (cinfo[nK - 1] >> 16) + ((cinfo[nK - 1] >> 8) & 0xFF) + 1;
  const int nrows = nslots + (UNIFORM ? P.W : 0);
  for (int q = wp; q < nrows; q += FT / 32) {
    const uint8_t* row = q < nslots ? gcol[q] : ccol[UNIFORM ? q - nslots : 0];
    int sum = 0;
#pragma unroll
    for (int r = 0; r < FT / 32; ++r) sum += row[lane + 32 * r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) {
      if (q < nslots) {
        atomicAdd(&plan->gapcnt[q], sum);
        if (!UNIFORM) atomicAdd(&csum[slotJ[q]], sum);
      } else {
        csum[q - nslots] = sum;
      }
    }
  }
  __syncthreads();
  const int nC = UNIFORM ? P.W : nK;
  if (t < nC) blk_counts[(int64_t)t * ntiles + blockIdx.x] = csum[t];   // the zone entries are added later
}

constexpr int ZT = 1024;          // k6_zone threads
constexpr int ZB = 2048;          // buckets over a zone
constexpr int kZoneSel = 2048;    // bucket entries staged for the exact selection (mean ~32 at 64M prompts)

// One CTA per zone: locate each split's threshold entry (the prompt at its class rank X) -- the zone's
// class prompts below it (gap counts + lower zones), a 2,048-bucket histogram of the zone's entries, the
// bucket holding rank X, an exact (kappa, p) selection inside that bucket -- into the DevPlan.
__global__ void __launch_bounds__(ZT, 1) k6_zone_select(DevPlan* __restrict__ plan, const KeyEntry* __restrict__ cand) {
  pdl_entry();
  __shared__ int hist[ZB + 1];
  __shared__ int wsum[ZT / 32];
  __shared__ uint64_t sel_k[kZoneSel];
  __shared__ int sel_p[kZoneSel];
  __shared__ int nsel;
  const int z = blockIdx.x, t = threadIdx.x;
  if (z >= plan->k6_nz || *reinterpret_cast<const volatile int*>(&plan->k6_fallback)) return;
  const int i = plan->z_cls[z];
  const int n = plan->z_fill[z];
  if (n > plan->z_cap[z]) return;   // overflow: k6_fused has set the fallback
  const KeyEntry* E = cand + plan->z_base[z];
  const uint64_t lo = plan->z_lo[z], width = plan->z_hi[z] - lo;
  int shift = 0;                     // bucket = (kappa - lo) >> shift, < ZB
  while ((width - 1) >> shift >= (uint64_t)ZB) ++shift;
  // class prompts below the zone: gaps 0..g and the lower zones of the class
  const int zi = z - plan->cls_zone0[i];
  int below = 0;
  for (int g = 0; g <= zi; ++g) below += plan->gapcnt[plan->cls_slot0[i] + g];
  for (int y = plan->cls_zone0[i]; y < z; ++y) below += plan->z_fill[y];
  for (int b = t; b <= ZB; b += ZT) hist[b] = 0;
  __syncthreads();
  for (int e = t; e < n; e += ZT) atomicAdd(&hist[(int)((E[e].key - lo) >> shift)], 1);
  __syncthreads();
  {   // exclusive scan of hist[0..ZB) in place (2 buckets per thread), hist[ZB] = n
    const int a0 = hist[2 * t], a1 = hist[2 * t + 1];
    int v = a0 + a1, incl = v;
    const int lane = t & 31, wp = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[wp] = incl;
    __syncthreads();
    int before = 0;
    for (int q = 0; q < wp; ++q) before += wsum[q];
    const int ex = before + incl - v;
    __syncthreads();
    hist[2 * t] = ex;
    hist[2 * t + 1] = ex + a0;
    if (t == ZT - 1) hist[ZB] = ex + v;
  }
  __syncthreads();
  const int s0 = plan->z_first[z], ns = plan->z_nsplit[z];
  for (int s = 0; s < ns; ++s) {
    const int r = plan->s_X[s0 + s] - below;
    if (r < 0 || r >= n) {   // the split's kappa lies outside its window: exact fallback
      if (t == 0) plan->k6_fallback = 1;
      return;                 // uniform across the CTA (r, n are block-uniform)
    }
    int b = 0;                // the last bucket with hist[b] <= r
    for (int step = ZB / 2; step > 0; step >>= 1)
      if (hist[b + step] <= r) b += step;
    if (t == 0) nsel = 0;
    __syncthreads();
    for (int e = t; e < n; e += ZT)
      if ((int)((E[e].key - lo) >> shift) == b) {
        const int q = atomicAdd(&nsel, 1);
        if (q < kZoneSel) {
          sel_k[q] = E[e].key;
          sel_p[q] = E[e].p;
        }
      }
    __syncthreads();
    const int m = nsel, want = r - hist[b];
    if (m > kZoneSel) {
      if (t == 0) plan->k6_fallback = 1;
      return;
    }
    for (int e = t; e < m; e += ZT) {   // the entry of rank `want` in the bucket by (kappa, p)
      int rk = 0;
      for (int f = 0; f < m; ++f) rk += entry_less(sel_k[f], sel_p[f], sel_k[e], sel_p[e]);
      if (rk == want) {
        plan->s_thr_k[s0 + s] = sel_k[e];
        plan->s_thr_p[s0 + s] = sel_p[e];
      }
    }
    __syncthreads();
  }
}

// Every zone entry, spread over many CTAs (blockIdx.y = zone): K' level = the level below the zone +
// the splits of the zone at or below it; K7 class and tile count.
template <int NCLS>
__global__ void __launch_bounds__(RT) k6_zone_apply(const __grid_constant__ RouteParams P, const DevPlan* __restrict__ plan,
                                                    const KeyEntry* __restrict__ cand, int32_t* __restrict__ K_prime,
                                                    uint8_t* __restrict__ cls7, int32_t* __restrict__ blk_counts,
                                                    int ntiles) {
  pdl_entry();
  const int z = blockIdx.y;
  if (z >= plan->k6_nz || *reinterpret_cast<const volatile int*>(&plan->k6_fallback)) return;
  const int n = plan->z_fill[z];
  if (n > plan->z_cap[z]) return;
  __shared__ uint64_t tk[kMaxZones];
  __shared__ int tp[kMaxZones], tm[kMaxZones];
  const int s0 = plan->z_first[z], ns = plan->z_nsplit[z];
  if (threadIdx.x < ns) {
    tk[threadIdx.x] = plan->s_thr_k[s0 + threadIdx.x];
    tp[threadIdx.x] = plan->s_thr_p[s0 + threadIdx.x];
    tm[threadIdx.x] = plan->s_mult[s0 + threadIdx.x];
  }
  __syncthreads();
  const KeyEntry* E = cand + plan->z_base[z];
  const int jb = plan->z_jbelow[z];
  const uint64_t bseq = batch_seq_of(P);
  for (int e = blockIdx.x * RT + threadIdx.x; e < n; e += gridDim.x * RT) {
    const uint64_t k = E[e].key;
    const int p = E[e].p;
    int j = jb;
    for (int s = 0; s < ns; ++s)
      if (!entry_less(k, p, tk[s], tp[s])) j += tm[s];
    PAS_CHECK(p >= 0 && p < P.N && j < P.nK, "K6 zone entry");
    K_prime[p] = P.grid[j];
    int c = j;
    if (NCLS > kMaxLevels) {
      const uint4 u = philox_stream(P.seed, bseq, (uint32_t)p, kStreamUniform);
      c = plan->inst_list[j][(uint32_t)(((uint64_t)u.x * (uint32_t)plan->n_inst[j]) >> 32)];
    }
    PAS_CHECK(c < NCLS, "K6 K7 class");
    cls7[p] = (uint8_t)c;
    atomicAdd(&blk_counts[(int64_t)c * ntiles + p / (FT * FPER)], 1);
  }
}

}  // namespace

int redirect_kb(int64_t N) {
  int b = 0;
  while (((int64_t)1 << b) < N) ++b;
  b -= 6;
  return b < 0 ? 0 : (b > kMaxK6Bits ? kMaxK6Bits : b);
}

cudaError_t launch_redirect(const uint8_t* level, const RouteParams& p, DevPlan* plan, const RedirectWs& w,
                            int32_t* K_prime, int32_t* blk_counts, int ntiles, int nC, cudaStream_t st,
                            int* launches, bool* counts_ready) {
  *counts_ready = false;
  if (p.N <= 0) return cudaSuccess;
  if (p.N < kWindowMinN) {   // small batches: the exact histogram path alone (fewer launches)
    cudaError_t e;
    if ((e = launch_zero(w.hist, (int64_t)p.nK << p.kb, w.used, 2, nullptr, 0, st))) return e;
    const unsigned blocks = (unsigned)((p.N + RT - 1) / RT);
    const unsigned hblocks = blocks < (unsigned)kNumSMs * 8 ? blocks : (unsigned)kNumSMs * 8;
    const int* ug = nullptr;   // ungated
    launch_pdl(k6_hist, hblocks, RT, 0, st, level, p, ug, w.key, w.hist);
    launch_pdl(k6_chunks, p.nK * kChunks, RT, 0, st, p, ug, w.hist, w.csum);
    launch_pdl(k6_bounds, p.nK, RT, 0, st, p, (const DevPlan*)plan, w.hist, w.csum, w.bnd, w.lists, w.used, ug);
    const unsigned ablocks = (!PAS_K6_GRIDCAP || blocks < (unsigned)kNumSMs * 8) ? blocks : (unsigned)kNumSMs * 8;
    launch_pdl(k6_assign, ablocks, RT, 0, st, level, w.key, p, (const DevPlan*)plan, w.bnd, w.lists, w.cand, K_prime,
               w.cls7, ug);
    launch_pdl(k6_resolve, p.nK * (p.nK - 1) > 0 ? p.nK * (p.nK - 1) : 1, RT, 0, st, p, (const DevPlan*)plan, w.bnd,
               w.lists, w.used, w.cand, K_prime, w.cls7, ug);
    *launches += 6;
    return cudaGetLastError();
  }
  *counts_ready = true;
  static_assert(FT * FPER == 4096, "k6_fused tiles are K7's tiles (batch_tiles)");
  const bool uniform = p.mode == PAS_UNIFORM;
  // the windowed pass and the zone resolves (K7's tile counts included)
  // zone entries per batch ~ 8 sqrt(h) per split: 64 CTAs per zone spread the apply over the SMs
  const dim3 agrid(64, kMaxZones);
  if (uniform) {
    launch_pdl(k6_fused<kMaxInst>, (unsigned)ntiles, FT, 0, st, level, p, plan, w.cand, K_prime, w.cls7, blk_counts, ntiles);
    launch_pdl(k6_zone_select, (unsigned)kMaxZones, ZT, 0, st, plan, (const KeyEntry*)w.cand);
    launch_pdl(k6_zone_apply<kMaxInst>, agrid, RT, 0, st, p, (const DevPlan*)plan, (const KeyEntry*)w.cand, K_prime,
               w.cls7, blk_counts, ntiles);
  } else {
    launch_pdl(k6_fused<kMaxLevels>, (unsigned)ntiles, FT, 0, st, level, p, plan, w.cand, K_prime, w.cls7, blk_counts, ntiles);
    launch_pdl(k6_zone_select, (unsigned)kMaxZones, ZT, 0, st, plan, (const KeyEntry*)w.cand);
    launch_pdl(k6_zone_apply<kMaxLevels>, agrid, RT, 0, st, p, (const DevPlan*)plan, (const KeyEntry*)w.cand, K_prime,
               w.cls7, blk_counts, ntiles);
  }
  (void)nC;
  // the exact histogram path, each kernel a no-op unless k6_fallback was set
  const int* gate = &plan->k6_fallback;
  const int64_t nzero = (int64_t)p.nK << p.kb;
  int64_t zb = (nzero + RT - 1) / RT;
  if (zb > kNumSMs * 8) zb = kNumSMs * 8;
  launch_pdl(k6_zero, (unsigned)zb, RT, 0, st, gate, w.hist, nzero, w.used, 2);
  const unsigned blocks = (unsigned)((p.N + RT - 1) / RT);
  const unsigned hblocks = blocks < (unsigned)kNumSMs * 8 ? blocks : (unsigned)kNumSMs * 8;
  launch_pdl(k6_hist, hblocks, RT, 0, st, level, p, gate, w.key, w.hist);
  launch_pdl(k6_chunks, p.nK * kChunks, RT, 0, st, p, gate, w.hist, w.csum);
  launch_pdl(k6_bounds, p.nK, RT, 0, st, p, (const DevPlan*)plan, w.hist, w.csum, w.bnd, w.lists, w.used, gate);
  const unsigned ablocks = (!PAS_K6_GRIDCAP || blocks < (unsigned)kNumSMs * 8) ? blocks : (unsigned)kNumSMs * 8;
  launch_pdl(k6_assign, ablocks, RT, 0, st, level, w.key, p, (const DevPlan*)plan, w.bnd, w.lists, w.cand, K_prime,
             w.cls7, gate);
  launch_pdl(k6_resolve, p.nK * (p.nK - 1) > 0 ? p.nK * (p.nK - 1) : 1, RT, 0, st, p, (const DevPlan*)plan, w.bnd,
             w.lists, w.used, w.cand, K_prime, w.cls7, gate);
  *launches += 9;
  return cudaGetLastError();
}

}  // namespace pas
