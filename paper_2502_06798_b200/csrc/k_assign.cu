// f4 -- the Resource Controller's Model Cache Assigner + Query Fraction Solver (PAPER.md P:88, P:207,
// P:223; R33-R36), solved exactly by enumerating every assignment on the GPU.
//
// An assignment n puts n_K of the W serving instances at level K (sum n = W): C(W + nK - 1, nK - 1)
// of them, 11.2M for the SPEC's scale (W = 64, 6 levels).  Each is scored in closed form (R34):
//   cap_K = n_K rate_K / lambda,  S = min(1, sum_K cap_K),  F = greedy fill of S by a_K descending,
//   q = sum F_K a_K,
// and the optimum is the lexicographic max of (S, q, n) with S, q rounded to multiples of 2^-40 (R35).
// k_assign_enum: every thread unranks the first assignment of its chunk (decreasing lexicographic
// order, stars and bars with a binomial table in shared memory), then walks the chunk with the O(1)
// successor, keeping its best key (qS, qq, n packed as bytes); warp shuffles + shared memory reduce
// to one key per CTA.  k_assign_final (one warp) reduces the CTA keys and re-scores the winner into
// F, F / S and the instance levels.  fp64 with explicit _rn intrinsics (no FMA contraction), the same
// operation order as oracle/controller.py.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int AT = 256;                  // threads per CTA
constexpr int BMAX = kMaxInst + kMaxLevels + 1;

struct Key {
  long long s, q;                        // quantised S and q (units of 2^-40)
  unsigned long long hi, lo;             // n_0..n_7 and n_8..n_15, one byte each, n_0 most significant
};

__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
  if (a.s != b.s) return a.s < b.s;
  if (a.q != b.q) return a.q < b.q;
  if (a.hi != b.hi) return a.hi < b.hi;
  return a.lo < b.lo;
}

__device__ __forceinline__ Key shfl_key(const Key& k, int src) {
  Key o;
  o.s = __shfl_sync(0xffffffffu, k.s, src);
  o.q = __shfl_sync(0xffffffffu, k.q, src);
  o.hi = __shfl_sync(0xffffffffu, k.hi, src);
  o.lo = __shfl_sync(0xffffffffu, k.lo, src);
  return o;
}

// rate_K (R33), a_K (R33), fill order (R34): a few dozen flops, recomputed by every CTA
__device__ void setup(const AssignParams& P, double* r, double* a, int* order, double* H) {
  for (int k = 0; k < P.nK; ++k) {   // the forecast: given, or the f1 predictor's window
    if (!P.fc) H[k] = P.H[k];
    else if (P.fc->n == 0) H[k] = __ddiv_rn(1.0, (double)P.nK);
    else H[k] = __ddiv_rn((double)P.fc->cnt[k], (double)P.fc->n);
  }
  for (int k = 0; k < P.nK; ++k) r[k] = __ddiv_rn(__dmul_rn((double)P.bstar, 1e6), (double)P.service_us[k]);
  for (int j = 0; j < P.nK; ++j) {
    double deg = 0.0;
    for (int i = 0; i < P.nK; ++i)
      if (P.grid[i] < P.grid[j]) deg = __dadd_rn(deg, __dmul_rn(H[i], P.c[P.grid[j] - P.grid[i]]));
    a[j] = __dsub_rn(1.0, deg);
  }
  for (int k = 0; k < P.nK; ++k) order[k] = k;
  for (int x = 1; x < P.nK; ++x)        // insertion sort by (a desc, k asc)
    for (int y = x; y > 0 && (a[order[y]] > a[order[y - 1]]); --y) {
      const int t = order[y];
      order[y] = order[y - 1];
      order[y - 1] = t;
    }
}

// S, q (and F if requested) of one assignment (R34)
__device__ __forceinline__ void score(const AssignParams& P, const int* n, const double* r, const double* a,
                                      const int* order, double& S, double& q, double* F) {
  double cap[kMaxLevels];
  if (P.lam == 0.0) {
    S = 1.0;
    for (int k = 0; k < P.nK; ++k) cap[k] = n[k] > 0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
  } else {
    double tot = 0.0;
    for (int k = 0; k < P.nK; ++k) {
      cap[k] = __ddiv_rn(__dmul_rn((double)n[k], r[k]), P.lam);
      tot = __dadd_rn(tot, cap[k]);
    }
    S = tot < 1.0 ? tot : 1.0;
  }
  double filled = 0.0;
  q = 0.0;
  for (int x = 0; x < P.nK; ++x) {
    const int k = order[x];
    const double room = __dsub_rn(S, filled);
    const double take = cap[k] < room ? cap[k] : room;
    if (F) F[k] = take;
    filled = __dadd_rn(filled, take);
    q = __dadd_rn(q, __dmul_rn(take, a[k]));
  }
}

__device__ __forceinline__ Key make_key(const AssignParams& P, const int* n, double S, double q) {
  Key k;
  k.s = __double2ll_rn(__dmul_rn(S, 1099511627776.0));   // 2^40 (exact scaling)
  k.q = __double2ll_rn(__dmul_rn(q, 1099511627776.0));
  k.hi = 0;
  k.lo = 0;
  for (int i = 0; i < kMaxLevels; ++i) {
    const unsigned long long v = i < P.nK ? (unsigned long long)n[i] : 0ull;
    if (i < 8) k.hi |= v << (8 * (7 - i));
    else k.lo |= v << (8 * (15 - i));
  }
  return k;
}

__global__ void __launch_bounds__(AT) k_assign_enum(const AssignParams P, int64_t total, int64_t chunk,
                                                    Key* __restrict__ block_best) {
  __shared__ long long binom[BMAX][kMaxLevels + 1];   // binom[m][p] = C(m, p)
  __shared__ double r_s[kMaxLevels], a_s[kMaxLevels];
  __shared__ int order_s[kMaxLevels];
  __shared__ double h_s[kMaxLevels];
  __shared__ Key warp_best[AT / 32];
  if (threadIdx.x == 0) {
    setup(P, r_s, a_s, order_s, h_s);
    for (int m = 0; m < BMAX; ++m)
      for (int p = 0; p <= kMaxLevels; ++p)
        binom[m][p] = p == 0 ? 1 : (m == 0 ? 0 : binom[m - 1][p - 1] + (p <= m - 1 ? binom[m - 1][p] : 0));
  }
  __syncthreads();
  const int nK = P.nK;
  Key best;
  best.s = best.q = LLONG_MIN;
  best.hi = best.lo = 0;
  const int64_t first = ((int64_t)blockIdx.x * AT + threadIdx.x) * chunk;
  if (first < total) {
    // unrank `first` in decreasing lexicographic order: compositions of m into p parts = C(m+p-1, p-1)
    int n[kMaxLevels];
    int64_t rr = first;
    int m = P.W;
    for (int i = 0; i + 1 < nK; ++i) {
      const int p = nK - i - 1;
      int v = m;
      for (; v > 0; --v) {
        const int64_t cnt = binom[m - v + p - 1][p - 1];
        if (rr < cnt) break;
        rr -= cnt;
      }
      n[i] = v;
      m -= v;
    }
    n[nK - 1] = m;
    const int64_t last = first + chunk < total ? first + chunk : total;
    for (int64_t t = first; t < last; ++t) {
      double S, q;
      score(P, n, r_s, a_s, order_s, S, q, nullptr);
      const Key k = make_key(P, n, S, q);
      if (key_less(best, k)) best = k;
      // successor: move the last part's remainder + 1 behind the last non-zero earlier part
      const int tail = n[nK - 1];
      n[nK - 1] = 0;
      int j = nK - 2;
      while (j >= 0 && n[j] == 0) --j;
      if (j < 0) break;
      n[j] -= 1;
      n[j + 1] = tail + 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const Key other = shfl_key(best, (threadIdx.x & 31) ^ o);
    if (key_less(best, other)) best = other;
  }
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Key b = warp_best[0];
    for (int w = 1; w < AT / 32; ++w)
      if (key_less(b, warp_best[w])) b = warp_best[w];
    block_best[blockIdx.x] = b;
  }
}

__global__ void __launch_bounds__(32) k_assign_final(const AssignParams P, const Key* __restrict__ block_best,
                                                     int nblocks, AssignOut* __restrict__ out) {
  __shared__ double r_s[kMaxLevels], a_s[kMaxLevels];
  __shared__ int order_s[kMaxLevels];
  __shared__ double h_s[kMaxLevels];
  if (threadIdx.x == 0) setup(P, r_s, a_s, order_s, h_s);
  Key best;
  best.s = best.q = LLONG_MIN;
  best.hi = best.lo = 0;
  for (int b = threadIdx.x; b < nblocks; b += 32)
    if (key_less(best, block_best[b])) best = block_best[b];
  for (int o = 16; o > 0; o >>= 1) {
    const Key other = shfl_key(best, threadIdx.x ^ o);
    if (key_less(best, other)) best = other;
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  int n[kMaxLevels];
  for (int i = 0; i < kMaxLevels; ++i)
    n[i] = (int)((i < 8 ? best.hi >> (8 * (7 - i)) : best.lo >> (8 * (15 - i))) & 0xFFull);
  double S, q, F[kMaxLevels];
  score(P, n, r_s, a_s, order_s, S, q, F);
  int w = 0;
  for (int k = 0; k < kMaxLevels; ++k) {
    out->n[k] = k < P.nK ? n[k] : 0;
    out->F[k] = k < P.nK ? F[k] : 0.0;
    out->F_route[k] = k < P.nK ? __ddiv_rn(F[k], S) : 0.0;
    out->H[k] = k < P.nK ? h_s[k] : 0.0;
    for (int i = 0; k < P.nK && i < n[k]; ++i) out->instance_level[w++] = k;
  }
  out->served = S;
  out->quality = q;
}

}  // namespace

int64_t assign_count(int W, int nK) {
  // C(W + nK - 1, nK - 1), saturating at 2^62
  long double v = 1;
  for (int i = 1; i <= nK - 1; ++i) v = v * (W + i) / i;
  return v > 4.0e18L ? ((int64_t)1 << 62) : (int64_t)(v + 0.5L);
}

cudaError_t launch_assign(const AssignParams& p, void* block_best, int max_blocks, AssignOut* out, cudaStream_t st) {
  const int64_t total = assign_count(p.W, p.nK);
  // chunks of >= 64 assignments per thread; at most max_blocks CTAs (a few waves over 148 SMs)
  int64_t threads = (total + 63) / 64;
  int64_t blocks = (threads + AT - 1) / AT;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  const int64_t chunk = (total + blocks * AT - 1) / (blocks * AT);
  k_assign_enum<<<(unsigned)blocks, AT, 0, st>>>(p, total, chunk, static_cast<Key*>(block_best));
  k_assign_final<<<1, 32, 0, st>>>(p, static_cast<const Key*>(block_best), (int)blocks, out);
  return cudaGetLastError();
}

size_t assign_key_bytes() { return sizeof(Key); }

}  // namespace pas
