// Device-wide exclusive prefix sum of int32 counts (counting sorts of K6 and K7).
//
// n <= 16384: one CTA walks coalesced tiles of 4096 with a running carry.  Larger n: the classic
// three-phase scan -- per-tile totals (k_tile_sum, 4096 per CTA), a one-CTA scan of the totals, and
// a per-tile scan seeded with its total prefix (k_tile_scan) -- two reads and one write of the input.
#include "pas_internal.cuh"

namespace pas {
namespace {

constexpr int THREADS = 1024;
constexpr int TILE = THREADS * 4;

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix and the block total.
__device__ __forceinline__ int block_exclusive(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wsum[lane] = x;
  }
  __syncthreads();
  total = wsum[31];
  const int ex = (w ? wsum[w - 1] : 0) + incl - v;
  __syncthreads();
  return ex;
}

__device__ __forceinline__ void load_tile(const int32_t* in, int n, int i0, int (&v)[4]) {
  if (i0 + 3 < n && (i0 & 3) == 0) {
    const int4 x = *reinterpret_cast<const int4*>(in + i0);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (i0 + j < n) ? in[i0 + j] : 0;
  }
}

__global__ void __launch_bounds__(THREADS) k_scan_small(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                                        int n) {
  pdl_entry();
  __shared__ int wsum[32];
  int carry = 0;
  for (int base = 0; base < n; base += TILE) {
    const int i0 = base + 4 * threadIdx.x;
    int v[4];
    load_tile(in, n, i0, v);
    int total;
    int run = carry + block_exclusive(v[0] + v[1] + v[2] + v[3], wsum, total);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j < n) out[i0 + j] = run;
      run += v[j];
    }
    carry += total;
  }
}

__global__ void __launch_bounds__(THREADS) k_tile_sum(const int32_t* __restrict__ in, int n,
                                                      int32_t* __restrict__ sums) {
  pdl_entry();
  __shared__ int wsum[32];
  const int i0 = blockIdx.x * TILE + 4 * threadIdx.x;
  int v[4];
  load_tile(in, n, i0, v);
  int total;
  block_exclusive(v[0] + v[1] + v[2] + v[3], wsum, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(THREADS) k_tile_scan(const int32_t* __restrict__ in, int n,
                                                       const int32_t* __restrict__ prefix, int32_t* __restrict__ out) {
  pdl_entry();
  __shared__ int wsum[32];
  const int i0 = blockIdx.x * TILE + 4 * threadIdx.x;
  int v[4];
  load_tile(in, n, i0, v);
  int total;
  int run = prefix[blockIdx.x] + block_exclusive(v[0] + v[1] + v[2] + v[3], wsum, total);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i0 + j < n) out[i0 + j] = run;
    run += v[j];
  }
}

__global__ void k_zero(int32_t* a, int64_t na, int32_t* b, int64_t nb, int32_t* c, int64_t nc) {
  pdl_entry();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb + nc; i += stride) {
    if (i < na) a[i] = 0;
    else if (i < na + nb) b[i - na] = 0;
    else c[i - na - nb] = 0;
  }
}

}  // namespace

cudaError_t launch_zero(int32_t* a, int64_t na, int32_t* b, int64_t nb, int32_t* c, int64_t nc, cudaStream_t st) {
  const int64_t n = na + nb + nc;
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  return launch_pdl(k_zero, (unsigned)blocks, 256, 0, st, a, na, b, nb, c, nc);
}

int scan_tmp_ints(int64_t n) { return (int)((n + TILE - 1) / TILE) + 1; }

cudaError_t launch_exclusive_scan(const int32_t* in, int32_t* out, int n, int32_t* tmp, cudaStream_t st,
                                  int* launches) {
  if (n <= 0) return cudaSuccess;
  if (n <= 4 * TILE) {
    launch_pdl(k_scan_small, 1, THREADS, 0, st, in, out, n);
    *launches += 1;
    return cudaGetLastError();
  }
  const int tiles = (n + TILE - 1) / TILE;
  launch_pdl(k_tile_sum, tiles, THREADS, 0, st, in, n, tmp);
  launch_pdl(k_scan_small, 1, THREADS, 0, st, tmp, tmp, tiles);   // in-place is safe: each element read before written
  launch_pdl(k_tile_scan, tiles, THREADS, 0, st, in, n, tmp, out);
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace pas
