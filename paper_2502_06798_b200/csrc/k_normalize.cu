// K1 -- normalise + quantise embedding rows (prompts per batch, cache rows at insert).
//
// v_hat_i = bf16_RNE( fp32_RN( v_i / sqrt(sum_j v_j^2) ) ), the sum of squares and the division in
// fp64 (R11).  Cosine "closeness" of two unit rows is then a dot
// product, which K2 computes on the tensor cores.  A row with a non-finite element or zero norm is
// invalid (R16): it is written as zeros and flagged (prompts) or counted (cache insert -> rejected).
//
// One warp per row, 128-bit loads (4 fp32 / 4 bf16 per lane per step); the row's loads are all in
// flight at once for the fp64 sum of squares, then the row is re-read (an L1 / L2 hit, no HBM bytes)
// for the quantised stores, so no value is live across the reduction: 40 registers, 6 resident CTAs
// (48 warps) per SM.  Measured (profiles/r01_k1c, r01_k1g): cache insert 5.43 TB/s (5.02 on
// a resident-CTA grid) vs 4.56 with
// the row held in registers at 3 CTAs/SM (80 registers) and 4.78 at 4 CTAs/SM (64 registers, spills).
// HBM-bound: algorithmic bytes per row = d*(in_bytes + 2) (+1 flag byte).
// Cache insert applies the shard filter of the round-robin partition (gid g lives on rank g % G at
// local row g / G): it stores only this rank's rows but checks every row's validity, so
// all ranks accept or reject a load together.
#include "pas_internal.cuh"

namespace pas {
namespace {

__device__ __forceinline__ void load4(const float* p, float (&v)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void load4(const __nv_bfloat16* p, float (&v)[4]) {
  const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
  v[0] = __uint_as_float(x.x << 16);
  v[1] = __uint_as_float(x.x & 0xFFFF0000u);
  v[2] = __uint_as_float(x.y << 16);
  v[3] = __uint_as_float(x.y & 0xFFFF0000u);
}

// fp32_RN(v / norm) without a per-element fp64 division: q = v * RN(1 / norm) is within 2 ulp (fp64)
// of v / norm, so fp32_RN(q) == fp32_RN(v / norm) unless v / norm lies within a few fp64 ulp of an
// fp32 rounding midpoint -- recognisable from the 29 bits of q below the fp32 mantissa being
// ~0x10000000 -- in which case (probability ~2^-25) the exact fp64 division decides.  Below 2^-126 the
// fp32 result is subnormal and rounds at a higher bit than those 29, so there the division always
// decides (a component < 2^-126 of its row's norm: never in real embeddings; the adversarial rows of
// tests/test_gpu_k1_exact.py put quotients exactly on subnormal midpoints).  One DMUL per element
// instead of a division sequence keeps K1 off the fp64 pipe's limit and on the HBM roofline.
__device__ __forceinline__ float div_rn(float v, double norm, double inv) {
  const double q = (double)v * inv;
  const long long low = __double_as_longlong(q) & 0x1FFFFFFFLL;
  if (llabs(low - 0x10000000LL) <= 16 || fabs(q) < 0x1p-126) return __double2float_rn((double)v / norm);
  return __double2float_rn(q);
}

// dup != nullptr: the same four values are also stored there (K2's duplicated-row small batches)
__device__ __forceinline__ void store_row4(__nv_bfloat16* dst, const float (&v)[4], double norm, bool valid,
                                           __nv_bfloat16* dup = nullptr) {
  __nv_bfloat162 lo, hi;
  if (valid) {
    const double inv = 1.0 / norm;
    lo = __floats2bfloat162_rn(div_rn(v[0], norm, inv), div_rn(v[1], norm, inv));
    hi = __floats2bfloat162_rn(div_rn(v[2], norm, inv), div_rn(v[3], norm, inv));
  } else {
    lo = __floats2bfloat162_rn(0.f, 0.f);
    hi = lo;
  }
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = pk;
  if (dup) *reinterpret_cast<uint2*>(dup) = pk;
}

// One warp per row.  VEC = d / 128 float4 (or 4 x bf16) per lane: all of a row's loads are in flight
// at once and the row is read from HBM exactly once; VEC = 0 is the generic two-pass path for d > 1024.
#ifndef PAS_K1_MINB
#define PAS_K1_MINB 6     // resident CTAs of 256 threads per SM (register budget 65536 / (256 MINB))
#endif
#ifndef PAS_K1_RELOAD
#define PAS_K1_RELOAD 1   // re-read the row for the stores (fewer live registers, more resident warps)
#endif
#ifndef PAS_K1_GRIDCAP
#define PAS_K1_GRIDCAP 0  // 0: one CTA per 8 rows, the block scheduler balances the tail (64 vs 70 us
                          // at C4, cache insert 5.43 vs 4.96 TB/s, profiles/r01_k1g/); 1: grid = the
                          // resident CTAs with grid-stride rows
#endif
#ifndef PAS_K1_ACC
#define PAS_K1_ACC 1      // independent fp64 partial sums per lane (shorter DFMA dependency chain)
#endif

// DUP: every row is also written dup_rows rows further down (K2's duplicated-row small batches); a
// compile-time switch so the common path carries no extra live state (40 registers, no spills).
template <typename T, int VEC, bool DUP>
__global__ void __launch_bounds__(256, PAS_K1_MINB) k_normalize(const T* __restrict__ in, int64_t rows, int d,
                                                   __nv_bfloat16* __restrict__ out, uint8_t* __restrict__ flags,
                                                   int64_t first_gid, int G, int rank, int* invalid_count,
                                                   uint32_t* epoch_bump, int64_t dup_rows) {
  pdl_entry();
  if (epoch_bump && blockIdx.x == 0 && threadIdx.x == 0) {   // the epoch of the K2 launch that follows
    const uint32_t e = *epoch_bump + 1;
    *epoch_bump = e ? e : 1;
  }
  const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp_global; i < rows; i += nwarps) {
    const int64_t gid = first_gid + i;
    // A row of another rank's shard is not stored here, but its validity is still checked when the
    // caller counts invalid rows (cache insert): every rank must accept or reject the same load
    // (pas.h: "nothing appended"), whichever rank owns the bad row.
    const bool own = G == 1 || (gid % G) == rank;
    if (!own && !invalid_count) continue;
    const int64_t orow = (G > 1) ? gid / G : gid;
    const T* src = in + i * (int64_t)d;
    __nv_bfloat16* dst = out + orow * (int64_t)d;
    double ss = 0.0;
    bool finite = true;
    if constexpr (VEC > 0) {
      float v[VEC][4];
#pragma unroll
      for (int c = 0; c < VEC; ++c) load4(src + c * 128 + lane * 4, v[c]);
      double part[PAS_K1_ACC];
#pragma unroll
      for (int a = 0; a < PAS_K1_ACC; ++a) part[a] = 0.0;
#pragma unroll
      for (int c = 0; c < VEC; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          finite &= isfinite(v[c][j]);
          part[(c * 4 + j) % PAS_K1_ACC] += (double)v[c][j] * (double)v[c][j];
        }
#pragma unroll
      for (int a = 0; a < PAS_K1_ACC; ++a) ss += part[a];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      finite = __all_sync(0xffffffffu, finite);
      const double norm = sqrt(ss);
      const bool valid = finite && norm > 0.0;
      if (!own) {
        if (lane == 0 && !valid) atomicAdd(invalid_count, 1);
        continue;
      }
#if PAS_K1_RELOAD
      // the row is re-read (L1 / L2 hit, no HBM traffic) instead of held across the reduction
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        float w[4];
        load4(src + c * 128 + lane * 4, w);
        store_row4(dst + c * 128 + lane * 4, w, norm, valid, DUP ? dst + dup_rows * d + c * 128 + lane * 4 : nullptr);
      }
#else
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        store_row4(dst + c * 128 + lane * 4, v[c], norm, valid, DUP ? dst + dup_rows * d + c * 128 + lane * 4 : nullptr);
      }
#endif
      if (lane == 0) {
        if (flags) flags[orow] = valid ? 0 : PAS_FLAG_INVALID;
        if (!valid && invalid_count) atomicAdd(invalid_count, 1);
      }
    } else {
      for (int c = lane * 4; c < d; c += 128) {
        float v[4];
        load4(src + c, v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          finite &= isfinite(v[j]);
          ss += (double)v[j] * (double)v[j];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      finite = __all_sync(0xffffffffu, finite);
      const double norm = sqrt(ss);
      const bool valid = finite && norm > 0.0;
      if (!own) {
        if (lane == 0 && !valid) atomicAdd(invalid_count, 1);
        continue;
      }
      for (int c = lane * 4; c < d; c += 128) {
        float v[4];
        load4(src + c, v);
        store_row4(dst + c, v, norm, valid, DUP ? dst + dup_rows * d + c : nullptr);
      }
      if (lane == 0) {
        if (flags) flags[orow] = valid ? 0 : PAS_FLAG_INVALID;
        if (!valid && invalid_count) atomicAdd(invalid_count, 1);
      }
    }
  }
}

template <typename T>
cudaError_t launch_t(const T* in, int64_t rows, int d, __nv_bfloat16* out, uint8_t* flags, int64_t first_gid, int G,
                     int rank, int* invalid_count, cudaStream_t st, uint32_t* eb, int64_t dup) {
  const int threads = 256;
  const int vec = d % 128 == 0 && d <= 1024 ? d / 128 : 0;
  // one warp per row, one CTA per 8 rows (PAS_K1_GRIDCAP 1: capped at the resident CTAs, grid-stride)
  int64_t blocks = (rows * 32 + threads - 1) / threads;
  const int64_t cap = (int64_t)kNumSMs * PAS_K1_MINB;
  if (PAS_K1_GRIDCAP && blocks > cap) blocks = cap;
  const unsigned g = (unsigned)blocks;
  auto go = [&](auto kern) {
    launch_pdl(kern, g, threads, 0, st, in, rows, d, out, flags, first_gid, G, rank, invalid_count, eb, dup);
  };
  switch (vec) {
    case 1: dup ? go(k_normalize<T, 1, true>) : go(k_normalize<T, 1, false>); break;
    case 2: dup ? go(k_normalize<T, 2, true>) : go(k_normalize<T, 2, false>); break;
    case 3: dup ? go(k_normalize<T, 3, true>) : go(k_normalize<T, 3, false>); break;
    case 4: dup ? go(k_normalize<T, 4, true>) : go(k_normalize<T, 4, false>); break;
    case 5: dup ? go(k_normalize<T, 5, true>) : go(k_normalize<T, 5, false>); break;
    case 6: dup ? go(k_normalize<T, 6, true>) : go(k_normalize<T, 6, false>); break;
    case 7: dup ? go(k_normalize<T, 7, true>) : go(k_normalize<T, 7, false>); break;
    case 8: dup ? go(k_normalize<T, 8, true>) : go(k_normalize<T, 8, false>); break;
    default: dup ? go(k_normalize<T, 0, true>) : go(k_normalize<T, 0, false>);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_normalize(const void* in, pas_dtype dtype, int64_t rows, int d, __nv_bfloat16* out,
                             uint8_t* flags, int64_t first_gid, int G, int rank, int* invalid_count,
                             cudaStream_t st, uint32_t* epoch_bump, int64_t dup_rows) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == PAS_F32)
    return launch_t(static_cast<const float*>(in), rows, d, out, flags, first_gid, G, rank, invalid_count, st,
                    epoch_bump, dup_rows);
  return launch_t(static_cast<const __nv_bfloat16*>(in), rows, d, out, flags, first_gid, G, rank, invalid_count, st,
                  epoch_bump, dup_rows);
}

}  // namespace pas
