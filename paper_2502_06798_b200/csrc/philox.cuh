// philox.cuh -- Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), device implementation.
// Counter layout (R18): key = (seed_lo, seed_hi); ctr = (p, 0, batch_lo,
// (stream << 24) | (batch_hi & 0xffffff)).  Streams: 1 = redirection key, 2 = uniform routing.
#pragma once
#include <stdint.h>

namespace pas {

constexpr uint32_t kStreamRedirect = 1;
constexpr uint32_t kStreamUniform = 2;
constexpr uint32_t kStreamForecast = 3;   // f1: i.i.d. K' draw from the forecast Route-Plan (R23)

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ uint4 philox_stream(uint64_t seed, uint64_t batch_seq, uint32_t p, uint32_t stream) {
  const uint4 ctr = make_uint4(p, 0u, (uint32_t)batch_seq, (stream << 24) | ((uint32_t)(batch_seq >> 32) & 0xFFFFFFu));
  return philox4x32_10(ctr, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

}  // namespace pas
