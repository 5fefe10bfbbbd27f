// K6 -- redirection sampling: every prompt gets its K' from the Route-Plan.
//
// Exact-count form (R3): within optimal-K class i, prompts are ranked by a 60-bit Philox
// key kappa_p (ties by prompt index), and rank_p in [X_i[j-1], X_i[j]) is served at K'_j, so exactly
// x_ij prompts of class i go to level j and the ranks are a uniformly random permutation of the class
// (R18: kappa depends only on seed, batch_seq, p -- not on the router GPU count).
//
// Ranking without a full sort: composite key (class << 60 | kappa) -> bucket (class, top kb bits of
// kappa) counting sort (count, scan, scatter of (key, p) into bucket order), then each entry counts
// the entries below it inside its own bucket, which is contiguous and cache-resident (kb keeps the
// mean bucket of a full class at <= 16 entries).  Global rank = bucket start + in-bucket rank = the
// position in the (key, p) order; rank within class = global rank - class start.
//
// Kernels: k_keys (Philox + bucket histogram), the device-wide scan (k_scan.cu), k_scatter, k_rank (rank, K', and the
// route-and-batch class: K' level in greedy mode, instance I_j[(u n_j) >> 32] in uniform mode).
#include "pas_internal.cuh"
#include "philox.cuh"

namespace pas {
namespace {

__global__ void k_keys(const uint8_t* __restrict__ level, RouteParams P, uint64_t* __restrict__ key,
                       int32_t* __restrict__ bucket, int32_t* __restrict__ bcount) {
  pdl_entry();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.N) return;
  const uint4 w = philox_stream(P.seed, P.batch_seq, (uint32_t)p, kStreamRedirect);
  const uint64_t kappa = (((uint64_t)w.y << 32) | w.x) >> 4;
  const uint32_t lvl = level[p];
  key[p] = ((uint64_t)lvl << 60) | kappa;
  const int32_t b = (int32_t)((lvl << P.kb) | (uint32_t)(P.kb ? (kappa >> (60 - P.kb)) : 0));
  bucket[p] = b;
  atomicAdd(&bcount[b], 1);
}

// Counting-sort scatter of (key, p) into bucket order (order inside a bucket is arbitrary).
__global__ void k_scatter(const uint64_t* __restrict__ key, const int32_t* __restrict__ bucket, int64_t N,
                          const int32_t* __restrict__ bstart, int32_t* __restrict__ bfill,
                          KeyEntry* __restrict__ sorted) {
  pdl_entry();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int b = bucket[p];
  sorted[bstart[b] + atomicAdd(&bfill[b], 1)] = KeyEntry{key[p], (int32_t)p, 0};
}

// Thread per bucket-ordered entry: its rank inside its (contiguous, cache-resident) bucket by
// (key, p), hence its global rank, its rank within its optimal-K class, its K' and its K7 class.
__global__ void k_rank(const KeyEntry* __restrict__ sorted, RouteParams P, const DevPlan* __restrict__ plan,
                       const int32_t* __restrict__ bcount, const int32_t* __restrict__ bstart,
                       uint8_t* __restrict__ cls7, int32_t* __restrict__ K_prime) {
  pdl_entry();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.N) return;
  const KeyEntry e = sorted[i];
  const uint32_t lvl = (uint32_t)(e.key >> 60);
  const int b = (int)(P.kb ? (e.key >> (60 - P.kb)) : lvl);
  const int start = bstart[b], n = bcount[b];
  int r = 0;
  for (int q = start; q < start + n; ++q) {
    const KeyEntry f = sorted[q];
    r += (f.key < e.key || (f.key == e.key && f.p < e.p)) ? 1 : 0;
  }
  const int rank = start + r - plan->class_start[lvl];
  int j = 0;
  while (j < P.nK - 1 && rank >= plan->X[lvl][j]) ++j;
  const int p = e.p;
  K_prime[p] = P.grid[j];
  if (P.mode == PAS_UNIFORM) {
    const uint4 w = philox_stream(P.seed, P.batch_seq, (uint32_t)p, kStreamUniform);
    const uint32_t nj = (uint32_t)plan->n_inst[j];
    cls7[p] = plan->inst_list[j][(uint32_t)(((uint64_t)w.x * nj) >> 32)];
  } else {
    cls7[p] = j;
  }
}

}  // namespace

cudaError_t launch_redirect(const uint8_t* level, const RouteParams& p, const DevPlan* plan, const RedirectWs& w,
                            int32_t* K_prime, cudaStream_t st, int* launches) {
  if (p.N <= 0) return cudaSuccess;
  const int nb = p.nK << p.kb;
  cudaError_t e;
  if ((e = launch_zero(w.bcount, nb, w.bfill, nb, nullptr, 0, st))) return e;
  *launches += 1;
  const unsigned blocks = (unsigned)((p.N + 255) / 256);
  launch_pdl(k_keys, blocks, 256, 0, st, level, p, w.key, w.bucket, w.bcount);
  if ((e = launch_exclusive_scan(w.bcount, w.bstart, nb, w.scan_tmp, st, launches))) return e;
  launch_pdl(k_scatter, blocks, 256, 0, st, w.key, w.bucket, p.N, w.bstart, w.bfill, w.sorted);
  launch_pdl(k_rank, blocks, 256, 0, st, w.sorted, p, plan, w.bcount, w.bstart, w.cls7, K_prime);
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace pas
