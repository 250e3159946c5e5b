// Device helpers shared by the pgpb kernels.
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>

#include "pgpb_internal.h"

namespace pgpb {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarpsPerBlock = 8;
constexpr int kThreads = kWarpsPerBlock * 32;
// Root row staged in shared memory up to this many bytes (2 arrays).
constexpr int kMaxSmemRootBytes = 160 * 1024;

int sm_count(int device);
void retain_pool(int device);
int current_device();

// Grid for a warp-per-item kernel: enough CTAs to cover `items` warps but
// no more than `per_sm` resident CTAs on each of the SMs (grid-stride beyond).
inline unsigned warp_grid(int64_t items, int per_sm) {
  const int64_t need = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = int64_t(sm_count(current_device())) * per_sm;
  int64_t g = need < cap ? need : cap;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// Cooperative copy of the dense root row into shared memory.
__device__ __forceinline__ void stage_root(const TableView &t, float *s_root, int32_t *s_next) {
  const int n4 = t.vocab_padded >> 2;
  const float4 *g4 = reinterpret_cast<const float4 *>(t.root_scores);
  const int4 *n4p = reinterpret_cast<const int4 *>(t.root_next);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    reinterpret_cast<float4 *>(s_root)[i] = __ldg(g4 + i);
    reinterpret_cast<int4 *>(s_next)[i] = __ldg(n4p + i);
  }
}

// Lexicographic "a beats b" for the first-max argmax: higher value, then
// lower index.  Scanning ascending with this rule reproduces the reference's
// strict-greater ascending scan (_kernels.pyx:143-148, np.argmax).
__device__ __forceinline__ bool argmax_better(float x, int v, float bx, int bv) {
  return x > bx || (x == bx && v < bv);
}

__device__ __forceinline__ void warp_argmax(float &best, int &idx) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_xor_sync(kFull, best, o);
    const int oi = __shfl_xor_sync(kFull, idx, o);
    if (argmax_better(ob, oi, best, idx)) {
      best = ob;
      idx = oi;
    }
  }
}

// Boosted rerank order (R6): higher fused score, then higher raw logprob,
// then lower token id (_kernels.pyx:197-200, decoding.py:129-149).
__device__ __forceinline__ bool rerank_better(double c, float lp, int v, double bc, float blp, int bv) {
  if (c != bc) return c > bc;
  if (lp != blp) return lp > blp;
  return v < bv;
}

// fp64 shallow fusion lp + lam * s, two separately rounded ops (no FMA),
// as the reference computes it (_kernels.pyx:176, :197; decoding.py:140).
__device__ __forceinline__ double fuse(float lp, double lam, float s) {
  return __dadd_rn(static_cast<double>(lp), __dmul_rn(lam, static_cast<double>(s)));
}

}  // namespace pgpb
