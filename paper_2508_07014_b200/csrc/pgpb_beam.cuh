// Candidate lists and cell resolution shared by the beam kernels.
#pragma once

#include "pgpb_common.cuh"

namespace pgpb {

constexpr int kBeamThreads = 256;
constexpr int kMaxTopK = 32;  // winners per merge pass (and the device beams' beam cap)

struct Cand {
  double key;
  double am;
  int cid;  // h_local * V + v; INT_MAX = empty
};

__device__ __forceinline__ bool cand_better(const Cand &a, const Cand &b) {
  if (a.key != b.key) return a.key > b.key;
  if (a.am != b.am) return a.am > b.am;
  return a.cid < b.cid;
}

template <int K>
__device__ __forceinline__ void list_insert(Cand (&l)[K], const Cand &c) {
  if (!cand_better(c, l[K - 1])) return;
  l[K - 1] = c;
#pragma unroll
  for (int i = K - 1; i > 0; --i) {
    if (cand_better(l[i], l[i - 1])) {
      Cand t = l[i];
      l[i] = l[i - 1];
      l[i - 1] = t;
    }
  }
}

template <int K>
__device__ __forceinline__ void list_pop(Cand (&l)[K]) {
#pragma unroll
  for (int i = 0; i < K - 1; ++i) l[i] = l[i + 1];
  l[K - 1] = Cand{-INFINITY, -INFINITY, INT_MAX};
}

__device__ __forceinline__ Cand shfl_cand(const Cand &c, int o) {
  Cand r;
  r.key = __shfl_xor_sync(kFull, c.key, o);
  r.am = __shfl_xor_sync(kFull, c.am, o);
  r.cid = __shfl_xor_sync(kFull, c.cid, o);
  return r;
}

// Resolve (score, next) of token v at a state via closure binary search.
__device__ __forceinline__ void resolve_cell(const TableView &t, const float *root, const int32_t *rnext,
                                             int state, int v, float &s, int &nx) {
  const int4 rec = __ldg(t.clo_rec + state);
  int lo = rec.x, hi = rec.x + rec.y;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&t.clo[mid].x) < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < rec.x + rec.y && __ldg(&t.clo[lo].x) == v) {
    const int4 e = __ldg(t.clo + lo);
    s = __int_as_float(e.z);
    nx = e.y;
  } else {
    s = __int_as_float(rec.z) + root[v];
    nx = rnext[v];
  }
}

// Resolve (score, next) of token v at a state whose closure tokens are set
// in the shared-memory bitmap bm_h (its closure record rec, loaded already):
// a closure token's entry is the rank(v)-th of the state's sorted closure
// (popcounts over the bitmap), so the lookup costs one load instead of the
// binary search's dependent chain; a dense token reads the root row.
__device__ __forceinline__ void resolve_ranked(const TableView &t, const float *root, const unsigned *bm_h,
                                               const int4 &rec, int v, float &s, int &nx) {
  const int wv = v >> 5;
  const unsigned w = bm_h[wv];
  if ((w >> (v & 31)) & 1u) {
    int rank = __popc(w & ((1u << (v & 31)) - 1u));
    for (int q = 0; q < wv; ++q) rank += __popc(bm_h[q]);
    const int4 e = __ldg(t.clo + rec.x + rank);
    s = __int_as_float(e.z);
    nx = e.y;
  } else {
    s = __int_as_float(rec.z) + root[v];
    nx = __ldg(t.root_next + v);
  }
}

}  // namespace pgpb
