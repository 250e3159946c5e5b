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

// Order-preserving unsigned key of a double (NaN excluded), -0.0 folded onto
// +0.0 so equal values compare equal as in cand_better.
__device__ __forceinline__ unsigned long long cand_dkey(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(x, 0.0)));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Warp argmax in cand_better's order with hardware reductions: the 64-bit
// key's two halves by redux.sync, am and then cid only among exact key ties,
// the winner shuffled from its lane (three shuffles instead of five
// butterfly levels of compares and fifteen shuffles).  Every lane returns it.
__device__ __forceinline__ Cand cand_warp_best(const Cand &mine) {
  const bool has = mine.cid != INT_MAX;
  const unsigned long long k = has ? cand_dkey(mine.key) : 0ull;
  const unsigned hi = unsigned(k >> 32), lo = unsigned(k);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  unsigned tie = __ballot_sync(0xffffffffu, has && hi == mhi && lo == mlo);
  if (__popc(tie) > 1) {
    const bool in = (tie >> (threadIdx.x & 31)) & 1u;
    const unsigned long long a = in ? cand_dkey(mine.am) : 0ull;
    const unsigned ahi = unsigned(a >> 32), alo = unsigned(a);
    const unsigned mahi = __reduce_max_sync(0xffffffffu, ahi);
    const unsigned malo = __reduce_max_sync(0xffffffffu, ahi == mahi ? alo : 0u);
    tie = __ballot_sync(0xffffffffu, in && ahi == mahi && alo == malo);
    if (__popc(tie) > 1) {
      const bool in2 = (tie >> (threadIdx.x & 31)) & 1u;
      const unsigned mc = __reduce_min_sync(0xffffffffu, in2 ? unsigned(mine.cid) : 0xffffffffu);
      tie = __ballot_sync(0xffffffffu, in2 && unsigned(mine.cid) == mc);
    }
  }
  const int src = tie ? __ffs(tie) - 1 : 0;
  Cand w;
  w.key = __shfl_sync(0xffffffffu, mine.key, src);
  w.am = __shfl_sync(0xffffffffu, mine.am, src);
  w.cid = __shfl_sync(0xffffffffu, mine.cid, src);
  return w;
}

// Warp-level merge of nw <= 32 per-warp top-k lists s_wl[w * k + i] (each
// sorted best first, empty entries cid == INT_MAX) into the block's top k:
// lane w holds warp w's current head, each round takes the warp best and the
// winning lane advances — no re-insertion of the nw * k entries.
__device__ __forceinline__ void merge_warp_lists(const Cand *s_wl, int nw, int k, int lane, int *s_win,
                                                 double *s_key, double *s_am) {
  const Cand none{-INFINITY, -INFINITY, INT_MAX};
  int ptr = 0;
  Cand head = lane < nw ? s_wl[lane * k] : none;
  for (int r = 0; r < k; ++r) {
    const Cand best = cand_warp_best(head);
    if (lane == 0) {
      s_win[r] = best.cid;
      s_key[r] = best.key;
      s_am[r] = best.am;
    }
    if (best.cid != INT_MAX && head.cid == best.cid) {
      ++ptr;
      head = ptr < k ? s_wl[lane * k + ptr] : none;
    }
  }
}

// Candidate whose ranking key is pre-folded to its order-preserving integer
// image (cand_dkey; 0 = empty): the per-thread list insertions and the warp
// reductions compare 64-bit integers, predicated, instead of chains of fp64
// compares whose per-lane outcomes diverge the warp; am and then cid only
// break exact key ties, so the order is cand_better's.
struct KCand {
  unsigned long long k;
  double am;
  int cid;
};

__device__ __forceinline__ KCand kcand(double key, double am, int cid) { return KCand{cand_dkey(key), am, cid}; }
__device__ __forceinline__ KCand kcand_none() { return KCand{0ull, -INFINITY, INT_MAX}; }

// Inverse of cand_dkey (-0.0 comes back as +0.0).
__device__ __forceinline__ double kcand_key(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

__device__ __forceinline__ bool kc_better(const KCand &a, const KCand &b) {
  if (a.k != b.k) return a.k > b.k;
  if (a.am != b.am) return a.am > b.am;
  return a.cid < b.cid;
}

template <int K>
__device__ __forceinline__ void klist_insert(KCand (&l)[K], const KCand &c) {
  if (!kc_better(c, l[K - 1])) return;
  l[K - 1] = c;
#pragma unroll
  for (int i = K - 1; i > 0; --i) {
    const bool sw = kc_better(l[i], l[i - 1]);
    const KCand x = l[i], y = l[i - 1];
    l[i - 1].k = sw ? x.k : y.k;
    l[i - 1].am = sw ? x.am : y.am;
    l[i - 1].cid = sw ? x.cid : y.cid;
    l[i].k = sw ? y.k : x.k;
    l[i].am = sw ? y.am : x.am;
    l[i].cid = sw ? y.cid : x.cid;
  }
}

template <int K>
__device__ __forceinline__ void klist_pop(KCand (&l)[K]) {
#pragma unroll
  for (int i = 0; i < K - 1; ++i) l[i] = l[i + 1];
  l[K - 1] = kcand_none();
}

// cand_warp_best on pre-folded keys.
__device__ __forceinline__ KCand kc_warp_best(const KCand &mine) {
  const bool has = mine.cid != INT_MAX;
  const unsigned long long k = has ? mine.k : 0ull;
  const unsigned hi = unsigned(k >> 32), lo = unsigned(k);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  unsigned tie = __ballot_sync(0xffffffffu, has && hi == mhi && lo == mlo);
  if (__popc(tie) > 1) {
    const bool in = (tie >> (threadIdx.x & 31)) & 1u;
    const unsigned long long a = in ? cand_dkey(mine.am) : 0ull;
    const unsigned ahi = unsigned(a >> 32), alo = unsigned(a);
    const unsigned mahi = __reduce_max_sync(0xffffffffu, ahi);
    const unsigned malo = __reduce_max_sync(0xffffffffu, ahi == mahi ? alo : 0u);
    tie = __ballot_sync(0xffffffffu, in && ahi == mahi && alo == malo);
    if (__popc(tie) > 1) {
      const bool in2 = (tie >> (threadIdx.x & 31)) & 1u;
      const unsigned mc = __reduce_min_sync(0xffffffffu, in2 ? unsigned(mine.cid) : 0xffffffffu);
      tie = __ballot_sync(0xffffffffu, in2 && unsigned(mine.cid) == mc);
    }
  }
  const int src = tie ? __ffs(tie) - 1 : 0;
  KCand w;
  w.k = __shfl_sync(0xffffffffu, mine.k, src);
  w.am = __shfl_sync(0xffffffffu, mine.am, src);
  w.cid = __shfl_sync(0xffffffffu, mine.cid, src);
  return w;
}

// merge_warp_lists on pre-folded keys.
__device__ __forceinline__ void kmerge_warp_lists(const KCand *s_wl, int nw, int k, int lane, int *s_win,
                                                  double *s_key, double *s_am) {
  int ptr = 0;
  KCand head = lane < nw ? s_wl[lane * k] : kcand_none();
  for (int r = 0; r < k; ++r) {
    const KCand best = kc_warp_best(head);
    if (lane == 0) {
      s_win[r] = best.cid;
      s_key[r] = best.cid != INT_MAX ? kcand_key(best.k) : -INFINITY;
      s_am[r] = best.am;
    }
    if (best.cid != INT_MAX && head.cid == best.cid) {
      ++ptr;
      head = ptr < k ? s_wl[lane * k + ptr] : kcand_none();
    }
  }
}

// Order-preserving u32 image of a float (NaN excluded) and its inverse.
__device__ __forceinline__ unsigned ford(float x) {
  const unsigned u = __float_as_uint(x);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ford_inv(unsigned k) { return __uint_as_float((k >> 31) ? (k & 0x7FFFFFFFu) : ~k); }

// k-th largest (1-based, counted with multiplicity) of the lanes' x, k <= 32;
// -inf when fewer than k lanes remain.  All 32 lanes must call it.
__device__ __forceinline__ float warp_kth_max(float x, int k) {
  unsigned u = ford(x), m = 0u;
  for (int r = 0; r < k; ++r) {
    m = __reduce_max_sync(0xffffffffu, u);
    const unsigned b = __ballot_sync(0xffffffffu, u == m);
    if (int(threadIdx.x & 31) == __ffs(b) - 1) u = 0u;
  }
  return m ? ford_inv(m) : -INFINITY;
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
