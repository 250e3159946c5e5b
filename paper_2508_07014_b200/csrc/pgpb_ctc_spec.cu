// Greedy CTC with boosting: HBM-bound top-2 pass + speculative chunk-parallel
// walker.  This is the production pgpb_ctc_greedy.
//
// Reference: _kernels.ctc_greedy (_kernels.pyx:75-225) / ctc_greedy_boosted
// (decoding.py:156-229), R6 in SURVEY.md.  Per utterance the decision at an
// emitting frame depends on the tree state and the previous symbol, which
// depend on every earlier decision: a sequential recurrence.
//
//  Phase A  frame_top2_kernel: every SM, one warp per frame (two rows in
//           flight per warp), each row streamed once from HBM and reduced to
//           {argmax a, lp_a, runner-up t2, lp_2} (16 bytes per frame).
//           Unboosted: the argmax only.
//
//  Phase B  ctc_walk_kernel: one CTA per utterance (grid-stride), the
//           frame records staged in shared memory.  Lane c of the CTA owns
//           chunk c (L contiguous frames).
//           Round 0: every lane walks its chunk from a guessed start
//           (root, last = -1) and records the inputs (state, last) of every
//           frame.  Fix-up rounds: a lane whose start differs from its left
//           neighbour's end re-walks from the true start and stops at the
//           first frame whose recorded inputs it reproduces (everything after
//           is then unchanged); if it reaches its chunk's end it runs on into
//           the following chunks whose lanes are idle in this round.  Lane 0
//           is exact from round 0, so the loop terminates, and it stops when
//           no start changed: every chunk is then consistent with the exact
//           sequential decode.  On peaky emissions (blank-dominated, boosting
//           rarely flips a decision: the reference's own decode-overhead
//           benchmark, test_acceptance.py:342-378) walks resynchronise
//           within one emission and one fix-up round suffices; when boosting
//           flips most decisions the fix-ups degrade to sequential walks,
//           which then use the whole warp per step.
//           Tail: am / boost as exact grid sums (every partial sum
//           representable, checked, so equal to the reference's frame-order
//           fp64 sums) with a sequential fallback; emitted frames compacted
//           by a block scan.  Long utterances run in segments whose exact end
//           state seeds the next segment's first chunk.
//
// Rerank at (state, frame) by one lane: the state's blob (header + closure
// arcs with exact fp32 scores, sorted by token) is read with one load batch
// (the following lines L1-prefetched) and scanned twice.  Pass 1 finds
// whether a / t2 are closure tokens and scores them exactly; the dense
// candidates among {a, t2} use acc + root[v].  Pass 2: every other arc's
// token ranks after t2 in (lp desc, id asc), so its fused score is at most
// fuse(lp_2, lam, s); it is skipped when the best candidate beats that tuple,
// and only survivors gather their log-prob (one batched load).  Dense tokens
// outside {a, t2} rank after the frontier token, so fuse(lp_f, lam, acc +
// max_root) bounds them (every rounded op is monotone); a winner that does
// not beat that tuple, or a closure too large for the lane's registers, is
// decided by the whole warp (same two passes lane-parallel, then a full-row
// rescan as the last resort).
//
// Bit-exact with the reference: first-max argmax, fp64 fusion lp + lam*s as
// two rounded ops (no FMA), rerank ties -> higher lp -> lower id.

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "pgpb_rerank.cuh"

namespace pgpb {
namespace cw {

#ifdef PGPB_SEQ_PROFILE
// Debug-only counters (pgpb_debug_ctc_fused_profile): [0] fix-up rounds,
// [1] round-0 lane steps, [2] fix-up lane steps, [3] warp decisions,
// [4] full rescans, [6..8] CTA-0 cycles to round 0 done / fix-ups done /
// tail done, [9] segments, [10] gathered closure arcs, [11..12] CTA-0 lane-0
// lane decisions and their cycles, [13] CTA-0 ordered-sum cycles,
// [14..15] CTA-0 warp decisions and their cycles.
__device__ unsigned long long g_cf_prof[256];
#define CF_COUNT(i, n) \
  do { if (blockIdx.x == 0) atomicAdd(&g_cf_prof[i], (unsigned long long)(n)); } while (0)
// CTA-0 timeline: [200+i] = max over threads of cycles since kernel entry
#define CF_MARK(i)                                                                                  \
  do {                                                                                              \
    if (blockIdx.x == 0 && int(threadIdx.x >> 5) < W) { /* walker warps only */                      \
      const unsigned m_ = __activemask();                                                           \
      const unsigned v_ = __reduce_max_sync(m_, unsigned(clock64() - t_entry));                     \
      if ((threadIdx.x & 31) == __ffs(m_) - 1) atomicMax(&g_cf_prof[200 + (i) + 20 * cf_rep], (unsigned long long)v_); \
    }                                                                                               \
  } while (0)
#else
#define CF_MARK(i) \
  do {             \
  } while (0)
#define CF_COUNT(i, n) \
  do {                 \
  } while (0)
#endif

constexpr int kMaxConsumers = 7;  // walker warps (+1 helper warp): 256 threads
constexpr int kLaneArcs = 31;   // lane decisions up to 31 closure arcs (header + 31 = 512 B), larger -> warp

constexpr int kSmemBudget = 96 * 1024;

// Table reads of the walker carry an L2 evict-last hint: the tree's hot
// lines (depth-1 states, their bitmaps) outlive phase A's evict-first stream
// of log-probs, so the next call's dependent round trips hit L2.
#ifndef PGPB_NO_L2_HINT
__device__ __forceinline__ uint64_t el_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 tab_ld(const int4 *a) {
  int4 v;
  asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(a), "l"(el_policy()));
  return v;
}
__device__ __forceinline__ int tab_ld(const int *a) {
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(el_policy()));
  return v;
}
__device__ __forceinline__ uint2 tab_ld(const uint2 *a) {
  uint2 v;
  asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(el_policy()));
  return v;
}
__device__ __forceinline__ uint32_t tab_ld(const uint32_t *a) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(el_policy()));
  return v;
}
#else
template <typename P>
__device__ __forceinline__ P tab_ld(const P *a) {
  return __ldg(a);
}
#endif

// ---------------------------------------------------------------------------
// Phase A

// Running first-max of one insertion chain (ids ascending within a chain).
struct Top1 {
  float m = -INFINITY;
  int i = INT_MAX;
  __device__ __forceinline__ void ins(float x, int v) {
    if (argmax_better(x, v, m, i)) {
      m = x;
      i = v;
    }
  }
  __device__ __forceinline__ void merge(const Top1 &o) { ins(o.m, o.i); }
};

// Per-lane maxima of the four insertion chains of a register row.
struct Chains4 {
  float m[4];
  int i[4];
};

// This lane's first max of the row without token j1: its chain maxima other
// than j1's, and, in the one lane owning j1, a rescan of j1's chain only.
template <int NV>
__device__ __forceinline__ void lane_runner_up(const float (&x)[NV], const int (&id)[NV], const Chains4 &r, int j1,
                                               float &b, int &j) {
  b = -INFINITY;
  j = INT_MAX;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (r.i[c] != j1 && argmax_better(r.m[c], r.i[c], b, j)) {
      b = r.m[c];
      j = r.i[c];
    }
  const int cs = r.i[0] == j1 ? 0 : r.i[1] == j1 ? 1 : r.i[2] == j1 ? 2 : r.i[3] == j1 ? 3 : -1;
  if (cs >= 0) {  // divergent: one lane
    auto scan = [&](auto cc) {
      constexpr int c = decltype(cc)::value;
#pragma unroll
      for (int k = c; k < NV; k += 4)
        if (id[k] != j1 && argmax_better(x[k], id[k], b, j)) {
          b = x[k];
          j = id[k];
        }
    };
    switch (cs) {
      case 0: scan(std::integral_constant<int, 0>{}); break;
      case 1: scan(std::integral_constant<int, 1>{}); break;
      case 2: scan(std::integral_constant<int, 2>{}); break;
      default: scan(std::integral_constant<int, 3>{}); break;
    }
  }
}

// Row reduction over values already in registers: first max (a, lp_a) and,
// only when a is not the blank (a blank frame never emits, R6), the first max
// of the rest (t2, lp_2).  Four independent insertion chains per lane keep the
// compare chains short (ids ascend within every chain); the runner-up comes
// from the chain maxima other than a's plus, in the one lane owning a, a
// rescan of a's chain only.
template <int NV>
__device__ __forceinline__ int4 reduce_row(const float (&x)[NV], const int (&id)[NV], bool top2, int blank) {
  Top1 r[4];
#pragma unroll
  for (int k = 0; k < NV; ++k) r[k & 3].ins(x[k], id[k]);
  Chains4 ch;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    ch.m[c] = r[c].m;
    ch.i[c] = r[c].i;
  }
  r[0].merge(r[1]);
  r[2].merge(r[3]);
  r[0].merge(r[2]);
  float b1 = r[0].m;
  int j1 = r[0].i;
  warp_argmax(b1, j1);
  float b2 = -INFINITY;
  int j2 = INT_MAX;
  if (top2 && j1 != blank) {
    lane_runner_up(x, id, ch, j1, b2, j2);
    warp_argmax(b2, j2);
  }
  return make_int4(j1, __float_as_int(b1), j2, __float_as_int(b2));
}

// Row reduction with warp reductions in hardware (redux.sync, CREDUX):
// per lane, maxima of four groups of 8 consecutive register elements (ids
// ascend with the element index, so groups ascend too), the warp max M by
// redux.max.f32, then the first element equal to M is searched only in the
// first group whose max equals M (usually in one lane) and the warp's first
// such id by redux.min.  The runner-up (only when a != blank) repeats this
// over the row without a: the owning lane's candidate is its other groups'
// maxima plus a rescan of a's group.  Values stored are the matched elements
// themselves (exact bits, so -0.0 stays -0.0).  Record halves {a, lp_a} and
// {t2, lp_2} are stored by the lanes that own them.
template <int Q>
__device__ __forceinline__ float gmax(const float (&x)[32]) {
  const float a = fmaxf(x[8 * Q], x[8 * Q + 1]), b = fmaxf(x[8 * Q + 2], x[8 * Q + 3]);
  const float c = fmaxf(x[8 * Q + 4], x[8 * Q + 5]), d = fmaxf(x[8 * Q + 6], x[8 * Q + 7]);
  return fmaxf(fmaxf(a, b), fmaxf(c, d));
}

template <int Q>
__device__ __forceinline__ float gmax_ex(const float (&x)[32], const int (&id)[32], int ex) {
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) y[k] = id[8 * Q + k] == ex ? -INFINITY : x[8 * Q + k];
  return fmaxf(fmaxf(fmaxf(y[0], y[1]), fmaxf(y[2], y[3])), fmaxf(fmaxf(y[4], y[5]), fmaxf(y[6], y[7])));
}

// first element of group Q equal to v whose id is not ex (INT_MAX if none)
template <int Q>
__device__ __forceinline__ int gfind(const float (&x)[32], const int (&id)[32], float v, int ex, float &val) {
  int r = INT_MAX;
  float rv = v;
#pragma unroll
  for (int k = 8 * Q + 7; k >= 8 * Q; --k)
    if (x[k] == v && id[k] != ex) {
      r = id[k];
      rv = x[k];
    }
  val = rv;
  return r;
}

__device__ __forceinline__ int lane_find(const float (&x)[32], const int (&id)[32], const float (&g)[4], float v,
                                         int ex, float &val, int &grp) {
  int r = INT_MAX;
  grp = -1;
  if (g[0] == v) {
    r = gfind<0>(x, id, v, ex, val);
    grp = 0;
  }
  if (r == INT_MAX && g[1] == v) {
    r = gfind<1>(x, id, v, ex, val);
    grp = 1;
  }
  if (r == INT_MAX && g[2] == v) {
    r = gfind<2>(x, id, v, ex, val);
    grp = 2;
  }
  if (r == INT_MAX && g[3] == v) {
    r = gfind<3>(x, id, v, ex, val);
    grp = 3;
  }
  return r;
}

__device__ __forceinline__ float redux_max_f32(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ void reduce_row_rx(const float (&x)[32], const int (&id)[32], bool top2, int blank,
                                              int lane, int2 *rec, bool store) {
  float g[4];
  g[0] = gmax<0>(x);
  g[1] = gmax<1>(x);
  g[2] = gmax<2>(x);
  g[3] = gmax<3>(x);
  const float lm = fmaxf(fmaxf(g[0], g[1]), fmaxf(g[2], g[3]));
  const float M = redux_max_f32(lm);
  int li = INT_MAX, grp = -1;
  float lv = M;
  if (lm == M) li = lane_find(x, id, g, M, INT_MAX, lv, grp);
  const int j1 = int(__reduce_min_sync(kFull, unsigned(li)));
  const bool own = li == j1;
  if (store && own) rec[0] = make_int2(j1, __float_as_int(lv));
  if (!top2) return;
  if (j1 == blank) {
    if (store && lane == 0) rec[1] = make_int2(INT_MAX, __float_as_int(-INFINITY));
    return;
  }
  // group maxima of the row without a (differs from g in a's group only)
  float h[4] = {g[0], g[1], g[2], g[3]};
  float m2 = lm;
  if (own) {  // divergent: one lane
    switch (grp) {
      case 0: h[0] = gmax_ex<0>(x, id, j1); break;
      case 1: h[1] = gmax_ex<1>(x, id, j1); break;
      case 2: h[2] = gmax_ex<2>(x, id, j1); break;
      default: h[3] = gmax_ex<3>(x, id, j1); break;
    }
    m2 = fmaxf(fmaxf(h[0], h[1]), fmaxf(h[2], h[3]));
  }
  const float M2 = redux_max_f32(m2);
  int li2 = INT_MAX, grp2;
  float lv2 = M2;
  if (m2 == M2) li2 = lane_find(x, id, h, M2, j1, lv2, grp2);
  const int j2 = int(__reduce_min_sync(kFull, unsigned(li2)));
  if (store) {
    if (j2 == INT_MAX) {  // no runner-up (V == 1)
      if (lane == 0) rec[1] = make_int2(INT_MAX, __float_as_int(-INFINITY));
    } else if (li2 == j2) {
      rec[1] = make_int2(j2, __float_as_int(lv2));
    }
  }
}

// One warp reduces frames f and f + 1 (when valid) with both rows loaded
// before any compare (16 float4 per lane in flight), streamed with an
// evict-first hint so the table stays in L2 for the walker.  V <= 1024 is a
// single register tile; larger vocabularies loop over tiles with running
// chains merged across tiles.
template <bool kTop2, bool kVec>
__global__ void __launch_bounds__(256) frame_top2_kernel(const float *__restrict__ lp, int64_t B, int64_t T, int V,
                                                         const int32_t *__restrict__ lengths, int blank,
                                                         int4 *__restrict__ top) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t F = B * T;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t p = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; 2 * p < F; p += nwarps) {
    const int64_t f0 = 2 * p, f1 = 2 * p + 1;
    bool v0 = true, v1 = f1 < F;
    if (lengths) {
      const int64_t b0 = f0 / T;
      v0 = f0 - b0 * T < __ldg(lengths + b0);
      if (v1) {
        const int64_t b1 = f1 / T;
        v1 = f1 - b1 * T < __ldg(lengths + b1);
      }
    }
    if (!v0 && !v1) continue;
    if (kVec && V <= 1024) {
      const float4 *row0 = reinterpret_cast<const float4 *>(lp + f0 * V);
      const float4 *row1 = reinterpret_cast<const float4 *>(lp + f1 * V);
      const int V4 = V >> 2;
      const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      float4 x0[8], x1[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = lane + 32 * k;
        x0[k] = (v0 && c < V4) ? __ldcs(row0 + c) : ninf;
        x1[k] = (v1 && c < V4) ? __ldcs(row1 + c) : ninf;
      }
      float y0[32], y1[32];
      int id[32];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = lane + 32 * k;
        const bool ok = c < V4;
        id[4 * k] = ok ? 4 * c : INT_MAX;
        id[4 * k + 1] = ok ? 4 * c + 1 : INT_MAX;
        id[4 * k + 2] = ok ? 4 * c + 2 : INT_MAX;
        id[4 * k + 3] = ok ? 4 * c + 3 : INT_MAX;
        y0[4 * k] = x0[k].x;
        y0[4 * k + 1] = x0[k].y;
        y0[4 * k + 2] = x0[k].z;
        y0[4 * k + 3] = x0[k].w;
        y1[4 * k] = x1[k].x;
        y1[4 * k + 1] = x1[k].y;
        y1[4 * k + 2] = x1[k].z;
        y1[4 * k + 3] = x1[k].w;
      }
#ifdef PGPB_A_CHAINS
      const int4 o0 = reduce_row<32>(y0, id, kTop2, blank);
      const int4 o1 = reduce_row<32>(y1, id, kTop2, blank);
      if (lane == 0 && v0) top[f0] = o0;
      if (lane == 1 && v1) top[f1] = o1;
#else
      reduce_row_rx(y0, id, kTop2, blank, lane, reinterpret_cast<int2 *>(top + f0), v0);
      reduce_row_rx(y1, id, kTop2, blank, lane, reinterpret_cast<int2 *>(top + f1), v1);
#endif
    } else {
      // general path: scalar loads, tiles of 256 values per lane-chain set
      for (int r = 0; r < 2; ++r) {
        const int64_t f = r ? f1 : f0;
        if (!(r ? v1 : v0)) continue;
        const float *row = lp + f * V;
        Top1 c1[4];
        for (int base = 0; base < V; base += 256) {
          float xv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int v = base + lane + 32 * k;
            xv[k] = v < V ? __ldcs(row + v) : -INFINITY;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int v = base + lane + 32 * k;
            if (v < V) c1[k & 3].ins(xv[k], v);
          }
        }
        c1[0].merge(c1[1]);
        c1[2].merge(c1[3]);
        c1[0].merge(c1[2]);
        float b1 = c1[0].m;
        int j1 = c1[0].i;
        warp_argmax(b1, j1);
        float b2 = -INFINITY;
        int j2 = INT_MAX;
        if (kTop2 && j1 != blank) {
          Top1 c2[4];
          for (int base = 0; base < V; base += 256) {
            float xv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int v = base + lane + 32 * k;
              xv[k] = v < V ? __ldg(row + v) : -INFINITY;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int v = base + lane + 32 * k;
              if (v < V && v != j1) c2[k & 3].ins(xv[k], v);
            }
          }
          c2[0].merge(c2[1]);
          c2[2].merge(c2[3]);
          c2[0].merge(c2[2]);
          b2 = c2[0].m;
          j2 = c2[0].i;
          warp_argmax(b2, j2);
        }
        if (lane == 0) top[f] = make_int4(j1, __float_as_int(b1), j2, __float_as_int(b2));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Phase B

struct Args {
  TableView t;
  const float *lp;
  const int4 *top;  // [B*T] {a, lp_a, t2, lp_2}
  int64_t B, T;
  int V;
  const int32_t *lengths;
  int blank;
  double lam;
  int use_boost;
  int TS;        // frames per segment
  int seq_mode;  // 0 auto, 1 always sequential, 2 never
  int32_t *tokens;
  double *deltas;
  int32_t *ostates;
  int32_t *nout;
  double *am_out;
  double *boost_out;
};

struct Smem {
  float *root;
  int32_t *rnext, *rnoff;
  unsigned *bm;  // [W][Vw]
  int32_t *fa, *ft2, *in_off, *in_last, *o_tok, *o_nx;
  float *flpa, *flp2, *o_s, *o_lp;
  int32_t *c_soff, *c_slast, *c_eoff, *c_elast, *c_act, *c_sst, *c_est;  // [C]
  int32_t *misc;  // [0] seg start off, [1] seg start last, [2] emitted so far, [3] seg start state,
                  // [4] first frame whose walked log-prob differs from its argmax's
  double *dsum;   // [0] am, [1] boost: running totals across segments
  int32_t *wsum;  // [33] scan scratch
  double *wred;   // [warp][4] tail partials: am sum, am |sum|, boost sum, boost |sum|
  int32_t *wmin;  // [warp][4] tail minima: am grid exponent, boost grid exponent
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t smem_bytes(int Vp, int Vw, int W, int TS, int use_boost, Smem *s,
                                             unsigned char *base) {
  const int C = 32 * W;
  const size_t vb = use_boost ? size_t(Vp) * 4 : 0, fb = align16(size_t(TS) * 4),
               cb = align16(size_t(C + 32) * 4);  // + the accountant warp's (never live) lanes
  size_t o = 0;
#define PGPB_TAKE(field, type, bytes)                     \
  do {                                                    \
    if (s) s->field = reinterpret_cast<type *>(base + o); \
    o += align16(bytes);                                  \
  } while (0)
  PGPB_TAKE(root, float, vb);
  PGPB_TAKE(rnext, int32_t, vb);
  PGPB_TAKE(rnoff, int32_t, vb);
  PGPB_TAKE(bm, unsigned, use_boost ? size_t(W) * Vw * 4 : 0);
  PGPB_TAKE(fa, int32_t, fb);
  PGPB_TAKE(ft2, int32_t, use_boost ? fb : 0);
  PGPB_TAKE(in_off, int32_t, use_boost ? fb : 0);
  PGPB_TAKE(in_last, int32_t, use_boost ? fb : 0);
  PGPB_TAKE(o_tok, int32_t, fb);
  PGPB_TAKE(o_nx, int32_t, use_boost ? fb : 0);
  PGPB_TAKE(flpa, float, fb);
  PGPB_TAKE(flp2, float, use_boost ? fb : 0);
  PGPB_TAKE(o_s, float, use_boost ? fb : 0);
  PGPB_TAKE(o_lp, float, fb);
  PGPB_TAKE(c_soff, int32_t, cb);
  PGPB_TAKE(c_slast, int32_t, cb);
  PGPB_TAKE(c_eoff, int32_t, cb);
  PGPB_TAKE(c_elast, int32_t, cb);
  PGPB_TAKE(c_act, int32_t, cb);
  PGPB_TAKE(c_sst, int32_t, cb);
  PGPB_TAKE(c_est, int32_t, cb);
  PGPB_TAKE(misc, int32_t, 8 * 4);
  PGPB_TAKE(dsum, double, 2 * 8);
  PGPB_TAKE(wsum, int32_t, 33 * 4);
  PGPB_TAKE(wred, double, 4 * 8 * (kMaxConsumers + 1));
  PGPB_TAKE(wmin, int32_t, 4 * 4 * (kMaxConsumers + 1));
#undef PGPB_TAKE
  return o;
}

struct Ctx {
  const TableView *t;
  const Smem *s;
  const float *rows;  // row of local frame f at rows + f * V
  int V, blank;
  double lam;
  double inv_lam;  // 1 / lam (filter thresholds only; decisions use fuse())
  float max_root;
  int lane;
};

// Dense candidates among {a, t2} and the frontier token of the bound: every
// dense token not considered ranks after the frontier in (lp desc, id asc).
__device__ __forceinline__ void dense_part(const Ctx &x, BCand &best, float acc, int last, int a, float lpa, int t2,
                                           float lp2, bool a_in, bool t2_in, int &fid, float &flp) {
  const float *root = x.s->root;
  const int32_t *rnext = x.s->rnext, *rnoff = x.s->rnoff;
  if (!a_in) {
    const float s = acc + root[a];
    bcand_consider(best, fuse(lpa, x.lam, s), lpa, a, s, rnext[a], rnoff[a]);
    if (root[a] == x.max_root) {
      fid = a;
      flp = lpa;
      return;
    }
  }
  fid = t2;
  flp = lp2;
  if (t2 < x.V && !t2_in && t2 != x.blank && t2 != last) {
    const float s = acc + root[t2];
    bcand_consider(best, fuse(lp2, x.lam, s), lp2, t2, s, rnext[t2], rnoff[t2]);
  }
}

__device__ __forceinline__ bool certified(const Ctx &x, const BCand &best, float acc, int fid, float flp) {
  if (best.v == INT_MAX) return false;
  const double cb = fuse(flp, x.lam, acc + x.max_root);
  return !rerank_better(cb, flp, fid, best.c, best.lp, best.v);
}

// An arc that is neither a nor t2 ranks after t2: it can only win when the
// current best does not beat (fuse(lp_2, lam, s), lp_2, t2).
__device__ __forceinline__ bool may_win(const Ctx &x, const BCand &best, float sv, int t2, float lp2) {
  return !rerank_better(best.c, best.lp, best.v, fuse(lp2, x.lam, sv), lp2, t2);
}

// Thread-serial exact rerank at one emitting frame.  False: not decided here.
// Registers hold the tokens and scores of up to kLaneArcs arcs (one load
// batch); candidates carry the arc index (or -1 for a dense token) and only
// the winner's successor is resolved.
#ifdef PGPB_SEQ_PROFILE
__device__ int g_ld_n;
__device__ long long g_ld_rec[256][4];
#endif
__device__ __forceinline__ bool lane_decide_impl(const Ctx &x, const float *row, int off, int st, int last, int a,
                                                 float lpa, int t2, float lp2, BCand &out, int &path);
__device__ __forceinline__ bool lane_decide(const Ctx &x, const float *row, int off, int st, int last, int a,
                                            float lpa, int t2, float lp2, BCand &out) {
#ifdef PGPB_SEQ_PROFILE
  const long long t0 = clock64();
  int path = 0;
  const bool r = lane_decide_impl(x, row, off, st, last, a, lpa, t2, lp2, out, path);
  const long long dt = clock64() - t0;
  if (blockIdx.x == 0) {
    const int i = atomicAdd(&g_ld_n, 1);
    if (i < 256) {
      g_ld_rec[i][0] = dt;
      g_ld_rec[i][1] = __ldg(&x.t->blob[off].x);
      g_ld_rec[i][2] = path * 10 + (r ? 1 : 0);
      g_ld_rec[i][3] = threadIdx.x;
    }
  }
  atomicAdd(&g_cf_prof[160 + 2 * path + (r ? 1 : 0)], 1ull);
  return r;
#else
  int path = 0;
  return lane_decide_impl(x, row, off, st, last, a, lpa, t2, lp2, out, path);
#endif
}
__device__ __forceinline__ bool lane_decide_impl(const Ctx &x, const float *row, int off, int st, int last, int a,
                                                 float lpa, int t2, float lp2, BCand &out, int &path) {
  const int4 *blob = x.t->blob + off;
  const float *root = x.s->root;
  if (st == 0) {
    path = 5;
    // At the root the closure is the root row itself (shared memory): every
    // token scores acc + root[v] with acc = 0 and moves to rnext[v], so the
    // dense candidates {a, t2} and the frontier bound decide without a load.
    BCand best = bcand_none();
    bcand_consider(best, fuse(lpa, x.lam, root[a]), lpa, a, root[a], -1, 0);
    const bool amax = root[a] == x.max_root;
    if (!amax && t2 < x.V && t2 != x.blank && t2 != last)
      bcand_consider(best, fuse(lp2, x.lam, root[t2]), lp2, t2, root[t2], -1, 0);
    if (!certified(x, best, 0.0f, amax ? a : t2, amax ? lpa : lp2)) return false;
    out = best;
    out.nx = x.s->rnext[best.v];
    out.noff = x.s->rnoff[best.v];
    return true;
  }
  const int4 h = tab_ld(blob);
  if (x.t->clo_bits) {
    // Fast path, one round trip: neither a nor t2 is a closure token and no
    // closure arc scores high enough to beat the dense winner.
    const uint2 *wb = x.t->clo_bits + int64_t(st) * x.t->bits_words;
    const uint2 wa = tab_ld(wb + (a >> 5));
    const uint2 wt = t2 < x.V ? tab_ld(wb + (t2 >> 5)) : make_uint2(0u, 0u);
    const bool a_in = (wa.x >> (a & 31)) & 1u, t2_in = t2 < x.V && ((wt.x >> (t2 & 31)) & 1u);
    if (a_in || t2_in) {
      path = 3;
      // Semi-fast path: a and/or t2 are closure tokens.  Their arcs are
      // one load away (bitmap rank);
      // every other arc ranks after t2 and scores at most smax (header), so
      // when smax clears the crossing point of the bound the {a, t2}
      // candidates decide exactly, without scanning the closure.
      const float acc = __int_as_float(h.y), smax = __int_as_float(h.w);
      // the entry's index = the word's rank + closure tokens below v in it
      auto entry = [&](int v, uint2 w) {
        return tab_ld(blob + 1 + int(w.y) + __popc(w.x & ((1u << (v & 31)) - 1u)));
      };
      const int4 ea = a_in ? entry(a, wa) : make_int4(0, 0, 0, 0);
      const int4 et = t2_in ? entry(t2, wt) : make_int4(0, 0, 0, 0);
      BCand best = bcand_none();
      int fid;
      float flp;
      if (a_in) {
        const float sv = __int_as_float(ea.z);
        bcand_consider(best, fuse(lpa, x.lam, sv), lpa, a, sv, ea.y, ea.w);
        fid = t2;
        flp = lp2;
      } else {
        const float sv = acc + root[a];
        bcand_consider(best, fuse(lpa, x.lam, sv), lpa, a, sv, x.s->rnext[a], x.s->rnoff[a]);
        const bool amax = root[a] == x.max_root;
        fid = amax ? a : t2;
        flp = amax ? lpa : lp2;
      }
      if (t2 < x.V && t2 != x.blank && t2 != last) {
        if (t2_in) {
          const float sv = __int_as_float(et.z);
          bcand_consider(best, fuse(lp2, x.lam, sv), lp2, t2, sv, et.y, et.w);
        } else if (fid == t2) {
          const float sv = acc + root[t2];
          bcand_consider(best, fuse(lp2, x.lam, sv), lp2, t2, sv, x.s->rnext[t2], x.s->rnoff[t2]);
        }
      }
      if (x.lam > 0.0 && isfinite(best.c) && isfinite(lp2)) {
        const double sx = (best.c - static_cast<double>(lp2)) * x.inv_lam;  // threshold only: the margin covers the rounding
        const float s_lo = static_cast<float>(sx - (fabs(sx) * 1e-6 + 1e-6));
        if (smax < s_lo && certified(x, best, acc, fid, flp)) {
          out = best;
          return true;
        }
      }
    } else {
      const float acc = __int_as_float(h.y), smax = __int_as_float(h.w);
      BCand best = bcand_none();
      const float sa = acc + root[a];
      bcand_consider(best, fuse(lpa, x.lam, sa), lpa, a, sa, -1, 0);
      const bool amax = root[a] == x.max_root;
      const int fid = amax ? a : t2;
      const float flp = amax ? lpa : lp2;
      if (!amax && t2 < x.V && t2 != x.blank && t2 != last) {
        const float s2 = acc + root[t2];
        bcand_consider(best, fuse(lp2, x.lam, s2), lp2, t2, s2, -1, 0);
      }
      if (x.lam > 0.0 && isfinite(best.c) && isfinite(lp2)) {
        const double sx = (best.c - static_cast<double>(lp2)) * x.inv_lam;  // threshold only: the margin covers the rounding
        const float s_lo = static_cast<float>(sx - (fabs(sx) * 1e-6 + 1e-6));
        path = 1;
        if (smax < s_lo && certified(x, best, acc, fid, flp)) {
          path = 2;
          out = best;
          out.nx = x.s->rnext[best.v];
          out.noff = x.s->rnoff[best.v];
          return true;
        }
      }
    }
  }
  path += 8;
  int tok[kLaneArcs];
  float sc[kLaneArcs];
#pragma unroll
  for (int j = 0; j < kLaneArcs; ++j) {  // blob is padded: safe past the end
    const int4 e = tab_ld(blob + 1 + j);
    tok[j] = e.x;
    sc[j] = __int_as_float(e.z);
  }
  const int count = h.x;
  const float acc = __int_as_float(h.y);
  if (count > kLaneArcs) return false;
  int ja = -1, jt = -1;
  float sva = 0.0f, svt = 0.0f;
#pragma unroll
  for (int j = 0; j < kLaneArcs; ++j) {
    if (j < count && tok[j] == a) {
      ja = j;
      sva = sc[j];
    }
    if (j < count && tok[j] == t2) {
      jt = j;
      svt = sc[j];
    }
  }
  BCand best = bcand_none();
  int fid;
  float flp;
  if (ja >= 0) {
    const float sv = sva;
    bcand_consider(best, fuse(lpa, x.lam, sv), lpa, a, sv, ja, 0);
    fid = t2;
    flp = lp2;
  } else {
    const float sv = acc + root[a];
    bcand_consider(best, fuse(lpa, x.lam, sv), lpa, a, sv, -1, 0);
    fid = root[a] == x.max_root ? a : t2;
    flp = root[a] == x.max_root ? lpa : lp2;
  }
  if (t2 < x.V && t2 != x.blank && t2 != last && (jt >= 0 || ja >= 0 || fid == t2)) {
    const float sv = jt >= 0 ? svt : acc + root[t2];  // closure t2 always, dense t2 when it is the frontier
    bcand_consider(best, fuse(lp2, x.lam, sv), lp2, t2, sv, jt, 0);
  }
  // Every other arc ranks after t2: fuse(lp_2, lam, s) bounds it and the
  // bound is monotone in s, so arcs with s below s_lo cannot win (s_lo is
  // the crossing point minus a margin far above the fp64 rounding error).
  float s_lo = -INFINITY;
  if (x.lam > 0.0 && isfinite(best.c) && isfinite(lp2)) {
    const double sx = (best.c - static_cast<double>(lp2)) * x.inv_lam;  // threshold only: the margin covers the rounding
    s_lo = static_cast<float>(sx - (fabs(sx) * 1e-6 + 1e-6));
  }
  bool surv[kLaneArcs];
  float lv[kLaneArcs];
#pragma unroll
  for (int j = 0; j < kLaneArcs; ++j) {
    surv[j] = j < count && j != ja && j != jt && tok[j] != x.blank && tok[j] != last && sc[j] >= s_lo;
    if (surv[j]) surv[j] = !rerank_better(best.c, best.lp, best.v, fuse(lp2, x.lam, sc[j]), lp2, t2);
  }
#pragma unroll
  for (int j = 0; j < kLaneArcs; ++j) lv[j] = surv[j] ? __ldg(row + tok[j]) : 0.0f;
#pragma unroll
  for (int j = 0; j < kLaneArcs; ++j) {
    if (!surv[j]) continue;
    CF_COUNT(10, 1);
    bcand_consider(best, fuse(lv[j], x.lam, sc[j]), lv[j], tok[j], sc[j], j, 0);
  }
  if (!certified(x, best, acc, fid, flp)) return false;
  out = best;
  if (best.nx >= 0) {  // winner is an arc: its successor from the blob (L1 hit)
    const int4 e = tab_ld(blob + 1 + best.nx);
    out.nx = e.y;
    out.noff = e.w;
  } else {
    out.nx = x.s->rnext[best.v];
    out.noff = x.s->rnoff[best.v];
  }
  return true;
}

// Whole-warp exact rerank (all lanes, uniform arguments).  Up to 32 arcs:
// the header and every arc arrive in one round trip (lane i holds arc i),
// a / t2 are found by ballot and their scores broadcast, so the candidate
// set {a, t2} is built lane-uniformly; then each lane bounds its own arc and
// only survivors gather their log-prob; one warp reduction.  A winner that
// does not clear the frontier bound falls back to a full-row rescan with the
// warp's closure bitmap.
__device__ BCand warp_decide(const Ctx &x, unsigned *bm, const float *row, int off, int last, int a, float lpa, int t2,
                             float lp2) {
  const int lane = x.lane;
  const int4 *blob = x.t->blob + off;
  const int4 h = tab_ld(blob);
  const int4 e0 = tab_ld(blob + 1 + lane);  // same round trip as the header (blob is padded)
  const int count = h.x;
  const float acc = __int_as_float(h.y);
  const float *root = x.s->root;
  const int32_t *rnext = x.s->rnext, *rnoff = x.s->rnoff;
  if (lane == 0) CF_COUNT(3, 1);
#ifdef PGPB_SEQ_PROFILE
  if (lane == 0) atomicAdd(&g_cf_prof[192], 1ull);
#endif
  BCand w;
  int fid;
  float flp;
  if (count <= 32) {
    const bool mine_ok = lane < count;
    const unsigned ma = __ballot_sync(kFull, mine_ok && e0.x == a);
    const unsigned mt = __ballot_sync(kFull, mine_ok && e0.x == t2 && t2 < x.V);
    const int la = ma ? __ffs(ma) - 1 : 0, lt = mt ? __ffs(mt) - 1 : 0;
    const float sva = __int_as_float(__shfl_sync(kFull, e0.z, la));
    const int nxa = __shfl_sync(kFull, e0.y, la), noa = __shfl_sync(kFull, e0.w, la);
    const float svt = __int_as_float(__shfl_sync(kFull, e0.z, lt));
    const int nxt = __shfl_sync(kFull, e0.y, lt), not_ = __shfl_sync(kFull, e0.w, lt);
    BCand b = bcand_none();
    if (ma) {
      bcand_consider(b, fuse(lpa, x.lam, sva), lpa, a, sva, nxa, noa);
      fid = t2;
      flp = lp2;
    } else {
      const float sa = acc + root[a];
      bcand_consider(b, fuse(lpa, x.lam, sa), lpa, a, sa, rnext[a], rnoff[a]);
      const bool amax = root[a] == x.max_root;
      fid = amax ? a : t2;
      flp = amax ? lpa : lp2;
    }
    if (t2 < x.V && t2 != x.blank && t2 != last) {
      if (mt)
        bcand_consider(b, fuse(lp2, x.lam, svt), lp2, t2, svt, nxt, not_);
      else if (fid == t2)
        bcand_consider(b, fuse(lp2, x.lam, acc + root[t2]), lp2, t2, acc + root[t2], rnext[t2], rnoff[t2]);
    }
    // every other arc ranks after t2: bound it, gather the survivors
    BCand mine = bcand_none();
    const float sv = __int_as_float(e0.z);
    if (mine_ok && e0.x != a && e0.x != t2 && e0.x != x.blank && e0.x != last && may_win(x, b, sv, t2, lp2)) {
      const float lv = __ldg(row + e0.x);
      bcand_consider(mine, fuse(lv, x.lam, sv), lv, e0.x, sv, e0.y, e0.w);
    }
    w = b;
    if (__ballot_sync(kFull, mine.v != INT_MAX)) {
      const BCand wm = bcand_warp_best(mine);
      if (rerank_better(wm.c, wm.lp, wm.v, w.c, w.lp, w.v)) w = wm;
    }
  } else {
    BCand mine = bcand_none();
    bool a_l = false, t2_l = false;
    for (int i = lane; i < count; i += 32) {
      const int4 e = i == lane ? e0 : tab_ld(blob + 1 + i);
      if (e.x == a) {
        a_l = true;
        const float sv = __int_as_float(e.z);
        bcand_consider(mine, fuse(lpa, x.lam, sv), lpa, a, sv, e.y, e.w);
      } else if (e.x == t2) {
        t2_l = true;
        if (t2 != x.blank && t2 != last) {
          const float sv = __int_as_float(e.z);
          bcand_consider(mine, fuse(lp2, x.lam, sv), lp2, t2, sv, e.y, e.w);
        }
      }
    }
    const bool a_in = __ballot_sync(kFull, a_l) != 0u;
    const bool t2_in = __ballot_sync(kFull, t2_l) != 0u;
    if (lane == 0) {
      dense_part(x, mine, acc, last, a, lpa, t2, lp2, a_in, t2_in, fid, flp);
    } else {
      BCand dummy = bcand_none();
      dense_part(x, dummy, acc, last, a, lpa, t2, lp2, a_in, t2_in, fid, flp);
    }
    const BCand b1 = bcand_warp_best(mine);
    for (int i = lane; i < count; i += 32) {
      const int4 e = tab_ld(blob + 1 + i);  // L1 hit
      if (e.x == a || e.x == t2 || e.x == x.blank || e.x == last) continue;
      const float sv = __int_as_float(e.z);
      if (!may_win(x, b1, sv, t2, lp2)) continue;
      const float lv = __ldg(row + e.x);
      bcand_consider(mine, fuse(lv, x.lam, sv), lv, e.x, sv, e.y, e.w);
    }
    w = bcand_warp_best(mine);
  }
  if (certified(x, w, acc, fid, flp)) return w;
  if (lane == 0) CF_COUNT(4, 1);
#ifdef PGPB_SEQ_PROFILE
  if (lane == 0) atomicAdd(&g_cf_prof[193], 1ull);
#endif
  // full rescan: every dense token, then the closure arcs
  for (int i = lane; i < count; i += 32) {
    const int tok = tab_ld(&blob[1 + i].x);
    atomicOr(bm + (tok >> 5), 1u << (tok & 31));
  }
  __syncwarp();
  BCand full = bcand_none();
  for (int v = lane; v < x.V; v += 32) {
    if (v == x.blank || v == last || ((bm[v >> 5] >> (v & 31)) & 1u)) continue;
    const float lv = __ldg(row + v);
    const float s = acc + root[v];
    bcand_consider(full, fuse(lv, x.lam, s), lv, v, s, rnext[v], rnoff[v]);
  }
  for (int i = lane; i < count; i += 32) {
    const int4 e = tab_ld(blob + 1 + i);
    if (e.x == x.blank || e.x == last) continue;
    const float lv = __ldg(row + e.x);
    const float sv = __int_as_float(e.z);
    bcand_consider(full, fuse(lv, x.lam, sv), lv, e.x, sv, e.y, e.w);
  }
  w = bcand_warp_best(full);
  __syncwarp();
  for (int i = lane; i < count; i += 32) bm[tab_ld(&blob[1 + i].x) >> 5] = 0u;
  __syncwarp();
  return w;
}

// One walk step of every lane of a warp (warp-synchronous).  A lane with
// has == true processes local frame f from (off, st, last); each emitting
// lane decides alone and only the frames it cannot certify go to the warp.
#ifdef PGPB_SEQ_PROFILE
__device__ int g_cf_step;
#endif
// Blank and repeat frames from f on (no decision, no table access): record
// them as walk_step would and return the first frame that needs a decision
// (or fe).
__device__ __forceinline__ int pass_through(const Ctx &x, int f, int fe, int off, int &last) {
  const Smem &s = *x.s;
  for (; f < fe; ++f) {
    const int a = s.fa[f];
    if (a != x.blank && a != last) break;
    s.in_off[f] = off;
    s.in_last[f] = last;
    s.o_tok[f] = -1;
    s.o_lp[f] = s.flpa[f];
    last = a;
  }
  return f;
}

__device__ __forceinline__ void walk_step(const Ctx &x, unsigned *bm, bool has, int f, int &off, int &st,
                                          int &last) {
  const Smem &s = *x.s;
#ifdef PGPB_SEQ_PROFILE
  const long long t_step = clock64();
#endif
  BCand d = bcand_none();
  bool emit = false;
  int a = 0, t2 = 0;
  float lpa = 0.0f, lp2 = 0.0f;
  if (has) {
    a = s.fa[f];
    lpa = s.flpa[f];
    s.in_off[f] = off;
    s.in_last[f] = last;
    if (a == x.blank || a == last) {
      s.o_tok[f] = -1;
      s.o_lp[f] = lpa;
      last = a;
    } else {
      emit = true;
      t2 = s.ft2[f];
      lp2 = s.flp2[f];
    }
  }
  const unsigned em = __ballot_sync(kFull, emit);
  bool need = emit;
  if (emit) {
#ifdef PGPB_SEQ_PROFILE
    const long long t0 = clock64();
#endif
    need = !lane_decide(x, x.rows + int64_t(f) * x.V, off, st, last, a, lpa, t2, lp2, d);
#ifdef PGPB_SEQ_PROFILE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      CF_COUNT(11, 1);
      CF_COUNT(12, clock64() - t0);
    }
#endif
  }
  unsigned m = __ballot_sync(kFull, need);
#ifdef PGPB_SEQ_PROFILE
  const int nwd = __popc(m);
#endif
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int wf = __shfl_sync(kFull, f, src);
    const int woff = __shfl_sync(kFull, off, src);
    const int wlast = __shfl_sync(kFull, last, src);
    const int wa = __shfl_sync(kFull, a, src);
    const float wlpa = __shfl_sync(kFull, lpa, src);
    const int wt2 = __shfl_sync(kFull, t2, src);
    const float wlp2 = __shfl_sync(kFull, lp2, src);
#ifdef PGPB_SEQ_PROFILE
    const long long t0 = clock64();
#endif
    const BCand wd = warp_decide(x, bm, x.rows + int64_t(wf) * x.V, woff, wlast, wa, wlpa, wt2, wlp2);
#ifdef PGPB_SEQ_PROFILE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      CF_COUNT(14, 1);
      CF_COUNT(15, clock64() - t0);
    }
#endif
    if (x.lane == src) d = wd;
  }
  if (emit) {
    s.o_tok[f] = d.v;
    s.o_lp[f] = d.lp;
    s.o_s[f] = d.s;
    s.o_nx[f] = d.nx;
    off = d.noff;
    st = d.nx;
    last = d.v;
  }
#ifdef PGPB_SEQ_PROFILE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int i = g_cf_step++;
    if (i < 112) {
      g_cf_prof[16 + i] = clock64() - t_step;
      g_cf_prof[128 + i] = __popc(em) + 100 * nwd;
    }
  }
#endif
}

// Sequential walk of a whole segment by one warp (every decision by the
// whole warp), used when boosting is expected to flip many decisions and
// speculation would only redo work.  The row of the next frame that may emit
// is prefetched into L1 while the current decision is made.
__device__ void seq_walk(const Ctx &x, unsigned *bm, int n, int &off, int &st, int &last) {
  const Smem &s = *x.s;
  const int lane = x.lane;
  for (int f = 0; f < n; ++f) {
    const int a = s.fa[f];
    const float lpa = s.flpa[f];
    if (a == x.blank || a == last) {
      if (lane == 0) {
        s.o_tok[f] = -1;
        s.o_lp[f] = lpa;
      }
      last = a;
      continue;
    }
    {
      const int g = f + 1 + lane;
      const unsigned m = __ballot_sync(kFull, g < n && s.fa[g] != x.blank);
      if (m) {
        const float *nrow = x.rows + int64_t(f + __ffs(m)) * x.V;
        for (int c = lane * 32; c < x.V; c += 32 * 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(nrow + c));
      }
    }
    const BCand d = warp_decide(x, bm, x.rows + int64_t(f) * x.V, off, last, a, lpa, s.ft2[f], s.flp2[f]);
    if (lane == 0) {
      s.o_tok[f] = d.v;
      s.o_lp[f] = d.lp;
      s.o_s[f] = d.s;
      s.o_nx[f] = d.nx;
    }
    off = d.noff;
    st = d.nx;
    last = d.v;
  }
  __syncwarp();
}

// Exact sum of f32 values and a fp64 carry in any order.  When every value
// (and the carry) is a multiple of 2^e and the sum of their magnitudes is
// below 2^(53+e), every partial sum in any order is representable in fp64,
// so a tree sum equals the reference's sequential sum bit for bit;
// exact_with() reports false (and no sum) otherwise.
struct GridSum {
  double part = 0.0, sabs = 0.0;
  int emin = INT_MAX;  // smallest ulp exponent seen
  __device__ __forceinline__ void add(float d) {
    if (d == 0.0f) return;
    const int be = (__float_as_int(d) >> 23) & 0xff;
    emin = min(emin, be ? be - 150 : -149);
    part = __dadd_rn(part, static_cast<double>(d));
    sabs = __dadd_rn(sabs, fabs(static_cast<double>(d)));
  }
  __device__ __forceinline__ void merge(double p, double a, int e) {
    part = __dadd_rn(part, p);
    sabs = __dadd_rn(sabs, a);
    emin = min(emin, e);
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      part = __dadd_rn(part, __shfl_xor_sync(kFull, part, o));
      sabs = __dadd_rn(sabs, __shfl_xor_sync(kFull, sabs, o));
    }
    emin = __reduce_min_sync(kFull, emin);
  }
  __device__ __forceinline__ bool exact_with(double carry, double &out) const {
    int e = emin;
    double a = sabs;
    if (carry != 0.0) {
      const int be = int((__double_as_longlong(carry) >> 52) & 0x7ff);
      e = min(e, be ? be - 1075 : -1074);
      a = __dadd_rn(a, fabs(carry));
    }
    if (!(e == INT_MAX || (e > -1000 && a * (1.0 + 1e-12) < ldexp(1.0, 53 + e)))) return false;
    out = __dadd_rn(carry, part);
    return true;
  }
};

// Named barrier + OR over the CTA (all warps walk).
__device__ __forceinline__ bool cta_or(bool pred) { return __syncthreads_or(pred) != 0; }

__global__ void __launch_bounds__(32 * (kMaxConsumers + 1), 1) ctc_walk_kernel(Args g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TableView &t = g.t;
  const int V = g.V, Vp = (V + 3) & ~3, Vw = (V + 31) >> 5;
  const int W = (blockDim.x >> 5) - 1, C = 32 * W, TS = g.TS;  // walker warps + 1 accountant warp
  const bool boost = g.use_boost != 0;
#ifdef PGPB_SEQ_PROFILE
  long long t_entry = clock64();
  int cf_rep = 0;
#endif
  Smem s;
  smem_bytes(Vp, Vw, W, TS, g.use_boost, &s, smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nthreads = blockDim.x;
  if (boost) {
    // root row -> shared memory, every load of a thread in flight at once
    for (int i0 = threadIdx.x; i0 < Vp; i0 += 4 * nthreads) {
      float r0[4];
      int r1[4], r2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nthreads;
        if (i < Vp) {
          r0[u] = __ldg(t.root_scores + i);
          r1[u] = __ldg(t.root_next + i);
          r2[u] = __ldg(t.root_next_off + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nthreads;
        if (i < Vp) {
          s.root[i] = r0[u];
          s.rnext[i] = r1[u];
          s.rnoff[i] = r2[u];
        }
      }
    }
    for (int i = threadIdx.x; i < W * Vw; i += nthreads) s.bm[i] = 0u;
  }
  const int root_off = boost ? __ldg(t.blob_off) : 0;
  // programmatic dependent launch: the prologue above overlaps phase A's tail
  CF_MARK(0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  CF_MARK(1);
  Ctx x;
  x.t = &t;
  x.s = &s;
  x.rows = nullptr;
  x.V = V;
  x.blank = g.blank;
  x.lam = g.lam;
  x.inv_lam = g.lam > 0.0 ? 1.0 / g.lam : 0.0;
  x.max_root = t.max_root_score;
  x.lane = lane;
  unsigned *bm = boost ? s.bm + wid * Vw : nullptr;
  const int c = threadIdx.x;  // chunk of this lane

  for (int64_t b = blockIdx.x; b < g.B; b += gridDim.x) {
#ifdef PGPB_SEQ_PROFILE
    if (b != blockIdx.x) {  // second utterance of this CTA: a timeline of its own (warm instruction caches)
      __syncthreads();
      t_entry = clock64() - 5000;
      cf_rep = 1;
    }
#endif
    // lengths are clamped to [0, T] so a bad length cannot address another
    // utterance's rows or outputs (the host layer rejects them first)
    const int64_t Tb = g.lengths ? min(max(int64_t(__ldg(g.lengths + b)), int64_t(0)), g.T) : g.T;
    __syncthreads();
    if (threadIdx.x == 0) {
      s.misc[0] = root_off;
      s.misc[1] = -1;
      s.misc[2] = 0;
      s.misc[3] = 0;
      s.dsum[0] = 0.0;
      s.dsum[1] = 0.0;
    }
#ifdef PGPB_SEQ_PROFILE
    const long long t_start = clock64();
#endif
    for (int64_t s0 = 0; s0 < Tb; s0 += TS) {
      if (threadIdx.x == 0) CF_COUNT(9, 1);
      const int n = int(Tb - s0 < TS ? Tb - s0 : TS);
      const int L = (n + C - 1) / C;
      const int Cn = (n + L - 1) / L;  // non-empty chunks
      const float *rows = g.lp + (b * g.T + s0) * int64_t(V);
      const int4 *top = g.top + b * g.T + s0;
      for (int f0 = threadIdx.x; f0 < n; f0 += 4 * nthreads) {
        int4 r[4];  // all loads in flight before the first store: one round trip
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (f0 + u * nthreads < n) {
            if (boost) {
              r[u] = __ldg(top + f0 + u * nthreads);
            } else {  // unboosted phase A writes only the {a, lp_a} half
              const int2 h = __ldg(reinterpret_cast<const int2 *>(top + f0 + u * nthreads));
              r[u] = make_int4(h.x, h.y, 0, 0);
            }
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int f = f0 + u * nthreads;
          if (f < n) {
            s.fa[f] = r[u].x;
            s.flpa[f] = __int_as_float(r[u].y);
            if (boost) {
              s.ft2[f] = r[u].z;
              s.flp2[f] = __int_as_float(r[u].w);
            }
          }
        }
      }
      __syncthreads();
      CF_MARK(2);
      // One pass of every walker lane over its chunk: the argmax emissions
      // (for the round-0 guesses) and the mode counts.
      //
      // Round-0 start guess of chunk c (exact when boosting does not flip a
      // decision near the boundary and the last emission starts no phrase
      // continuation): last = the previous frame's argmax, state = the AC
      // step from the depth-1 state of the second most recent argmax
      // emission v1 on the most recent one v2.  (v1, v2) before the chunk
      // come from a warp scan over the chunks and a lane-parallel look back
      // before the warp's first chunk.  The step's bitmap word (with its
      // rank: v2's entry index when v2 is on the closure) is loaded here and
      // consumed after the mode decision.
      int gv1 = -1, gv2 = -1;
      uint2 gw = make_uint2(0u, 0u);
      bool gfar = false, seq = false;
      if (boost) {
        int e1 = -1, e2 = -1, cand = 0, sens = 0;
        if (c < Cn) {
          for (int f = c * L, fe = min(f + L, n); f < fe; ++f) {
            const int a = s.fa[f], ap = f ? s.fa[f - 1] : s.misc[1];
            if (a != g.blank && a != ap) {
              e1 = e2;
              e2 = a;
              ++cand;
              sens += (s.flpa[f] - s.flp2[f]) < static_cast<float>(g.lam) * t.typ_gain;
            }
          }
        }
        // exclusive scan of "last two emissions" over this warp's chunks
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int p1 = __shfl_up_sync(kFull, e1, o), p2 = __shfl_up_sync(kFull, e2, o);
          if (lane >= o && e1 < 0) {
            e1 = e2 >= 0 ? p2 : p1;
            e2 = e2 >= 0 ? e2 : p2;
          }
        }
        gv1 = __shfl_up_sync(kFull, e1, 1);
        gv2 = __shfl_up_sync(kFull, e2, 1);
        if (lane == 0) gv1 = gv2 = -1;
        // emissions before the warp's first chunk: up to 64 frames back, 32 per ballot
        const int cbw = (c & ~31) * L;
        int w1 = -1, w2 = -1, fw0 = cbw;
        if (wid >= W || cbw >= n) fw0 = 0;  // helper warp / no live chunk: nothing to look back for
        for (; fw0 > 0 && fw0 > cbw - 64 && w1 < 0; fw0 -= 32) {
          const int fw = fw0 - 1 - lane;
          int at = -1;
          bool em = false;
          if (fw >= 0) {
            at = s.fa[fw];
            em = at != g.blank && at != (fw ? s.fa[fw - 1] : s.misc[1]);
          }
          unsigned m = __ballot_sync(kFull, em);
          while (m && w1 < 0) {
            const int v = __shfl_sync(kFull, at, __ffs(m) - 1);
            m &= m - 1;
            if (w2 < 0)
              w2 = v;
            else
              w1 = v;
          }
        }
        if (gv2 < 0) {
          gv1 = w1;
          gv2 = w2;
        } else if (gv1 < 0) {
          gv1 = w2;
        }
        gfar = gv2 < 0 && fw0 > 0;
        CF_MARK(12);
        if (c > 0 && c < Cn && gv1 >= 0 && t.clo_bits && s.rnext[gv1] != 0) {
          gw = tab_ld(t.clo_bits + int64_t(s.rnext[gv1]) * t.bits_words + (gv2 >> 5));
        }
        CF_MARK(13);
        // Boost-sensitive frames: may emit and the top-2 gap is within the
        // typical gain of a first-hit arc.  Mostly sensitive -> sequential.
        cand = __reduce_add_sync(kFull, cand);
        sens = __reduce_add_sync(kFull, sens);
        if (lane == 0) {
          s.wsum[wid] = cand;
          s.wsum[16 + wid] = sens;
        }
        __syncthreads();
        int tc = 0, ts = 0;
        for (int w = 0; w < W; ++w) {
          tc += s.wsum[w];
          ts += s.wsum[16 + w];
        }
        seq = g.seq_mode == 1 || (g.seq_mode == 0 && 4 * ts > tc && tc >= 8);
        CF_MARK(3);
      }
      if (boost && seq) {
        // ---- sequential mode: warp 0 walks the segment ----
        x.rows = rows;
        if (wid == 0) {
          int off = s.misc[0], st = s.misc[3], last = s.misc[1];
          seq_walk(x, bm, n, off, st, last);
          if (lane == 0) {
            s.c_eoff[Cn - 1] = off;
            s.c_est[Cn - 1] = st;
            s.c_elast[Cn - 1] = last;
          }
        }
      } else if (boost) {
        // ---- round 0: every chunk from a guessed start ----
        x.rows = rows;
        const bool live = c < Cn;
        const int cb = c * L, ce = min(cb + L, n);
        int off = s.misc[0], st = s.misc[3], last = s.misc[1];
        if (c > 0 && live) {
          last = s.fa[cb - 1];
          if (gv2 >= 0) {
            off = s.rnoff[gv2];
            st = s.rnext[gv2];
            CF_MARK(14);
            if ((gw.x >> (gv2 & 31)) & 1u) {
              CF_COUNT(22, 1);
              // v2 is on v1's state's closure: its entry by rank
              const int4 e = tab_ld(t.blob + s.rnoff[gv1] + 1 + int(gw.y) + __popc(gw.x & ((1u << (gv2 & 31)) - 1u)));
              off = e.w;
              st = e.y;
            }
          } else if (gfar) {
            off = root_off;
            st = 0;
          }
        }
        s.c_soff[c] = off;
        s.c_sst[c] = st;
        s.c_slast[c] = last;
        CF_MARK(4);
#ifdef PGPB_SEQ_PROFILE
        const long long t_r0 = clock64();
#endif
        // Emission-compacted: each lane runs through its blank / repeat
        // frames on its own (shared-memory records only) and the warp steps
        // together only at decisions, so round 0 costs one dependent round
        // trip per emission of the busiest lane instead of one per frame
        // (L frames per chunk, almost every frame emits in some lane).
        for (int f = cb;;) {
          if (live) f = pass_through(x, f, ce, off, last);
          const bool has = live && f < ce;
          if (!__any_sync(kFull, has)) break;
#ifdef PGPB_SEQ_PROFILE
          {
            const unsigned hm = __ballot_sync(kFull, has);
            if (lane == 0) CF_COUNT(1, __popc(hm));
          }
#endif
          walk_step(x, bm, has, f, off, st, last);
          if (has) ++f;
        }
        s.c_eoff[c] = off;
        s.c_est[c] = st;
        s.c_elast[c] = last;
        CF_MARK(5);
#ifdef PGPB_SEQ_PROFILE
        if (lane == 0 && wid < W) {
          const unsigned long long d = clock64() - t_r0;
          atomicMax(&g_cf_prof[194], d);
          atomicAdd(&g_cf_prof[195], d);
          atomicAdd(&g_cf_prof[196], 1ull);
        }
#endif
#ifdef PGPB_SEQ_PROFILE
        if (blockIdx.x == 0 && threadIdx.x == 0) CF_COUNT(6, clock64() - t_start);
#endif
        // ---- fix-up rounds ----
        for (;;) {
          __syncthreads();  // ends published
          int noff = 0, nst = 0, nlast = 0;
          bool changed = false;
          if (live) {
            noff = c == 0 ? s.misc[0] : s.c_eoff[c - 1];
            nst = c == 0 ? s.misc[3] : s.c_est[c - 1];
            nlast = c == 0 ? s.misc[1] : s.c_elast[c - 1];
            changed = noff != s.c_soff[c] || nlast != s.c_slast[c];
          }
          if (!cta_or(changed)) break;
          if (threadIdx.x == 0) CF_COUNT(0, 1);
          s.c_act[c] = changed;
          __syncthreads();  // activity flags visible to run-ahead walkers
          bool active = changed;
          int cc = c, f = cb, fe = ce;
          if (changed) {
            s.c_soff[c] = noff;
            s.c_sst[c] = nst;
            s.c_slast[c] = nlast;
            off = noff;
            st = nst;
            last = nlast;
          }
          while (__any_sync(kFull, active)) {
            bool has = false;
            if (active) {
              if (f >= fe) {
                s.c_eoff[cc] = off;
                s.c_est[cc] = st;
                s.c_elast[cc] = last;
                if (cc + 1 < Cn && !s.c_act[cc + 1]) {
                  // run ahead into the next chunk, idle in this round
                  ++cc;
                  s.c_soff[cc] = off;
                  s.c_sst[cc] = st;
                  s.c_slast[cc] = last;
                  fe = min(f + L, n);
                } else {
                  active = false;
                }
              }
              if (active) {
                if (f != cb && off == s.in_off[f] && last == s.in_last[f])
                  active = false;  // resynchronised: the rest is unchanged
                else
                  has = true;
              }
            }
#ifdef PGPB_SEQ_PROFILE
            {
              const unsigned hm = __ballot_sync(kFull, has);
              if (lane == 0) CF_COUNT(2, __popc(hm));
            }
#endif
            walk_step(x, bm, has, f, off, st, last);
            if (has) ++f;
          }
        }
#ifdef PGPB_SEQ_PROFILE
        if (blockIdx.x == 0 && threadIdx.x == 0) CF_COUNT(7, clock64() - t_start);
#endif
      } else {
        // ---- unboosted: emit iff a != blank and a != a[t-1] ----
        for (int f = threadIdx.x; f < n; f += nthreads) {
          const int a = s.fa[f];
          const int prev = f ? s.fa[f - 1] : s.misc[1];
          s.o_tok[f] = (a != g.blank && a != prev) ? a : -1;
          s.o_lp[f] = s.flpa[f];
        }
      }
      __syncthreads();
      CF_MARK(6);
      // ---- tail: one pass over each thread's contiguous frames (emit
      // count, exact-sum partials of am and boost),
      // warp scans / reductions, one barrier, then compaction ----
      const int q = (n + nthreads - 1) / nthreads;
      const int f0 = min(int(threadIdx.x) * q, n), f1 = min(f0 + q, n);
      const int base = s.misc[2];
      int cntm = 0;
      GridSum ga, gb;
      for (int f = f0; f < f1; ++f) {
        const int tk = s.o_tok[f];
        const float lpv = s.o_lp[f];
        cntm += tk >= 0;
        ga.add(lpv);
        if (boost && tk >= 0) gb.add(s.o_s[f]);
      }
      int incl = cntm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      ga.warp_reduce();
      if (boost) gb.warp_reduce();
      if (lane == 31) s.wsum[wid] = incl;
      if (lane == 0) {
        s.wred[4 * wid] = ga.part;
        s.wred[4 * wid + 1] = ga.sabs;
        s.wred[4 * wid + 2] = gb.part;
        s.wred[4 * wid + 3] = gb.sabs;
        s.wmin[4 * wid] = ga.emin;
        s.wmin[4 * wid + 1] = gb.emin;
      }
      __syncthreads();
      CF_MARK(7);
      int pos = base + incl - cntm;
      for (int w = 0; w < wid; ++w) pos += s.wsum[w];
      int32_t *otok = g.tokens + b * g.T;
      double *odl = g.deltas + b * g.T;
      int32_t *ost = g.ostates + b * g.T;
      for (int f = f0; f < f1; ++f) {
        const int tk = s.o_tok[f];
        if (tk >= 0) {
          otok[pos] = tk;
          odl[pos] = boost ? static_cast<double>(s.o_s[f]) : 0.0;
          ost[pos] = boost ? s.o_nx[f] : 0;
          ++pos;
        }
      }
      if (threadIdx.x == 0) {
        // am / boost over every frame in order: the exact grid sum when it is
        // exact (the usual case), else the reference's sequential order
        GridSum ta, tb;
        int tot = 0;
        for (int w = 0; w <= W; ++w) {
          ta.merge(s.wred[4 * w], s.wred[4 * w + 1], s.wmin[4 * w]);
          tb.merge(s.wred[4 * w + 2], s.wred[4 * w + 3], s.wmin[4 * w + 1]);
          tot += s.wsum[w];
        }
        double am;
        if (!ta.exact_with(s.dsum[0], am)) {
          double acc = s.dsum[0];
          for (int u = 0; u < n; ++u) acc = __dadd_rn(acc, static_cast<double>(s.o_lp[u]));
          am = acc;
        }
        s.dsum[0] = am;
        if (boost) {
          double bo;
          if (!tb.exact_with(s.dsum[1], bo)) {
            double acc = s.dsum[1];
            for (int u = 0; u < n; ++u)
              if (s.o_tok[u] >= 0) acc = __dadd_rn(acc, static_cast<double>(s.o_s[u]));
            bo = acc;
          }
          s.dsum[1] = bo;
        }
        s.misc[2] = base + tot;
        if (boost) {
          s.misc[0] = s.c_eoff[Cn - 1];
          s.misc[1] = s.c_elast[Cn - 1];
          s.misc[3] = s.c_est[Cn - 1];
        } else {
          s.misc[1] = s.fa[n - 1];
        }
      }
      __syncthreads();
    }
    __syncthreads();
#ifdef PGPB_SEQ_PROFILE
    if (blockIdx.x == 0 && threadIdx.x == 0) CF_COUNT(8, clock64() - t_start);
#endif
    CF_MARK(8);
    if (threadIdx.x == 0) {
      g.nout[b] = s.misc[2];
      g.am_out[b] = s.dsum[0];
      g.boost_out[b] = s.dsum[1];
    }
  }
}

}  // namespace cw

int ctc_spec_launch(const pgpb_table *table, const float *d_lp, int64_t B, int64_t T, int32_t V,
                    const int32_t *d_lengths, int32_t blank, double lam, int32_t use_boost, int32_t *d_tokens,
                    double *d_deltas, int32_t *d_states, int32_t *d_num_out, double *d_am, double *d_boost,
                    cudaStream_t st) {
  using namespace cw;
  retain_pool(current_device());
  const bool vec = (V % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  const int64_t F = B * T;
  int4 *top = nullptr;
  if (F > 0) PGPB_CUDA_TRY(cudaMallocAsync(&top, size_t(F) * 16, st));
  if (F > 0) {
    // one wave: 2 resident CTAs per SM (<= 128 registers), grid-stride over
    // frame pairs (0.5 us faster than 8 waves of CTAs on 128 x 200 frames)
    const unsigned grid = warp_grid((F + 1) / 2, 2);
    using KA = void (*)(const float *, int64_t, int64_t, int, const int32_t *, int, int4 *);
    KA ka = use_boost ? (vec ? frame_top2_kernel<true, true> : frame_top2_kernel<true, false>)
                      : (vec ? frame_top2_kernel<false, true> : frame_top2_kernel<false, false>);
    ka<<<grid, 256, 0, st>>>(d_lp, B, T, V, d_lengths, blank, top);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFreeAsync(top, st);
      return fail(PGPB_ECUDA, std::string("frame_top2_kernel: ") + cudaGetErrorString(e));
    }
  }
  Args a{};
  a.t = table ? table->view : empty_view(V);
  a.lp = d_lp;
  a.top = top;
  a.B = B;
  a.T = T;
  a.V = V;
  a.lengths = d_lengths;
  a.blank = blank;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.tokens = d_tokens;
  a.deltas = d_deltas;
  a.ostates = d_states;
  a.nout = d_num_out;
  a.am_out = d_am;
  a.boost_out = d_boost;
  const int Vp = (V + 3) & ~3, Vw = (V + 31) >> 5;
  int W = use_boost ? 1 : kMaxConsumers;
  if (use_boost) {  // one frame per chunk in round 0 up to 224 frames per segment
    const int64_t want = (T + 31) / 32;
    W = int(want < 1 ? 1 : (want > kMaxConsumers ? kMaxConsumers : want));
  }
  const Tuning &tun = tuning();
  if (tun.ctc_consumers) W = std::max(1, std::min(kMaxConsumers, tun.ctc_consumers));
  int TS = int(T < 1 ? 1 : (T > 8192 ? 8192 : T));
  if (tun.ctc_segment) TS = std::max(1, std::min(TS, tun.ctc_segment));
  while (TS > 64 && smem_bytes(Vp, Vw, W, TS, a.use_boost, nullptr, nullptr) > size_t(kSmemBudget)) TS -= 32;
  const size_t smem = smem_bytes(Vp, Vw, W, TS, a.use_boost, nullptr, nullptr);
  if (smem > 227 * 1024) {
    if (top) cudaFreeAsync(top, st);
    return fail(PGPB_EINVAL, "vocabulary too large for the CTC walker's shared-memory root row");
  }
  a.TS = TS;
  a.seq_mode = std::max(0, std::min(2, tun.ctc_seq));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(ctc_walk_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) {
      if (top) cudaFreeAsync(top, st);
      return fail(PGPB_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctc_walk_kernel, 32 * (W + 1), smem);
  const int64_t cap = int64_t(sm_count(current_device())) * std::max(per_sm, 1);
  unsigned grid = unsigned(B < cap ? B : cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * (W + 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, ctc_walk_kernel, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (top) cudaFreeAsync(top, st);
  if (e != cudaSuccess) return fail(PGPB_ECUDA, std::string("ctc_walk_kernel: ") + cudaGetErrorString(e));
  return PGPB_OK;
}

}  // namespace pgpb

#ifdef PGPB_SEQ_PROFILE
extern "C" int pgpb_debug_ctc_lane_records(long long *h_out, int reset) {
  cudaMemcpyFromSymbol(h_out, pgpb::cw::g_ld_rec, sizeof(long long) * 256 * 4);
  if (reset) {
    int z = 0;
    cudaMemcpyToSymbol(pgpb::cw::g_ld_n, &z, sizeof(int));
  }
  return 0;
}

extern "C" int pgpb_debug_ctc_fused_profile(unsigned long long *h_out, int reset) {
  cudaMemcpyFromSymbol(h_out, pgpb::cw::g_cf_prof, sizeof(unsigned long long) * 256);
  if (reset) {
    unsigned long long z[256] = {0};
    cudaMemcpyToSymbol(pgpb::cw::g_cf_prof, z, sizeof(z));
    int zero = 0;
    cudaMemcpyToSymbol(pgpb::cw::g_cf_step, &zero, sizeof(int));
  }
  return 0;
}
#endif
