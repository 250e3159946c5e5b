// Warp-level rerank helpers shared by the greedy / step / CTC kernels.
#pragma once

#include "pgpb_common.cuh"

namespace pgpb {


struct RerankOut {
  int chosen;
  float lp;
  double delta;
  int next;
};

// Marks the state's closure tokens in the warp's shared bitmap.
__device__ __forceinline__ void mark_closure(const TableView &t, const int4 rec, unsigned *bm, int lane,
                                             bool set) {
  for (int i = lane; i < rec.y; i += 32) {
    const int tok = __ldg(&t.clo[rec.x + i].x);
    if (set)
      atomicOr(bm + (tok >> 5), 1u << (tok & 31));
    else
      bm[tok >> 5] = 0u;
  }
}

// Boosted rerank of one row by one warp: argmax over v not in {ex1, ex2}
// of lp[v] + lam * score[state, v], ties -> higher lp -> lower v.
template <bool kVec>
__device__ RerankOut warp_rerank(const TableView &t, const float *root, const int32_t *rnext,
                                 unsigned *bm, const float *__restrict__ row, int V, int state,
                                 int ex1, int ex2, double lam, int lane) {
  const int4 rec = __ldg(t.clo_rec + state);
  const float acc = __int_as_float(rec.z);
  mark_closure(t, rec, bm, lane, true);
  __syncwarp();
  double bc = -INFINITY;
  float blp = -INFINITY, bsv = 0.0f;
  int bv = INT_MAX, bnx = 0;
  auto consider = [&](int v, float x, float sv, int nx) {
    const double c = fuse(x, lam, sv);
    if (rerank_better(c, x, v, bc, blp, bv)) {
      bc = c;
      blp = x;
      bv = v;
      bsv = sv;
      bnx = nx;
    }
  };
  // Dense candidates: tokens without an explicit arc on the chain.
  if (kVec) {
    const float4 *row4 = reinterpret_cast<const float4 *>(row);
    for (int i = lane; i < (V >> 2); i += 32) {
      const float4 x4 = __ldcg(row4 + i);
      const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v = 4 * i + j;
        if (v == ex1 || v == ex2) continue;
        if ((bm[v >> 5] >> (v & 31)) & 1u) continue;
        consider(v, xs[j], acc + root[v], rnext[v]);
      }
    }
  } else {
    for (int v = lane; v < V; v += 32) {
      if (v == ex1 || v == ex2) continue;
      if ((bm[v >> 5] >> (v & 31)) & 1u) continue;
      consider(v, __ldcg(row + v), acc + root[v], rnext[v]);
    }
  }
  // Explicit first-hit arcs of the chain.
  for (int i = lane; i < rec.y; i += 32) {
    const int4 e = __ldg(t.clo + rec.x + i);
    if (e.x == ex1 || e.x == ex2) continue;
    consider(e.x, __ldcg(row + e.x), __int_as_float(e.z), e.y);
  }
  // Warp reduction on (c, lp, v); the winning lane then broadcasts (s, next).
  double rc = bc;
  float rlp = blp;
  int rv = bv;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(kFull, rc, o);
    const float olp = __shfl_xor_sync(kFull, rlp, o);
    const int ov = __shfl_xor_sync(kFull, rv, o);
    if (rerank_better(oc, olp, ov, rc, rlp, rv)) {
      rc = oc;
      rlp = olp;
      rv = ov;
    }
  }
  const unsigned owner = __ballot_sync(kFull, bv == rv);
  const int src = owner ? __ffs(owner) - 1 : 0;
  RerankOut out;
  out.chosen = rv;
  out.lp = rlp;
  out.delta = static_cast<double>(__shfl_sync(kFull, bsv, src));
  out.next = __shfl_sync(kFull, bnx, src);
  __syncwarp();
  mark_closure(t, rec, bm, lane, false);
  __syncwarp();
  return out;
}

// First argmax of a row (value, lowest index among equals).
template <bool kVec>
__device__ __forceinline__ void warp_row_argmax(const float *__restrict__ row, int V, int lane,
                                                float &best, int &idx) {
  best = -INFINITY;
  idx = INT_MAX;
  if (kVec) {
    const float4 *row4 = reinterpret_cast<const float4 *>(row);
#pragma unroll 4
    for (int i = lane; i < (V >> 2); i += 32) {
      const float4 x = __ldcg(row4 + i);
      const int v = 4 * i;
      if (argmax_better(x.x, v, best, idx)) { best = x.x; idx = v; }
      if (argmax_better(x.y, v + 1, best, idx)) { best = x.y; idx = v + 1; }
      if (argmax_better(x.z, v + 2, best, idx)) { best = x.z; idx = v + 2; }
      if (argmax_better(x.w, v + 3, best, idx)) { best = x.w; idx = v + 3; }
    }
  } else {
    for (int v = lane; v < V; v += 32) {
      const float x = __ldcg(row + v);
      if (argmax_better(x, v, best, idx)) { best = x; idx = v; }
    }
  }
  warp_argmax(best, idx);
}

__device__ __forceinline__ void setup_smem(const TableView &t, bool use_boost, bool smem_root,
                                           unsigned char *smem, const float *&root,
                                           const int32_t *&rnext, unsigned *&bm) {
  const int bm_words = (t.vocab_size + 31) >> 5;
  size_t off = 0;
  root = t.root_scores;
  rnext = t.root_next;
  if (use_boost && smem_root) {
    float *s_root = reinterpret_cast<float *>(smem);
    int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(t.vocab_padded) * 4);
    stage_root(t, s_root, s_next);
    root = s_root;
    rnext = s_next;
    off = size_t(t.vocab_padded) * 8;
  }
  unsigned *all_bm = reinterpret_cast<unsigned *>(smem + off);
  if (use_boost)
    for (int i = threadIdx.x; i < bm_words * kWarpsPerBlock; i += blockDim.x) all_bm[i] = 0u;
  bm = all_bm + (threadIdx.x >> 5) * bm_words;
  __syncthreads();
}

static inline size_t greedy_smem(const TableView &t, bool use_boost, bool &smem_root) {
  const size_t bm = size_t((t.vocab_size + 31) >> 5) * 4 * kWarpsPerBlock;
  const size_t root = size_t(t.vocab_padded) * 8;
  smem_root = use_boost && root + bm <= size_t(kMaxSmemRootBytes);
  return (use_boost ? bm : 0) + (smem_root ? root : 0);
}

template <typename F>
static inline int prep_kernel(F fn, size_t smem) {
  if (smem > 48 * 1024) {
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  return PGPB_OK;
}

// Placeholder view for unboosted calls without a table.
static inline TableView empty_view(int V) {
  TableView v{};
  v.num_states = 1;
  v.vocab_size = V;
  v.vocab_padded = (V + 3) & ~3;
  return v;
}

}  // namespace pgpb

namespace pgpb {

// ---------------------------------------------------------------------------
// Blob-based boosted rerank (fast path shared by the CTC sequential kernel
// and the transducer step kernel).

struct BCand {
  double c;
  float lp;
  int v;
  float s;
  int nx;
  int noff;
};

__device__ __forceinline__ BCand bcand_none() { return BCand{-INFINITY, -INFINITY, INT_MAX, 0.0f, 0, 0}; }

__device__ __forceinline__ void bcand_consider(BCand &b, double c, float x, int v, float s, int nx, int noff) {
  if (rerank_better(c, x, v, b.c, b.lp, b.v)) b = BCand{c, x, v, s, nx, noff};
}

// Order-preserving unsigned keys for IEEE values (NaN excluded).  -0.0 is
// folded onto +0.0 (x + 0 under round-to-nearest) so the keys order
// exactly as the reference's float compares, which call them equal.
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(x, 0.0)));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned fkey(float x) {
  const unsigned u = __float_as_uint(__fadd_rn(x, 0.0f));
  return (u >> 31) ? ~u : (u | 0x80000000u);
}

// Warp argmax on (c desc, lp desc, v asc) with redux.sync on the 64-bit
// order-preserving key of c (two 32-bit halves), then lp and v only when c
// ties; the winner's payload is shuffled from its lane.  Lanes without a
// candidate carry v == INT_MAX.
__device__ __forceinline__ BCand bcand_warp_best(const BCand &mine) {
  const bool has = mine.v != INT_MAX;
  const unsigned long long k = has ? dkey(mine.c) : 0ull;
  const unsigned hi = static_cast<unsigned>(k >> 32), lo = static_cast<unsigned>(k);
  const unsigned mhi = __reduce_max_sync(kFull, hi);
  const unsigned mlo = __reduce_max_sync(kFull, hi == mhi ? lo : 0u);
  unsigned tie = __ballot_sync(kFull, has && hi == mhi && lo == mlo);
  if (__popc(tie) > 1) {
    const bool in = (tie >> (threadIdx.x & 31)) & 1u;
    const unsigned lk = in ? fkey(mine.lp) : 0u;
    const unsigned mlk = __reduce_max_sync(kFull, lk);
    tie = __ballot_sync(kFull, in && lk == mlk);
    if (__popc(tie) > 1) {
      const bool in2 = (tie >> (threadIdx.x & 31)) & 1u;
      const unsigned mv = __reduce_min_sync(kFull, in2 ? static_cast<unsigned>(mine.v) : 0xffffffffu);
      tie = __ballot_sync(kFull, in2 && static_cast<unsigned>(mine.v) == mv);
    }
  }
  const int src = tie ? __ffs(tie) - 1 : 0;
  BCand w;
  w.c = __shfl_sync(kFull, mine.c, src);
  w.lp = __shfl_sync(kFull, mine.lp, src);
  w.v = __shfl_sync(kFull, mine.v, src);
  w.s = __shfl_sync(kFull, mine.s, src);
  w.nx = __shfl_sync(kFull, mine.nx, src);
  w.noff = __shfl_sync(kFull, mine.noff, src);
  return w;
}

__device__ __forceinline__ void prefetch_blob_l1(const int4 *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 8));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 16));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 24));
}

// A state's blob held in registers: lane 0 = header, lanes 1..31 the first
// 31 arcs (b0), lanes 0..31 arcs 31..62 (b1).  Both loads are issued
// together (the blob array is padded), so one L2/L1 round trip.
struct BlobRegs {
  int4 b0, b1;
  int off;
};

__device__ __forceinline__ BlobRegs load_blob(const TableView &t, int soff, int lane) {
  BlobRegs r;
  r.b0 = __ldg(t.blob + soff + lane);
  r.b1 = __ldg(t.blob + soff + 32 + lane);
  r.off = soff;
  return r;
}

// Blob offset of the successor on token v (the state's arc if v is on its
// closure, else the root row's).
__device__ __forceinline__ int blob_next_off(const BlobRegs &r, int count, const int32_t *rnoff, int v, int lane) {
  const bool v0 = lane >= 1 && lane <= count && r.b0.x == v;
  const bool v1 = count > 31 && lane + 32 <= count && r.b1.x == v;
  const unsigned m0 = __ballot_sync(kFull, v0), m1 = __ballot_sync(kFull, v1);
  if (m0) return __shfl_sync(kFull, r.b0.w, __ffs(m0) - 1);
  if (m1) return __shfl_sync(kFull, r.b1.w, __ffs(m1) - 1);
  return rnoff[v];
}

// Rerank at the state whose blob is in `cur`.  Candidates: the state's
// closure arcs (exact scores) and the M dense tokens tv[]/tx[] (the row's
// top-M by logprob, identical in every lane); tokens ex1/ex2 are excluded.
// The winner is exact when it beats the bound on dense tokens outside the
// top-M (see pgpb_ctc.cu header); otherwise the full row is rescanned using
// the shared bitmap `bm` (cleared again before return).  `root`, `rnext`,
// `rnoff` may be shared or global copies of the root row.
template <int M>
__device__ BCand blob_rerank_regs(const TableView &t, const BlobRegs &cur, const float *root, const int32_t *rnext,
                                  const int32_t *rnoff, unsigned *bm, const float *row, int V, const int (&tv)[M],
                                  const float (&tx)[M], int ex1, int ex2, double lam, float max_root, int lane) {
  const int4 b0 = cur.b0, b1 = cur.b1;
  const int count = __shfl_sync(kFull, b0.x, 0);
  const float acc = __int_as_float(__shfl_sync(kFull, b0.y, 0));
  const int soff = cur.off;
  const bool v0 = lane >= 1 && lane <= count;
  const bool v1 = count > 31 && lane + 32 <= count;
  BCand mine = bcand_none();
  const bool regs_ok = count <= 63;
  // every load the fast path may need, issued together (one round trip):
  // the closure arcs' log-probs and the argmax's root-row entries
  const int av0 = tv[0];
  const bool av_ok = av0 < V;
  const float x0 = v0 ? row[b0.x] : 0.0f;
  const float x1 = v1 ? row[b1.x] : 0.0f;
  const float root_av = av_ok ? root[av0] : 0.0f;
  const int rnext_av = av_ok ? rnext[av0] : 0;
  const int rnoff_av = av_ok ? rnoff[av0] : 0;
  // Fast path.  If the stage-1 argmax a = tv[0] is a dense token (not on
  // the closure) whose root weight is the row maximum, every dense token v
  // has lp_v <= lp_a and s_v <= s_a, so (all rounded ops being monotone,
  // ties going to the higher lp, then the lower id = a as the first max) a
  // beats every dense token: only closure arcs can win.  One ballot decides.
  if (regs_ok && tv[0] < V) {
    const int av = tv[0];
    const bool in_a = __ballot_sync(kFull, (v0 && b0.x == av) || (v1 && b1.x == av)) != 0u;
    if (!in_a && root_av == max_root && av != ex1 && av != ex2) {
      const float sa = acc + root_av;
      const double ca = fuse(tx[0], lam, sa);
      // fp32 pre-filter: an arc whose fp32 fused score is below a's by more
      // than the fp32 rounding error of either sum cannot win; only the
      // near ties take the exact fp64 comparison.
      const float lamf = static_cast<float>(lam);
      const float ca32 = __fadd_rn(tx[0], __fmul_rn(lamf, sa));
      const float tol = 1e-4f * (fabsf(tx[0]) + fabsf(lamf * sa) + 1.0f);
      if (v0 && b0.x != ex1 && b0.x != ex2) {
        const float x = x0;
        const float sv = __int_as_float(b0.z);
        const float c32 = __fadd_rn(x, __fmul_rn(lamf, sv));
        if (c32 >= ca32 - (tol + 1e-4f * (fabsf(x) + fabsf(lamf * sv)))) {
          const double c = fuse(x, lam, sv);
          if (rerank_better(c, x, b0.x, ca, tx[0], av)) mine = BCand{c, x, b0.x, sv, b0.y, b0.w};
        }
      }
      if (v1 && b1.x != ex1 && b1.x != ex2) {
        const float x = x1;
        const float sv = __int_as_float(b1.z);
        const float c32 = __fadd_rn(x, __fmul_rn(lamf, sv));
        if (c32 >= ca32 - (tol + 1e-4f * (fabsf(x) + fabsf(lamf * sv)))) {
          const double c = fuse(x, lam, sv);
          if (rerank_better(c, x, b1.x, ca, tx[0], av)) bcand_consider(mine, c, x, b1.x, sv, b1.y, b1.w);
        }
      }
      if (__ballot_sync(kFull, mine.v != INT_MAX) == 0u) return BCand{ca, tx[0], av, sa, rnext_av, rnoff_av};
      return bcand_warp_best(mine);
    }
  }
  if (regs_ok) {
    if (v0 && b0.x != ex1 && b0.x != ex2) {
      const float x = x0;
      bcand_consider(mine, fuse(x, lam, __int_as_float(b0.z)), x, b0.x, __int_as_float(b0.z), b0.y, b0.w);
    }
    if (v1 && b1.x != ex1 && b1.x != ex2) {
      const float x = x1;
      bcand_consider(mine, fuse(x, lam, __int_as_float(b1.z)), x, b1.x, __int_as_float(b1.z), b1.y, b1.w);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int v = tv[j];
      const bool in_clo = __ballot_sync(kFull, (v0 && b0.x == v) || (v1 && b1.x == v)) != 0u;
      if (lane == j && v < V && v != ex1 && v != ex2 && !in_clo) {
        const float s = acc + root[v];
        bcand_consider(mine, fuse(tx[j], lam, s), tx[j], v, s, rnext[v], rnoff[v]);
      }
    }
  }
  BCand w = bcand_warp_best(mine);
  bool exact = regs_ok && (V <= M || w.c > fuse(tx[M - 1], lam, acc + max_root));
  if (!exact) {
    // full rescan: mark every closure token, scan the dense row, then the arcs
    for (int k = lane; k < count; k += 32) {
      const int tok = __ldg(&t.blob[soff + 1 + k].x);
      atomicOr(bm + (tok >> 5), 1u << (tok & 31));
    }
    __syncwarp();
    // Dense tokens: a token can only beat (or tie) the current winner w when
    // fuse(x, lam, acc + max_root) >= w.c, i.e. x >= w.c - lam*(acc +
    // max_root) up to rounding; an fp32 threshold below that (with a margin
    // far above the rounding of either sum) skips the exact fp64 scoring of
    // every other token.  w stays a candidate, so the result is unchanged.
    BCand full = w;
    float thr = -INFINITY;
    if (w.v != INT_MAX && isfinite(w.c) && lam >= 0.0) {
      const double sm = lam * static_cast<double>(acc + max_root);
      const double tb = w.c - sm;
      thr = static_cast<float>(tb - (1e-5 * (fabs(w.c) + fabs(sm)) + 1e-5));
    }
    for (int v = lane; v < V; v += 32) {
      if (v == ex1 || v == ex2 || ((bm[v >> 5] >> (v & 31)) & 1u)) continue;
      const float x = row[v];
      if (x < thr) continue;
      const float s = acc + root[v];
      bcand_consider(full, fuse(x, lam, s), x, v, s, rnext[v], rnoff[v]);
    }
    for (int k = lane; k < count; k += 32) {
      const int4 e = __ldg(t.blob + soff + 1 + k);
      if (e.x == ex1 || e.x == ex2) continue;
      const float x = row[e.x];
      bcand_consider(full, fuse(x, lam, __int_as_float(e.z)), x, e.x, __int_as_float(e.z), e.y, e.w);
    }
    w = bcand_warp_best(full);
    __syncwarp();
    for (int k = lane; k < count; k += 32) bm[__ldg(&t.blob[soff + 1 + k].x) >> 5] = 0u;
    __syncwarp();
  }
  return w;
}

template <int M>
__device__ __forceinline__ BCand blob_rerank(const TableView &t, const float *root, const int32_t *rnext,
                                             const int32_t *rnoff, unsigned *bm, const float *row, int V, int soff,
                                             const int (&tv)[M], const float (&tx)[M], int ex1, int ex2, double lam,
                                             float max_root, int lane) {
  const BlobRegs cur = load_blob(t, soff, lane);
  return blob_rerank_regs<M>(t, cur, root, rnext, rnoff, bm, row, V, tv, tx, ex1, ex2, lam, max_root, lane);
}

// Per-lane top-M insertion by (value desc, index asc).
template <int M>
__device__ __forceinline__ void topm_insert(float (&lv)[M], int (&li)[M], float x, int v) {
  if (!argmax_better(x, v, lv[M - 1], li[M - 1])) return;
  lv[M - 1] = x;
  li[M - 1] = v;
#pragma unroll
  for (int i = M - 1; i > 0; --i) {
    if (argmax_better(lv[i], li[i], lv[i - 1], li[i - 1])) {
      const float tx = lv[i];
      lv[i] = lv[i - 1];
      lv[i - 1] = tx;
      const int ti = li[i];
      li[i] = li[i - 1];
      li[i - 1] = ti;
    }
  }
}

// Warp top-M of a row: every lane ends with the same sorted (tv, tx).
template <int M, bool kVec>
__device__ __forceinline__ void warp_row_topm(const float *__restrict__ row, int V, int lane, int (&tv)[M],
                                              float (&tx)[M]) {
  float lv[M];
  int li[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    lv[i] = -INFINITY;
    li[i] = INT_MAX;
  }
  if (kVec) {
    const float4 *row4 = reinterpret_cast<const float4 *>(row);
#pragma unroll 4
    for (int c = lane; c < (V >> 2); c += 32) {
      const float4 x = __ldcg(row4 + c);
      topm_insert<M>(lv, li, x.x, 4 * c);
      topm_insert<M>(lv, li, x.y, 4 * c + 1);
      topm_insert<M>(lv, li, x.z, 4 * c + 2);
      topm_insert<M>(lv, li, x.w, 4 * c + 3);
    }
  } else {
    for (int v = lane; v < V; v += 32) topm_insert<M>(lv, li, __ldcg(row + v), v);
  }
#pragma unroll
  for (int r = 0; r < M; ++r) {
    float bx = lv[0];
    int bi = li[0];
    warp_argmax(bx, bi);
    if (li[0] == bi && bi != INT_MAX) {
#pragma unroll
      for (int i = 0; i < M - 1; ++i) {
        lv[i] = lv[i + 1];
        li[i] = li[i + 1];
      }
      lv[M - 1] = -INFINITY;
      li[M - 1] = INT_MAX;
    }
    tv[r] = bi;
    tx[r] = bx;
  }
}

}  // namespace pgpb

namespace pgpb {

// Top-M of a row held in registers (NC float4 chunks per lane, V <= 128*NC),
// every lane ends with the same sorted (tv, tx).  Threshold method: the M-th
// largest lane maximum bounds the row's M-th largest value from below, so
// only elements >= it (normally exactly M) are ranked; ties producing more
// than 32 survivors fall back to the insertion network.  `sv`/`si` are 32
// shared slots private to the warp.
template <int M, int NC>
__device__ __forceinline__ void warp_regs_topm_thr(const float4 (&x)[NC], int V, int lane, float *sv, int *si,
                                                   int (&tv)[M], float (&tx)[M]);

template <int M, int NC>
__device__ __forceinline__ void warp_row_topm_thr(const float *__restrict__ row, int V, int lane, float *sv, int *si,
                                                  int (&tv)[M], float (&tx)[M]) {
  const float4 *row4 = reinterpret_cast<const float4 *>(row);
  const int V4 = V >> 2;
  float4 x[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = lane + 32 * k;
    x[k] = c < V4 ? __ldcg(row4 + c) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  }
  warp_regs_topm_thr<M, NC>(x, V, lane, sv, si, tv, tx);
}

// The same over a row already in registers: x[k] holds elements
// 4 * (lane + 32 k) .. + 3 (-inf past the row's end).
template <int M, int NC>
__device__ __forceinline__ void warp_regs_topm_thr(const float4 (&x)[NC], int V, int lane, float *sv, int *si,
                                                   int (&tv)[M], float (&tx)[M]) {
  float lm = -INFINITY;
  int li = INT_MAX;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int v = 4 * (lane + 32 * k);
    if (argmax_better(x[k].x, v, lm, li)) { lm = x[k].x; li = v; }
    if (argmax_better(x[k].y, v + 1, lm, li)) { lm = x[k].y; li = v + 1; }
    if (argmax_better(x[k].z, v + 2, lm, li)) { lm = x[k].z; li = v + 2; }
    if (argmax_better(x[k].w, v + 3, lm, li)) { lm = x[k].w; li = v + 3; }
  }
  float thr = -INFINITY;
  {
    float v = lm;
    int id = li;
#pragma unroll
    for (int r = 0; r < M; ++r) {
      float bx = v;
      int bi = id;
      warp_argmax(bx, bi);
      thr = bx;
      if (r == 0) {
        tv[0] = bi;
        tx[0] = bx;
      }
      if (id == bi) {
        v = -INFINITY;
        id = INT_MAX;
      }
    }
  }
  if (M == 1) return;
  int mine = 0;
#pragma unroll
  for (int k = 0; k < NC; ++k) mine += (x[k].x >= thr) + (x[k].y >= thr) + (x[k].z >= thr) + (x[k].w >= thr);
  int pos = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, pos, o);
    if (lane >= o) pos += y;
  }
  const int total = __shfl_sync(kFull, pos, 31);
  pos -= mine;
  if (total <= 32) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int v = 4 * (lane + 32 * k);
      if (x[k].x >= thr) { sv[pos] = x[k].x; si[pos++] = v; }
      if (x[k].y >= thr) { sv[pos] = x[k].y; si[pos++] = v + 1; }
      if (x[k].z >= thr) { sv[pos] = x[k].z; si[pos++] = v + 2; }
      if (x[k].w >= thr) { sv[pos] = x[k].w; si[pos++] = v + 3; }
    }
    __syncwarp();
    float cv = lane < total ? sv[lane] : -INFINITY;
    int ci = lane < total ? si[lane] : INT_MAX;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < M; ++r) {
      float bx = cv;
      int bi = ci;
      warp_argmax(bx, bi);
      if (ci == bi) {
        cv = -INFINITY;
        ci = INT_MAX;
      }
      tv[r] = bi;
      tx[r] = bx;
    }
  } else {
    float lv[M];
    int lix[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      lv[i] = -INFINITY;
      lix[i] = INT_MAX;
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int v = 4 * (lane + 32 * k);
      if (v < V) {
        topm_insert<M>(lv, lix, x[k].x, v);
        topm_insert<M>(lv, lix, x[k].y, v + 1);
        topm_insert<M>(lv, lix, x[k].z, v + 2);
        topm_insert<M>(lv, lix, x[k].w, v + 3);
      }
    }
#pragma unroll
    for (int r = 0; r < M; ++r) {
      float bx = lv[0];
      int bi = lix[0];
      warp_argmax(bx, bi);
      if (lix[0] == bi && bi != INT_MAX) {
#pragma unroll
        for (int i = 0; i < M - 1; ++i) {
          lv[i] = lv[i + 1];
          lix[i] = lix[i + 1];
        }
        lv[M - 1] = -INFINITY;
        lix[M - 1] = INT_MAX;
      }
      tv[r] = bi;
      tx[r] = bx;
    }
  }
}

}  // namespace pgpb
