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
      const float4 x4 = __ldg(row4 + i);
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
      consider(v, __ldg(row + v), acc + root[v], rnext[v]);
    }
  }
  // Explicit first-hit arcs of the chain.
  for (int i = lane; i < rec.y; i += 32) {
    const int4 e = __ldg(t.clo + rec.x + i);
    if (e.x == ex1 || e.x == ex2) continue;
    consider(e.x, __ldg(row + e.x), __int_as_float(e.z), e.y);
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
      const float4 x = __ldg(row4 + i);
      const int v = 4 * i;
      if (argmax_better(x.x, v, best, idx)) { best = x.x; idx = v; }
      if (argmax_better(x.y, v + 1, best, idx)) { best = x.y; idx = v + 1; }
      if (argmax_better(x.z, v + 2, best, idx)) { best = x.z; idx = v + 2; }
      if (argmax_better(x.w, v + 3, best, idx)) { best = x.w; idx = v + 3; }
    }
  } else {
    for (int v = lane; v < V; v += 32) {
      const float x = __ldg(row + v);
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
