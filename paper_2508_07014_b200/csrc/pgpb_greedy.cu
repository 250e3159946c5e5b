// Fused boosted greedy decoding kernels.
//
//  * ctc_greedy_kernel: batched two-stage greedy CTC (_kernels.pyx:75-225,
//    decoding.py:156-229, R6).  One warp per utterance walks its frames in
//    order; the boosted rerank resolves the current state's scores on the
//    fly from the flattened closure + shared-memory root row, so the [B,V]
//    score matrix never exists.
//  * greedy_step_kernel: one label-looping transducer step over B rows
//    (decoding.py:373-392, R7): argmax, blank test, boosted rerank.
//  * row_max_kernel: max_v score[s, v] per state (AED eos bump,
//    decoding.py:546-552).
//
// Numerics: fused score = (double)lp + lam * (double)s, two separately
// rounded fp64 ops (no FMA, as the reference's compiled code); ties break
// toward higher raw logprob, then lower token id.

#include <string>

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

template <bool kVec>
__global__ void __launch_bounds__(kThreads)
    ctc_greedy_kernel(TableView t, int use_boost, int smem_root, const float *__restrict__ lp,
                      int64_t B, int64_t T, int V, const int32_t *__restrict__ lengths, int blank,
                      double lam, int32_t *__restrict__ tokens, double *__restrict__ deltas,
                      int32_t *__restrict__ ostates, int32_t *__restrict__ nout,
                      double *__restrict__ am_out, double *__restrict__ boost_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const float *root;
  const int32_t *rnext;
  unsigned *bm;
  setup_smem(t, use_boost, smem_root, smem, root, rnext, bm);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < B; b += nwarps) {
    const int64_t Tb = lengths ? static_cast<int64_t>(__ldg(lengths + b)) : T;
    double am = 0.0, boost = 0.0;
    int last = -1, state = 0;
    int64_t n = 0;
    for (int64_t tt = 0; tt < Tb; ++tt) {
      const float *row = lp + (b * T + tt) * V;
      float best;
      int a;
      warp_row_argmax<kVec>(row, V, lane, best, a);
      if (a == blank || a == last) {  // blank / repeat pass through (R6)
        am += static_cast<double>(best);
        last = a;
        continue;
      }
      RerankOut r;
      if (use_boost) {
        r = warp_rerank<kVec>(t, root, rnext, bm, row, V, state, blank, last, lam, lane);
      } else {
        r.chosen = a;
        r.lp = best;
        r.delta = 0.0;
        r.next = 0;
      }
      if (lane == 0) {
        tokens[b * T + n] = r.chosen;
        deltas[b * T + n] = r.delta;
        ostates[b * T + n] = r.next;
      }
      ++n;
      am += static_cast<double>(r.lp);
      boost += r.delta;
      state = r.next;
      last = r.chosen;
    }
    if (lane == 0) {
      nout[b] = static_cast<int32_t>(n);
      am_out[b] = am;
      boost_out[b] = boost;
    }
  }
}

template <bool kVec>
__global__ void __launch_bounds__(kThreads)
    greedy_step_kernel(TableView t, int use_boost, int smem_root, const float *__restrict__ lp,
                       int64_t ld, int64_t R, int V, const int32_t *__restrict__ states,
                       const uint8_t *__restrict__ active, int blank, double lam,
                       int32_t *__restrict__ chosen, float *__restrict__ lp_chosen,
                       double *__restrict__ delta, int32_t *__restrict__ next_state,
                       uint8_t *__restrict__ is_blank) {
  extern __shared__ __align__(16) unsigned char smem[];
  const float *root;
  const int32_t *rnext;
  unsigned *bm;
  setup_smem(t, use_boost, smem_root, smem, root, rnext, bm);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    if (active && !__ldg(active + r)) continue;
    const float *row = lp + r * ld;
    float best;
    int a;
    warp_row_argmax<kVec>(row, V, lane, best, a);
    RerankOut o;
    const bool blk = (a == blank);
    if (blk || !use_boost) {
      o.chosen = a;
      o.lp = best;
      o.delta = 0.0;
      o.next = 0;
    } else {
      o = warp_rerank<kVec>(t, root, rnext, bm, row, V, __ldg(states + r), blank, -1, lam, lane);
    }
    if (lane == 0) {
      chosen[r] = o.chosen;
      lp_chosen[r] = o.lp;
      delta[r] = o.delta;
      next_state[r] = o.next;
      is_blank[r] = blk ? 1 : 0;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    row_max_kernel(TableView t, int smem_root, float *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const float *root;
  const int32_t *rnext;
  unsigned *bm;
  setup_smem(t, true, smem_root, smem, root, rnext, bm);
  const int lane = threadIdx.x & 31;
  const int V = t.vocab_size;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < t.num_states; s += nwarps) {
    const int4 rec = __ldg(t.clo_rec + s);
    const float acc = __int_as_float(rec.z);
    mark_closure(t, rec, bm, lane, true);
    __syncwarp();
    float m = -INFINITY;
    for (int v = lane; v < V; v += 32)
      if (!((bm[v >> 5] >> (v & 31)) & 1u)) m = fmaxf(m, acc + root[v]);
    for (int i = lane; i < rec.y; i += 32) m = fmaxf(m, __int_as_float(__ldg(&t.clo[rec.x + i].z)));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) out[s] = m;
    __syncwarp();
    mark_closure(t, rec, bm, lane, false);
    __syncwarp();
  }
}

static size_t greedy_smem(const TableView &t, bool use_boost, bool &smem_root) {
  const size_t bm = size_t((t.vocab_size + 31) >> 5) * 4 * kWarpsPerBlock;
  const size_t root = size_t(t.vocab_padded) * 8;
  smem_root = use_boost && root + bm <= size_t(kMaxSmemRootBytes);
  return (use_boost ? bm : 0) + (smem_root ? root : 0);
}

template <typename F>
static int prep_kernel(F fn, size_t smem) {
  if (smem > 48 * 1024) {
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  return PGPB_OK;
}

// Placeholder view for unboosted calls without a table.
static TableView empty_view(int V) {
  TableView v{};
  v.num_states = 1;
  v.vocab_size = V;
  v.vocab_padded = (V + 3) & ~3;
  return v;
}

}  // namespace pgpb

extern "C" {

int pgpb_ctc_greedy(const pgpb_table *table, const float *d_lp, int64_t B, int64_t T, int32_t V,
                    const int32_t *d_lengths, int32_t blank, double lam, int32_t use_boost,
                    int32_t *d_tokens, double *d_deltas, int32_t *d_states, int32_t *d_num_out,
                    double *d_am, double *d_boost, void *stream) {
  using namespace pgpb;
  if (B < 0 || T < 0 || V < 1) return fail(PGPB_EINVAL, "bad shape");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "emission vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (B == 0) return PGPB_OK;
  const TableView t = table ? table->view : empty_view(V);
  bool smem_root = false;
  const size_t smem = greedy_smem(t, use_boost != 0, smem_root);
  const bool vec = (V % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  auto fn = vec ? ctc_greedy_kernel<true> : ctc_greedy_kernel<false>;
  int rc = prep_kernel(fn, smem);
  if (rc) return rc;
  const unsigned grid = warp_grid(B, 4);
  fn<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      t, use_boost ? 1 : 0, smem_root ? 1 : 0, d_lp, B, T, V, d_lengths, blank, lam, d_tokens,
      d_deltas, d_states, d_num_out, d_am, d_boost);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_ctc_greedy_host(const pgpb_table *table, const float *h_lp, int64_t T, int32_t V,
                         int32_t blank, double lam, int32_t use_boost, int32_t *h_tokens,
                         double *h_deltas, int32_t *h_states, int64_t *num_out, double *h_am,
                         double *h_boost, void *stream) {
  using namespace pgpb;
  if (T < 0 || V < 1) return fail(PGPB_EINVAL, "bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t lp_bytes = size_t(T) * size_t(V) * 4;
  const size_t Tn = size_t(T > 0 ? T : 1);
  // layout: lp | tokens | states | deltas | am | boost | nout
  const size_t o_tok = ((lp_bytes + 255) / 256) * 256;
  const size_t o_st = o_tok + ((Tn * 4 + 255) / 256) * 256;
  const size_t o_dl = o_st + ((Tn * 4 + 255) / 256) * 256;
  const size_t o_am = o_dl + ((Tn * 8 + 255) / 256) * 256;
  const size_t total = o_am + 256;
  char *buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, total, st);
  if (e != cudaSuccess) return fail(PGPB_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  int32_t *d_tok = reinterpret_cast<int32_t *>(buf + o_tok);
  int32_t *d_st = reinterpret_cast<int32_t *>(buf + o_st);
  double *d_dl = reinterpret_cast<double *>(buf + o_dl);
  double *d_am = reinterpret_cast<double *>(buf + o_am);
  double *d_bo = d_am + 1;
  int32_t *d_n = reinterpret_cast<int32_t *>(d_am + 2);
  int rc = PGPB_OK;
  e = cudaMemcpyAsync(buf, h_lp, lp_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    rc = pgpb_ctc_greedy(table, reinterpret_cast<const float *>(buf), 1, T, V, nullptr, blank, lam,
                         use_boost, d_tok, d_dl, d_st, d_n, d_am, d_bo, stream);
  double scal[2] = {0.0, 0.0};
  int32_t n = 0;
  if (e == cudaSuccess && rc == PGPB_OK) e = cudaMemcpyAsync(scal, d_am, 16, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && rc == PGPB_OK) e = cudaMemcpyAsync(&n, d_n, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && rc == PGPB_OK) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && rc == PGPB_OK && n > 0) {
    e = cudaMemcpyAsync(h_tokens, d_tok, size_t(n) * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_states, d_st, size_t(n) * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_deltas, d_dl, size_t(n) * 8, cudaMemcpyDeviceToHost, st);
  }
  cudaFreeAsync(buf, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (rc != PGPB_OK) return rc;
  if (e != cudaSuccess) return fail(PGPB_ECUDA, std::string("ctc_greedy_host: ") + cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(PGPB_ECUDA, std::string("ctc_greedy_host sync: ") + cudaGetErrorString(e2));
  *num_out = n;
  *h_am = scal[0];
  *h_boost = scal[1];
  return PGPB_OK;
}

int pgpb_greedy_step(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t R, int32_t V,
                     const int32_t *d_states, const uint8_t *d_active, int32_t blank, double lam,
                     int32_t use_boost, int32_t *d_chosen, float *d_lp_chosen, double *d_delta,
                     int32_t *d_next, uint8_t *d_is_blank, void *stream) {
  using namespace pgpb;
  if (R < 0 || V < 1 || ld < V) return fail(PGPB_EINVAL, "bad shape");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "step model vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (R == 0) return PGPB_OK;
  const TableView t = table ? table->view : empty_view(V);
  bool smem_root = false;
  const size_t smem = greedy_smem(t, use_boost != 0, smem_root);
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  auto fn = vec ? greedy_step_kernel<true> : greedy_step_kernel<false>;
  int rc = prep_kernel(fn, smem);
  if (rc) return rc;
  const unsigned grid = warp_grid(R, 4);
  fn<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      t, use_boost ? 1 : 0, smem_root ? 1 : 0, d_lp, ld, R, V, d_states, d_active, blank, lam,
      d_chosen, d_lp_chosen, d_delta, d_next, d_is_blank);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_row_max(const pgpb_table *table, float *d_out, void *stream) {
  using namespace pgpb;
  if (!table || !d_out) return fail(PGPB_EINVAL, "NULL argument");
  const TableView &t = table->view;
  bool smem_root = false;
  const size_t smem = greedy_smem(t, true, smem_root);
  int rc = prep_kernel(row_max_kernel, smem);
  if (rc) return rc;
  const unsigned grid = warp_grid(t.num_states, 4);
  row_max_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(t, smem_root ? 1 : 0, d_out);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

}  // extern "C"
