// Fused boosted greedy decoding kernels.
//
//  (the batched greedy CTC kernels live in pgpb_ctc.cu)
//  * greedy_step_kernel: one label-looping transducer step over B rows
//    (decoding.py:373-392, R7): argmax, blank test, boosted rerank.
//  * row_max_kernel: max_v score[s, v] per state (AED eos bump,
//    decoding.py:546-552).
//
// Numerics: fused score = (double)lp + lam * (double)s, two separately
// rounded fp64 ops (no FMA, as the reference's compiled code); ties break
// toward higher raw logprob, then lower token id.

#include <string>

#include "pgpb_rerank.cuh"

namespace pgpb {

constexpr int kStepTopM = 4;

// One label-looping step: a warp per row makes one pass over the row for
// its top-M tokens (entry 0 = the argmax), then, for non-blank rows with
// boosting on, resolves the rerank with blob_rerank (closure arcs exact,
// dense tokens among the top-M, exact bound, full-row fallback).
template <bool kVec>
__global__ void __launch_bounds__(kThreads)
    greedy_step_kernel(TableView t, int use_boost, const float *__restrict__ lp, int64_t ld, int64_t R,
                       int V, const int32_t *__restrict__ states, const uint8_t *__restrict__ active,
                       int blank, double lam, int32_t *__restrict__ chosen, float *__restrict__ lp_chosen,
                       double *__restrict__ delta, int32_t *__restrict__ next_state,
                       uint8_t *__restrict__ is_blank) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Vp = t.vocab_padded, Vw = (V + 31) >> 5;
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_rnext = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  int32_t *s_rnoff = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 8);
  unsigned *bm = reinterpret_cast<unsigned *>(smem + size_t(Vp) * 12) + (threadIdx.x >> 5) * Vw;
  const int lane = threadIdx.x & 31;
  if (use_boost) {
    for (int i = threadIdx.x; i < Vp; i += blockDim.x) {
      s_root[i] = __ldg(t.root_scores + i);
      s_rnext[i] = __ldg(t.root_next + i);
      s_rnoff[i] = __ldg(t.root_next_off + i);
    }
    for (int i = lane; i < Vw; i += 32) bm[i] = 0u;
  }
  __syncthreads();
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    if (active && !__ldg(active + r)) continue;
    const float *row = lp + r * ld;
    int tv[kStepTopM];
    float tx[kStepTopM];
    warp_row_topm<kStepTopM, kVec>(row, V, lane, tv, tx);
    const int a = tv[0];
    const bool blk = (a == blank);
    int c = a, nx = 0;
    float lpc = tx[0];
    double d = 0.0;
    if (!blk && use_boost) {
      const int soff = __ldg(t.blob_off + __ldg(states + r));
      const BCand w = blob_rerank<kStepTopM>(t, s_root, s_rnext, s_rnoff, bm, row, V, soff, tv, tx, blank, -1,
                                             lam, t.max_root_score, lane);
      c = w.v;
      lpc = w.lp;
      d = static_cast<double>(w.s);
      nx = w.nx;
    }
    if (lane == 0) {
      chosen[r] = c;
      lp_chosen[r] = lpc;
      delta[r] = d;
      next_state[r] = nx;
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

}  // namespace pgpb

extern "C" {

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
  const size_t smem = use_boost ? size_t(t.vocab_padded) * 12 + size_t(kWarpsPerBlock) * ((V + 31) >> 5) * 4 : 0;
  if (smem > 220 * 1024) return fail(PGPB_EINVAL, "vocabulary too large for the shared-memory root row");
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  auto fn = vec ? greedy_step_kernel<true> : greedy_step_kernel<false>;
  int rc = prep_kernel(fn, smem);
  if (rc) return rc;
  const unsigned grid = warp_grid(R, 4);
  fn<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      t, use_boost ? 1 : 0, d_lp, ld, R, V, d_states, d_active, blank, lam, d_chosen, d_lp_chosen, d_delta,
      d_next, d_is_blank);
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
