// Batched fused greedy CTC with shallow-fusion boosting: C-ABI entry points.
//
// Reference: _kernels.ctc_greedy (_kernels.pyx:75-225) and
// ctc_greedy_boosted (decoding.py:156-229), R6 in SURVEY.md.  The kernels
// live in pgpb_ctc_spec.cu: phase A (frame_top2_kernel, HBM-bound argmax +
// runner-up per frame) and phase B (ctc_walk_kernel, the speculative
// chunked walker with the fused boosted rerank); DESIGN.md §4.  The earlier
// two-phase kernels (top-M + one warp per utterance) are retired; their
// measurements are in profiles/r1_ctc_summary.md.
//
// Bit-exact with the reference per utterance: argmax first-max semantics,
// fp64 fusion lp + lam*s with two separately rounded ops, ties broken by
// higher raw logprob then lower token id.

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

int ctc_spec_launch(const pgpb_table *table, const float *d_lp, int64_t B, int64_t T, int32_t V,
                    const int32_t *d_lengths, int32_t blank, double lam, int32_t use_boost, int32_t *d_tokens,
                    double *d_deltas, int32_t *d_states, int32_t *d_num_out, double *d_am, double *d_boost,
                    cudaStream_t st);

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
  return ctc_spec_launch(table, d_lp, B, T, V, d_lengths, blank, lam, use_boost, d_tokens, d_deltas, d_states,
                         d_num_out, d_am, d_boost, static_cast<cudaStream_t>(stream));
}

int pgpb_ctc_greedy_host(const pgpb_table *table, const float *h_lp, int64_t T, int32_t V,
                         int32_t blank, double lam, int32_t use_boost, int32_t *h_tokens,
                         double *h_deltas, int32_t *h_states, int64_t *num_out, double *h_am,
                         double *h_boost, void *stream) {
  using namespace pgpb;
  if (T < 0 || V < 1) return fail(PGPB_EINVAL, "bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  retain_pool(current_device());
  const size_t lp_bytes = size_t(T) * size_t(V) * 4;
  const size_t Tn = size_t(T > 0 ? T : 1);
  // layout: lp | tokens | states | deltas | am, boost, nout
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

}  // extern "C"
