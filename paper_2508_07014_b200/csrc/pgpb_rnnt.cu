// Prediction / joint network kernels of the config-2 label-looping RNN-T
// decoder (rnnt.py).  These are not reference interfaces: the reference
// decodes with a host StepModel (acoustic.py:203-255); the networks here are
// the random-init stand-ins of the paper's shapes (LSTM-640 prediction net +
// joint) that produce the log-probs the GPU-PB step consumes.
// They fuse the elementwise glue around the library GEMMs so that one label
// iteration is 3 GEMMs + 3 kernels (joint hidden, fused log-softmax + boosted
// step in pgpb_greedy.cu, LSTM cell update) instead of ~18 framework kernels.
//
//  * joint_hidden_kernel: z[b] = relu(enc_proj[b, min(t[b], len[b]-1)] +
//    pred_proj[b]) in bf16 (the frame gather, add and ReLU of the joint).
//  * lstm_update_kernel: gates = E[feed[b]] + hg[b] (E = emb @ W_ih^T + b_ih
//    precomputed per token, hg = h @ W_hh^T + b_hh), torch's LSTM cell
//    (gate order i, f, g, o; fp32 math, bf16 state), and h, c overwritten
//    only for rows that emitted (the prediction net advances on emissions).

#include <cuda_bf16.h>

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

__global__ void __launch_bounds__(256)
    joint_hidden_kernel(const __nv_bfloat16 *__restrict__ enc, int64_t ld_b, int J, const int64_t *__restrict__ t,
                        const int64_t *__restrict__ lengths, const __nv_bfloat16 *__restrict__ pp, int64_t ld_pp,
                        __nv_bfloat16 *__restrict__ z) {
  const int64_t b = blockIdx.x;
  const int64_t len = lengths[b];
  int64_t tf = t[b];
  const int64_t lim = len > 0 ? len - 1 : 0;
  if (tf > lim) tf = lim;
  const __nv_bfloat16 *e = enc + b * ld_b + tf * J;
  const __nv_bfloat16 *p = pp + b * ld_pp;
  __nv_bfloat16 *o = z + b * J;
  if ((J & 7) == 0 && ((reinterpret_cast<uintptr_t>(e) | reinterpret_cast<uintptr_t>(p) |
                        reinterpret_cast<uintptr_t>(o)) & 15) == 0) {
    // 8 bf16 per 16-byte access
    for (int j = threadIdx.x; j < (J >> 3); j += blockDim.x) {
      const uint4 qe = reinterpret_cast<const uint4 *>(e)[j], qp = reinterpret_cast<const uint4 *>(p)[j];
      const __nv_bfloat162 *he = reinterpret_cast<const __nv_bfloat162 *>(&qe);
      const __nv_bfloat162 *hp = reinterpret_cast<const __nv_bfloat162 *>(&qp);
      uint4 qo;
      __nv_bfloat162 *ho = reinterpret_cast<__nv_bfloat162 *>(&qo);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 a = __bfloat1622float2(he[i]), c = __bfloat1622float2(hp[i]);
        const __nv_bfloat162 sum = __floats2bfloat162_rn(a.x + c.x, a.y + c.y);
        const float2 r = __bfloat1622float2(sum);
        ho[i] = __floats2bfloat162_rn(r.x > 0.0f ? r.x : 0.0f, r.y > 0.0f ? r.y : 0.0f);
      }
      reinterpret_cast<uint4 *>(o)[j] = qo;
    }
    return;
  }
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const __nv_bfloat16 s = __float2bfloat16_rn(__bfloat162float(e[j]) + __bfloat162float(p[j]));
    o[j] = __hgt(s, __float2bfloat16_rn(0.0f)) ? s : __float2bfloat16_rn(0.0f);
  }
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

__global__ void __launch_bounds__(256)
    lstm_update_kernel(const __nv_bfloat16 *__restrict__ E, const int64_t *__restrict__ feed,
                       const __nv_bfloat16 *__restrict__ hg, int64_t ld_hg, const uint8_t *__restrict__ emit,
                       __nv_bfloat16 *__restrict__ h, __nv_bfloat16 *__restrict__ c, int H) {
  const int64_t b = blockIdx.x;
  if (emit && !emit[b]) return;
  const __nv_bfloat16 *ex = E + feed[b] * int64_t(4 * H);
  const __nv_bfloat16 *hx = hg + b * ld_hg;
  if ((H & 1) == 0) {
    // two hidden units per thread (bf16x2 accesses)
    const __nv_bfloat162 *e2 = reinterpret_cast<const __nv_bfloat162 *>(ex);
    const __nv_bfloat162 *x2 = reinterpret_cast<const __nv_bfloat162 *>(hx);
    __nv_bfloat162 *c2 = reinterpret_cast<__nv_bfloat162 *>(c + b * H);
    __nv_bfloat162 *h2 = reinterpret_cast<__nv_bfloat162 *>(h + b * H);
    const int H2 = H >> 1;
    for (int j = threadIdx.x; j < H2; j += blockDim.x) {
      float2 g[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 a = __bfloat1622float2(e2[q * H2 + j]), d = __bfloat1622float2(x2[q * H2 + j]);
        g[q] = make_float2(a.x + d.x, a.y + d.y);
      }
      const float2 cp = __bfloat1622float2(c2[j]);
      const float cx = sigm(g[1].x) * cp.x + sigm(g[0].x) * tanhf(g[2].x);
      const float cy = sigm(g[1].y) * cp.y + sigm(g[0].y) * tanhf(g[2].y);
      c2[j] = __floats2bfloat162_rn(cx, cy);
      h2[j] = __floats2bfloat162_rn(sigm(g[3].x) * tanhf(cx), sigm(g[3].y) * tanhf(cy));
    }
    return;
  }
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float gi = __bfloat162float(ex[j]) + __bfloat162float(hx[j]);
    const float gf = __bfloat162float(ex[H + j]) + __bfloat162float(hx[H + j]);
    const float gg = __bfloat162float(ex[2 * H + j]) + __bfloat162float(hx[2 * H + j]);
    const float go = __bfloat162float(ex[3 * H + j]) + __bfloat162float(hx[3 * H + j]);
    const float cn = sigm(gf) * __bfloat162float(c[b * H + j]) + sigm(gi) * tanhf(gg);
    const float hn = sigm(go) * tanhf(cn);
    c[b * H + j] = __float2bfloat16_rn(cn);
    h[b * H + j] = __float2bfloat16_rn(hn);
  }
}

// Stateless-transducer beam joint (beams.py): z[b, k] = relu(enc_proj[b,
// min(t[b], len[b]-1)] + pred_j[ctx]), ctx = last[b, k] (blank when < 0),
// one block per (b, k) row.
__global__ void __launch_bounds__(128)
    beam_hidden_kernel(const __nv_bfloat16 *__restrict__ enc, int64_t ld_b, int J, const int32_t *__restrict__ t,
                       const int32_t *__restrict__ lengths, const __nv_bfloat16 *__restrict__ pred_j,
                       const int32_t *__restrict__ last, int K, int blank, __nv_bfloat16 *__restrict__ z) {
  const int64_t row = blockIdx.x, b = row / K;
  const int len = lengths[b];
  int tf = t[b];
  const int lim = len > 0 ? len - 1 : 0;
  if (tf > lim) tf = lim;
  const int ctx = last[row] < 0 ? blank : last[row];
  const __nv_bfloat16 *e = enc + b * ld_b + int64_t(tf) * J;
  const __nv_bfloat16 *p = pred_j + int64_t(ctx) * J;
  __nv_bfloat16 *o = z + row * J;
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const float sv = __bfloat162float(__float2bfloat16_rn(__bfloat162float(e[j]) + __bfloat162float(p[j])));
    o[j] = __float2bfloat16_rn(sv > 0.0f ? sv : 0.0f);
  }
}

}  // namespace pgpb

extern "C" {

int pgpb_rnnt_beam_hidden(const void *d_enc_proj, int64_t ld_b, int32_t J, const int32_t *d_t,
                          const int32_t *d_lengths, const void *d_pred_j, const int32_t *d_last, int64_t B, int32_t K,
                          int32_t blank, void *d_z, void *stream) {
  using namespace pgpb;
  if (B < 0 || J < 1 || K < 1 || ld_b < J) return fail(PGPB_EINVAL, "bad shape");
  if (B == 0) return PGPB_OK;
  if (!d_enc_proj || !d_t || !d_lengths || !d_pred_j || !d_last || !d_z) return fail(PGPB_EINVAL, "NULL buffer");
  beam_hidden_kernel<<<unsigned(B * K), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16 *>(d_enc_proj), ld_b, J, d_t, d_lengths,
      static_cast<const __nv_bfloat16 *>(d_pred_j), d_last, K, blank, static_cast<__nv_bfloat16 *>(d_z));
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_rnnt_joint_hidden(const void *d_enc_proj, int64_t ld_b, int32_t J, const int64_t *d_t,
                           const int64_t *d_lengths, const void *d_pred_proj, int64_t ld_pred, void *d_z, int64_t B,
                           void *stream) {
  using namespace pgpb;
  if (B < 0 || J < 1 || ld_b < J || ld_pred < J) return fail(PGPB_EINVAL, "bad shape");
  if (B == 0) return PGPB_OK;
  if (!d_enc_proj || !d_t || !d_lengths || !d_pred_proj || !d_z) return fail(PGPB_EINVAL, "NULL buffer");
  joint_hidden_kernel<<<unsigned(B), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16 *>(d_enc_proj), ld_b, J, d_t, d_lengths,
      static_cast<const __nv_bfloat16 *>(d_pred_proj), ld_pred, static_cast<__nv_bfloat16 *>(d_z));
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_rnnt_lstm_update(const void *d_E, const int64_t *d_feed, const void *d_hg, int64_t ld_hg,
                          const uint8_t *d_emit, void *d_h, void *d_c, int64_t B, int32_t H, void *stream) {
  using namespace pgpb;
  if (B < 0 || H < 1 || ld_hg < 4 * int64_t(H)) return fail(PGPB_EINVAL, "bad shape");
  if (B == 0) return PGPB_OK;
  if (!d_E || !d_feed || !d_hg || !d_h || !d_c) return fail(PGPB_EINVAL, "NULL buffer");
  lstm_update_kernel<<<unsigned(B), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16 *>(d_E), d_feed, static_cast<const __nv_bfloat16 *>(d_hg), ld_hg, d_emit,
      static_cast<__nv_bfloat16 *>(d_h), static_cast<__nv_bfloat16 *>(d_c), H);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

}  // extern "C"
