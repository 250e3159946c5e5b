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

#include <algorithm>
#include <cstdlib>
#include <string>

#include <cuda_bf16.h>

#include "pgpb_rerank.cuh"

namespace pgpb {

constexpr int kStepTopM = 4;

// Per-row decision shared by the step and label-loop kernels: one pass over
// the row for its top-M tokens (entry 0 = the stage-1 argmax); for a
// non-blank argmax with boosting on, blob_rerank (closure arcs exact, dense
// tokens among the top-M, exact bound, full-row fallback).  Root-row reads
// go through L1/L2 (a handful per row), so no shared staging is needed.
struct RowDecision {
  int chosen;
  float lp;
  double delta;
  int next;
  bool blank;
  int noff;  // blob offset of next (boosted decisions)
};

// decide_row with the state's blob already loaded (issued before the row's
// own work, so its dependent round trips overlap the top-M pass).
__device__ __forceinline__ RowDecision decide_topm(const TableView &t, const float *row, int V, int blank, double lam,
                                                   int use_boost, const BlobRegs &cur, unsigned *bm,
                                                   const int (&tv)[kStepTopM], const float (&tx)[kStepTopM],
                                                   int lane) {
  RowDecision d{tv[0], tx[0], 0.0, 0, tv[0] == blank, -1};
  if (!d.blank && use_boost) {
    const BCand w = blob_rerank_regs<kStepTopM>(t, cur, t.root_scores, t.root_next, t.root_next_off, bm, row, V, tv,
                                                tx, blank, -1, lam, t.max_root_score, lane);
    d.chosen = w.v;
    d.lp = w.lp;
    d.delta = static_cast<double>(w.s);
    d.next = w.nx;
    d.noff = w.noff;
  }
  return d;
}

template <int NC>
__device__ __forceinline__ RowDecision decide_row_pre(const TableView &t, const float *row, int V, int blank,
                                                      double lam, int use_boost, const BlobRegs &cur, unsigned *bm,
                                                      float *sv, int *si, int lane) {
  int tv[kStepTopM];
  float tx[kStepTopM];
  if (NC > 0)
    warp_row_topm_thr<kStepTopM, (NC > 0 ? NC : 1)>(row, V, lane, sv, si, tv, tx);
  else
    warp_row_topm<kStepTopM, false>(row, V, lane, tv, tx);
  return decide_topm(t, row, V, blank, lam, use_boost, cur, bm, tv, tx, lane);
}

// Log-softmax of bf16 logits into registers in the float4-chunk layout of
// the register top-M (x[k] = elements 4 (lane + 32 k) .. + 3), written out
// to y as well.  V % 4 == 0, 8-byte aligned logits, 16-byte aligned y.
template <int NC>
__device__ __forceinline__ void lsm_regs_bf16(const __nv_bfloat16 *__restrict__ x, float *__restrict__ y, int V,
                                              int lane, float4 (&o)[NC]) {
  const int V4 = V >> 2;
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = lane + 32 * k;
    uint2 q = make_uint2(0u, 0u);
    if (c < V4) q = __ldg(reinterpret_cast<const uint2 *>(x) + c);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&q.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&q.y));
    o[k] = c < V4 ? make_float4(a.x, a.y, b.x, b.y) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    m = fmaxf(m, fmaxf(fmaxf(o[k].x, o[k].y), fmaxf(o[k].z, o[k].w)));
  }
  float mr;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < NC; ++k)
    s += expf(o[k].x - mr) + expf(o[k].y - mr) + expf(o[k].z - mr) + expf(o[k].w - mr);
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  const float ls = logf(s);
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c = lane + 32 * k;
    if (c < V4) {
      o[k] = make_float4((o[k].x - mr) - ls, (o[k].y - mr) - ls, (o[k].z - mr) - ls, (o[k].w - mr) - ls);
      reinterpret_cast<float4 *>(y)[c] = o[k];
    }
  }
  __syncwarp();  // the row may be read back by the decision (memory ordering)
}

template <int NC>
__device__ __forceinline__ RowDecision decide_row(const TableView &t, const float *row, int V, int blank, double lam,
                                                  int use_boost, int state, unsigned *bm, float *sv, int *si,
                                                  int lane) {
  int tv[kStepTopM];
  float tx[kStepTopM];
  if (NC > 0)
    warp_row_topm_thr<kStepTopM, (NC > 0 ? NC : 1)>(row, V, lane, sv, si, tv, tx);
  else
    warp_row_topm<kStepTopM, false>(row, V, lane, tv, tx);
  RowDecision d{tv[0], tx[0], 0.0, 0, tv[0] == blank};
  if (!d.blank && use_boost) {
    const int soff = __ldg(t.blob_off + state);
    const BCand w = blob_rerank<kStepTopM>(t, t.root_scores, t.root_next, t.root_next_off, bm, row, V, soff, tv, tx,
                                           blank, -1, lam, t.max_root_score, lane);
    d.chosen = w.v;
    d.lp = w.lp;
    d.delta = static_cast<double>(w.s);
    d.next = w.nx;
  }
  return d;
}

struct StepScratch {
  unsigned *bm;
  float *sv;
  int *si;
};

__device__ __forceinline__ StepScratch step_scratch(unsigned char *smem, int V, int use_boost) {
  const int Vw = (V + 31) >> 5;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StepScratch s;
  s.sv = reinterpret_cast<float *>(smem) + wib * 64;
  s.si = reinterpret_cast<int *>(s.sv + 32);
  s.bm = reinterpret_cast<unsigned *>(smem + kWarpsPerBlock * 256) + wib * Vw;
  if (use_boost)
    for (int i = lane; i < Vw; i += 32) s.bm[i] = 0u;
  __syncwarp();
  return s;
}

template <int NC>
__global__ void __launch_bounds__(kThreads)
    greedy_step_kernel(TableView t, int use_boost, const float *__restrict__ lp, int64_t ld, int64_t R, int V,
                       const int32_t *__restrict__ states, const uint8_t *__restrict__ active, int blank, double lam,
                       int32_t *__restrict__ chosen, float *__restrict__ lp_chosen, double *__restrict__ delta,
                       int32_t *__restrict__ next_state, uint8_t *__restrict__ is_blank) {
  extern __shared__ __align__(16) unsigned char smem[];
  const StepScratch sc = step_scratch(smem, V, use_boost);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    if (active && !__ldg(active + r)) continue;
    const RowDecision d = decide_row<NC>(t, lp + r * ld, V, blank, lam, use_boost,
                                         use_boost ? __ldg(states + r) : 0, sc.bm, sc.sv, sc.si, lane);
    if (lane == 0) {
      chosen[r] = d.chosen;
      lp_chosen[r] = d.lp;
      delta[r] = d.delta;
      next_state[r] = d.next;
      is_blank[r] = d.blank ? 1 : 0;
    }
  }
}

// Row log-softmax of bf16 logits into f32 (torch's formula order:
// (x - max) - log(sum exp(x - max)), accurate expf / logf), one warp.
__device__ __forceinline__ void warp_log_softmax_bf16(const __nv_bfloat16 *__restrict__ x, float *__restrict__ y,
                                                      int V, int lane) {
  if (V <= 1024 && (V & 7) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
    // register path: 8 bf16 per 16-byte load, the row read once
    const int V8 = V >> 3;
    float v[32];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = lane + 32 * k;
      uint4 q = make_uint4(0u, 0u, 0u, 0u);
      if (c < V8) q = __ldg(reinterpret_cast<const uint4 *>(x) + c);
      const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&q);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        v[8 * k + 2 * i] = c < V8 ? f.x : -INFINITY;
        v[8 * k + 2 * i + 1] = c < V8 ? f.y : -INFINITY;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) m = fmaxf(m, v[i]);
    float mr;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 32; ++i) s += expf(v[i] - mr);  // padding: expf(-inf) = 0
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    const float ls = logf(s);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = lane + 32 * k;
      if (c < V8) {
        float4 *o4 = reinterpret_cast<float4 *>(y + 8 * c);
        o4[0] = make_float4((v[8 * k] - mr) - ls, (v[8 * k + 1] - mr) - ls, (v[8 * k + 2] - mr) - ls,
                            (v[8 * k + 3] - mr) - ls);
        o4[1] = make_float4((v[8 * k + 4] - mr) - ls, (v[8 * k + 5] - mr) - ls, (v[8 * k + 6] - mr) - ls,
                            (v[8 * k + 7] - mr) - ls);
      }
    }
    __syncwarp();
    return;
  }
  float m = -INFINITY;
  for (int v = lane; v < V; v += 32) m = fmaxf(m, __bfloat162float(x[v]));
  float mr;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
  float s = 0.0f;
  for (int v = lane; v < V; v += 32) s += expf(__bfloat162float(x[v]) - mr);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  const float ls = logf(s);
  for (int v = lane; v < V; v += 32) y[v] = (__bfloat162float(x[v]) - mr) - ls;
  __syncwarp();  // the row is read back by the whole warp (memory ordering)
}

template <int NC>
__global__ void __launch_bounds__(kThreads)
    label_loop_kernel(TableView t, int use_boost, const float *lp, int64_t ld, int64_t R, int V,
                      int blank, double lam, pgpb_label_loop_state st, uint8_t *__restrict__ emit,
                      int64_t *__restrict__ feed, int32_t *__restrict__ any_active,
                      const __nv_bfloat16 *__restrict__ logits, int64_t ld_logits) {
  extern __shared__ __align__(16) unsigned char smem[];
  const StepScratch sc = step_scratch(smem, V, use_boost);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const bool regs_ok = logits && (V & 3) == 0 && (ld_logits & 3) == 0 &&
                       (reinterpret_cast<uintptr_t>(logits) & 7) == 0;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    const int64_t tr = st.t[r], len = st.lengths[r];
    if (tr >= len) {  // finished utterance: nothing to decide
      if (lane == 0) {
        emit[r] = 0;
        feed[r] = st.last[r];
      }
      continue;
    }
    // the row's bookkeeping state, loaded up front so that its round trips
    // overlap the row's work (the R7 update below is then register-only)
    const double am0 = st.am[r], bo0 = st.boost[r];
    const int64_t k0 = st.k[r], n0 = st.n[r];
    const int dur = st.durations ? st.durations[r] : -1;  // TDT duration head argmax, or RNN-T
    // the tree state's blob first: its two dependent round trips overlap
    // the row's log-softmax and top-M pass
    BlobRegs cur{};
    if (use_boost) {
      int so = st.tree_off ? st.tree_off[r] : -1;
      if (so < 0) so = __ldg(t.blob_off + st.tree[r]);
      cur = load_blob(t, so, lane);
    }
    // fused joint tail: log-softmax of the row's logits, written out (the
    // row the decision reads, and the record of what was decided on); with
    // the register top-M the row's values go straight from the softmax
    RowDecision d;
    if (logits && NC > 0 && regs_ok) {
      float4 x[NC > 0 ? NC : 1];
      lsm_regs_bf16<(NC > 0 ? NC : 1)>(logits + r * ld_logits, const_cast<float *>(lp) + r * ld, V, lane, x);
      int tv[kStepTopM];
      float tx[kStepTopM];
      warp_regs_topm_thr<kStepTopM, (NC > 0 ? NC : 1)>(x, V, lane, sc.sv, sc.si, tv, tx);
      d = decide_topm(t, lp + r * ld, V, blank, lam, use_boost, cur, sc.bm, tv, tx, lane);
    } else {
      if (logits) warp_log_softmax_bf16(logits + r * ld_logits, const_cast<float *>(lp) + r * ld, V, lane);
      d = decide_row_pre<NC>(t, lp + r * ld, V, blank, lam, use_boost, cur, sc.bm, sc.sv, sc.si, lane);
    }
    if (lane == 0) {
      // R7 bookkeeping (decoding.py:371-392)
      st.am[r] = am0 + static_cast<double>(d.lp);
      int64_t tn = tr;
      if (d.blank) {
        tn = tr + (dur > 1 ? dur : 1);
        st.k[r] = 0;
        emit[r] = 0;
        feed[r] = st.last[r];
      } else {
        const int64_t n = n0;
        if (n < st.lmax) {
          st.tokens[r * st.lmax + n] = d.chosen;
          st.deltas[r * st.lmax + n] = d.delta;
          st.states[r * st.lmax + n] = d.next;
        }
        st.n[r] = n + 1;
        st.boost[r] = bo0 + d.delta;
        st.tree[r] = d.next;
        if (st.tree_off && use_boost) st.tree_off[r] = d.noff;
        const int64_t k = k0 + 1;
        if (dur > 0) {  // TDT: the emission also consumes dur frames
          tn = tr + dur;
          st.k[r] = 0;
        } else if (k >= st.cap) {  // symbol cap: next frame, no blank score
          tn = tr + 1;
          st.k[r] = 0;
        } else {
          st.k[r] = k;
        }
        st.last[r] = d.chosen;
        emit[r] = 1;
        feed[r] = d.chosen;
      }
      st.t[r] = tn;
      if (tn < len) atomicOr(any_active, 1);
    }
  }
}

using StepFn = void (*)(TableView, int, const float *, int64_t, int64_t, int, const int32_t *, const uint8_t *, int,
                        double, int32_t *, float *, double *, int32_t *, uint8_t *);
using LoopFn = void (*)(TableView, int, const float *, int64_t, int64_t, int, int, double, pgpb_label_loop_state,
                        uint8_t *, int64_t *, int32_t *, const __nv_bfloat16 *, int64_t);

// NC = float4 chunks per lane for the register top-M (V <= 1024, 16-byte
// rows); 0 selects the generic path.
static int step_nc(int V, int64_t ld, const float *lp) {
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(lp) % 16) == 0;
  const int nc = (V + 127) / 128;
  return (vec && nc <= 8) ? nc : 0;
}

static StepFn step_fn(int nc) {
  static const StepFn f[9] = {greedy_step_kernel<0>, greedy_step_kernel<1>, greedy_step_kernel<2>,
                              greedy_step_kernel<3>, greedy_step_kernel<4>, greedy_step_kernel<5>,
                              greedy_step_kernel<6>, greedy_step_kernel<7>, greedy_step_kernel<8>};
  return f[nc];
}

static LoopFn loop_fn(int nc) {
  static const LoopFn f[9] = {label_loop_kernel<0>, label_loop_kernel<1>, label_loop_kernel<2>,
                              label_loop_kernel<3>, label_loop_kernel<4>, label_loop_kernel<5>,
                              label_loop_kernel<6>, label_loop_kernel<7>, label_loop_kernel<8>};
  return f[nc];
}

static size_t step_smem(int V) { return size_t(kWarpsPerBlock) * 256 + size_t(kWarpsPerBlock) * ((V + 31) >> 5) * 4; }

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

namespace pgpb {
// eos bump's final part (decoding.py:546-552): final_score[s] on final
// states (clo_rec.w = is_final), 0 elsewhere.
__global__ void final_bonus_kernel(TableView t, float *__restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < t.num_states) out[s] = __ldg(&t.clo_rec[s].w) ? __ldg(t.final_score + s) : 0.0f;
}
__global__ void backoff_total_kernel(TableView t, float *__restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < t.num_states) out[s] = __int_as_float(__ldg(&t.clo_rec[s].z));
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
  const size_t smem = step_smem(V);
  const int nc = step_nc(V, ld, d_lp);
  StepFn fn = step_fn(nc);
  int rc = prep_kernel(fn, smem);
  if (rc) return rc;
  const unsigned grid = static_cast<unsigned>((R + kWarpsPerBlock - 1) / kWarpsPerBlock);
  fn<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(t, use_boost ? 1 : 0, d_lp, ld, R, V, d_states,
                                                                  d_active, blank, lam, d_chosen, d_lp_chosen,
                                                                  d_delta, d_next, d_is_blank);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

static int label_loop_launch(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t R, int32_t V,
                             int32_t blank, double lam, int32_t use_boost, const pgpb_label_loop_state *state,
                             uint8_t *d_emit, int64_t *d_feed, int32_t *d_any_active, const void *d_logits,
                             int64_t ld_logits, void *stream);

int pgpb_label_loop_step(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t R, int32_t V, int32_t blank,
                         double lam, int32_t use_boost, const pgpb_label_loop_state *state, uint8_t *d_emit,
                         int64_t *d_feed, int32_t *d_any_active, void *stream) {
  return label_loop_launch(table, d_lp, ld, R, V, blank, lam, use_boost, state, d_emit, d_feed, d_any_active,
                           nullptr, 0, stream);
}

int pgpb_label_loop_step_logits(const pgpb_table *table, const void *d_logits_bf16, int64_t ld_logits,
                                float *d_lp_out, int64_t R, int32_t V, int32_t blank, double lam, int32_t use_boost,
                                const pgpb_label_loop_state *state, uint8_t *d_emit, int64_t *d_feed,
                                int32_t *d_any_active, void *stream) {
  using namespace pgpb;
  if (!d_logits_bf16 || !d_lp_out) return fail(PGPB_EINVAL, "NULL buffer");
  if (ld_logits < V) return fail(PGPB_EINVAL, "bad shape");
  return label_loop_launch(table, d_lp_out, V, R, V, blank, lam, use_boost, state, d_emit, d_feed, d_any_active,
                           d_logits_bf16, ld_logits, stream);
}

static int label_loop_launch(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t R, int32_t V,
                             int32_t blank, double lam, int32_t use_boost, const pgpb_label_loop_state *state,
                             uint8_t *d_emit, int64_t *d_feed, int32_t *d_any_active, const void *d_logits,
                             int64_t ld_logits, void *stream) {
  using namespace pgpb;
  if (R < 0 || V < 1 || ld < V || !state) return fail(PGPB_EINVAL, "bad shape");
  if (state->cap < 1) return fail(PGPB_EINVAL, "cap must be >= 1");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "step model vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (R == 0) return PGPB_OK;
  const TableView t = table ? table->view : empty_view(V);
  const size_t smem = step_smem(V);
  const int nc = step_nc(V, ld, d_lp);
  LoopFn fn = loop_fn(nc);
  int rc = prep_kernel(fn, smem);
  if (rc) return rc;
  // Warps per CTA: one row per warp is latency-bound, so spread the rows
  // over more SMs (fewer warps sharing an SM's schedulers) while the batch
  // is small next to the GPU.  pgpb_set_tuning("ll.warps") overrides.
  int wpb = kWarpsPerBlock;
  {
    const int64_t nsm = sm_count(current_device());
    if (tuning().ll_warps) {
      wpb = std::max(1, std::min(kWarpsPerBlock, tuning().ll_warps));
    } else {
      while (wpb > 2 && (R + wpb / 2 - 1) / (wpb / 2) <= nsm) wpb /= 2;
    }
  }
  const unsigned grid = static_cast<unsigned>((R + wpb - 1) / wpb);
  fn<<<grid, 32 * wpb, smem, static_cast<cudaStream_t>(stream)>>>(
      t, use_boost ? 1 : 0, d_lp, ld, R, V, blank, lam, *state, d_emit, d_feed, d_any_active,
      static_cast<const __nv_bfloat16 *>(d_logits), ld_logits);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_final_bonus(const pgpb_table *table, float *d_out, void *stream) {
  using namespace pgpb;
  if (!table || !d_out) return fail(PGPB_EINVAL, "NULL argument");
  const TableView &t = table->view;
  final_bonus_kernel<<<unsigned((t.num_states + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(t, d_out);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

int pgpb_backoff_total(const pgpb_table *table, float *d_out, void *stream) {
  using namespace pgpb;
  if (!table || !d_out) return fail(PGPB_EINVAL, "NULL argument");
  const TableView &t = table->view;
  backoff_total_kernel<<<unsigned((t.num_states + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(t, d_out);
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
