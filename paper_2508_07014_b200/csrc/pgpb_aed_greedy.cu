// Batched boosted greedy AED step (pgpb_aed_greedy_step).
//
// Reference: aed_beam_boosted (decoding.py:502-587, R10) at beam 1 — the
// paper's AED greedy row.  With one hypothesis the step
// keeps the best of
//   * the eos candidate: am + lp[eos], boost + bump, bump = max(0, max_v
//     score[s, v]) + final_score[s] if s is final (decoding.py:546-552);
//   * every token v != eos: am + lp[v], boost + score[s, v];
// ranked by key = am' + lam * boost' (fp64, two rounded ops), then am',
// then the token tuple (the eos candidate keeps the shorter tuple, so it
// wins exact ties; extensions tie-break by lower v) — _rank_key,
// decoding.py:407-411.  One CTA per utterance: the state's closure tokens
// are marked in a shared bitmap, dense tokens are scored from the root row
// shifted by the state's backoff total, closure tokens exactly; the
// winner's (score, next) ride along the warp and block reductions.  The
// [B, V] score matrix is never written.

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

namespace {

constexpr int kAgThreads = 256;

struct AgCand {
  double key, am;
  int id;      // -1 = eos, else token
  float s;     // tree score of the token
  int next;    // next tree state
};

__device__ __forceinline__ bool ag_better(const AgCand &a, const AgCand &b) {
  if (a.key != b.key) return a.key > b.key;
  if (a.am != b.am) return a.am > b.am;
  return a.id < b.id;
}

struct AgArgs {
  TableView t;
  const float *lp;
  int64_t ld;
  int64_t B;
  int V;
  double lam;
  int use_boost;
  pgpb_aed_greedy_state s;
};

__device__ __forceinline__ void ag_warp_best(AgCand &best) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    AgCand oc;
    oc.key = __shfl_xor_sync(kFull, best.key, o);
    oc.am = __shfl_xor_sync(kFull, best.am, o);
    oc.id = __shfl_xor_sync(kFull, best.id, o);
    oc.s = __shfl_xor_sync(kFull, best.s, o);
    oc.next = __shfl_xor_sync(kFull, best.next, o);
    if (ag_better(oc, best)) best = oc;
  }
}

// One CTA (kAgThreads) per utterance: the V tokens split over all threads
// (V=4096: 16 per thread, the root row read as float4 / int4 alongside the
// log-prob float4), closure tokens marked in a shared bitmap, then a warp
// and a block reduction of (key, am, id) that carries the winner's
// (score, next).
template <bool kVec>
__global__ void __launch_bounds__(kAgThreads) aed_greedy_kernel(AgArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ AgCand s_best[kAgThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int V = a.V, Vw = (V + 31) >> 5;
  unsigned *bm = reinterpret_cast<unsigned *>(smem);
  const pgpb_aed_greedy_state &S = a.s;
  const TableView &t = a.t;
  const bool boost = a.use_boost != 0;
  const int eos = S.eos;
  for (int64_t b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int pos = S.len[b];
    if (S.ended[b] || pos >= S.max_len) continue;  // uniform over the CTA
    const int st = S.tree[b];
    const double am0 = S.am[b], bo0 = S.boost[b];
    const float *row = a.lp + b * a.ld;
    int4 rec = make_int4(0, 0, 0, 0);
    __syncthreads();  // bm reuse across utterances
    if (boost) {
      rec = __ldg(t.clo_rec + st);
      for (int w = threadIdx.x; w < Vw; w += blockDim.x) bm[w] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < rec.y; i += blockDim.x) {
        const int tok = __ldg(&t.clo[rec.x + i].x);
        atomicOr(bm + (tok >> 5), 1u << (tok & 31));
      }
      __syncthreads();
    }
    const float acc = __int_as_float(rec.z);
    AgCand best{-INFINITY, -INFINITY, INT_MAX, 0.0f, 0};
    auto consider = [&](int v, float x, float s, int nx) {
      const double amv = __dadd_rn(am0, static_cast<double>(x));
      const double bv = __dadd_rn(bo0, boost ? static_cast<double>(s) : 0.0);
      const AgCand c{__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, v, s, nx};
      if (ag_better(c, best)) best = c;
    };
    auto dense = [&](int v, float x, float r, int rn) {
      if (v == eos) return;
      if (boost) {
        if ((bm[v >> 5] >> (v & 31)) & 1u) return;
        consider(v, x, acc + r, rn);
      } else {
        consider(v, x, 0.0f, 0);
      }
    };
    if (kVec) {
      const float4 *r4 = reinterpret_cast<const float4 *>(row);
      const float4 *s4 = reinterpret_cast<const float4 *>(t.root_scores);
      const int4 *n4 = reinterpret_cast<const int4 *>(t.root_next);
      for (int i = threadIdx.x; i < (V >> 2); i += blockDim.x) {
        const float4 x = __ldg(r4 + i);
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        int4 rn = make_int4(0, 0, 0, 0);
        if (boost) {
          r = __ldg(s4 + i);
          rn = __ldg(n4 + i);
        }
        dense(4 * i, x.x, r.x, rn.x);
        dense(4 * i + 1, x.y, r.y, rn.y);
        dense(4 * i + 2, x.z, r.z, rn.z);
        dense(4 * i + 3, x.w, r.w, rn.w);
      }
    } else {
      for (int v = threadIdx.x; v < V; v += blockDim.x)
        dense(v, __ldg(row + v), boost ? __ldg(t.root_scores + v) : 0.0f, boost ? __ldg(t.root_next + v) : 0);
    }
    if (boost) {
      for (int i = threadIdx.x; i < rec.y; i += blockDim.x) {
        const int4 e = __ldg(t.clo + rec.x + i);
        if (e.x == eos) continue;
        consider(e.x, __ldg(row + e.x), __int_as_float(e.z), e.y);
      }
    }
    // eos candidate: the bump is a double sum of two f32 values
    double bump = 0.0;
    if (boost && S.row_max) {
      const float m = __ldg(S.row_max + st);
      bump = m > 0.0f ? static_cast<double>(m) : 0.0;
      bump = __dadd_rn(bump, static_cast<double>(__ldg(S.final_bonus + st)));
    }
    if (boost && S.rollback)  // extension: the unfinished phrase's credit goes back at eos
      bump = __dadd_rn(bump, static_cast<double>(__int_as_float(__ldg(&t.clo_rec[st].z))));
    if (threadIdx.x == 0) {
      const double amv = __dadd_rn(am0, static_cast<double>(__ldg(row + eos)));
      const double bv = __dadd_rn(bo0, bump);
      const AgCand c{__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, -1, 0.0f, st};
      if (ag_better(c, best)) best = c;
    }
    ag_warp_best(best);
    if (lane == 0) s_best[wid] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < int(blockDim.x >> 5); ++w)
        if (ag_better(s_best[w], best)) best = s_best[w];
      const int64_t tb = b * int64_t(S.max_len + 1);
      if (best.id == -1) {
        S.am[b] = best.am;
        S.boost[b] = __dadd_rn(bo0, bump);
        S.ended[b] = 1;
        S.deltas[tb + pos] = bump;
        S.states[tb + pos] = st;
        S.feed[b] = eos;
      } else {
        const int v = best.id;
        S.am[b] = best.am;
        S.boost[b] = __dadd_rn(bo0, boost ? static_cast<double>(best.s) : 0.0);
        S.tree[b] = boost ? best.next : 0;
        S.tokens[b * int64_t(S.max_len) + pos] = v;
        S.deltas[tb + pos] = boost ? static_cast<double>(best.s) : 0.0;
        S.states[tb + pos] = boost ? best.next : 0;
        S.len[b] = pos + 1;
        S.feed[b] = v;
        if (pos + 1 < S.max_len) atomicExch(S.any_active, 1);
      }
    }
  }
}

}  // namespace

}  // namespace pgpb

extern "C" int pgpb_aed_greedy_step(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t B, int32_t V,
                                    double lam, int32_t use_boost, const pgpb_aed_greedy_state *state,
                                    void *stream) {
  using namespace pgpb;
  if (!state) return fail(PGPB_EINVAL, "state is NULL");
  if (B < 0 || V < 1 || ld < V) return fail(PGPB_EINVAL, "bad shape");
  if (state->eos < 0 || state->eos >= V) return fail(PGPB_EINVAL, "eos out of range");
  if (state->max_len < 1) return fail(PGPB_EINVAL, "max_len must be >= 1");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "step model vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (use_boost && state->row_max && !state->final_bonus)
    return fail(PGPB_EINVAL, "eos bump needs final_bonus with row_max");
  if (B == 0) return PGPB_OK;
  AgArgs a{};
  if (table) {
    a.t = table->view;
  } else {
    a.t.vocab_size = V;
    a.t.vocab_padded = (V + 3) & ~3;
  }
  a.lp = d_lp;
  a.ld = ld;
  a.B = B;
  a.V = V;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.s = *state;
  const size_t smem = size_t((V + 31) >> 5) * 4;
  if (smem > 200 * 1024) return fail(PGPB_EINVAL, "vocabulary too large");
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  auto fn = vec ? aed_greedy_kernel<true> : aed_greedy_kernel<false>;
  if (smem > 48 * 1024)
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t cap = int64_t(sm_count(current_device())) * 8;
  const unsigned grid = unsigned(B < cap ? B : cap);
  fn<<<grid, kAgThreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}
