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
// decoding.py:407-411.  One warp per utterance: the state's closure tokens
// are marked in a per-warp shared bitmap, dense tokens are scored from the
// root row shifted by the state's backoff total, closure tokens exactly;
// the winner's (score, next) ride along the warp reduction.  The [B, V]
// score matrix is never written.

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

namespace {

constexpr int kAgWarps = 4;

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

template <bool kVec>
__global__ void __launch_bounds__(32 * kAgWarps) aed_greedy_kernel(AgArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int V = a.V, Vw = (V + 31) >> 5;
  unsigned *bm = reinterpret_cast<unsigned *>(smem) + size_t(wib) * Vw;
  const int64_t b = int64_t(blockIdx.x) * kAgWarps + wib;
  if (b >= a.B) return;
  const pgpb_aed_greedy_state &S = a.s;
  const int pos = S.len[b];
  if (S.ended[b] || pos >= S.max_len) return;
  const TableView &t = a.t;
  const bool boost = a.use_boost != 0;
  const int eos = S.eos;
  const int st = S.tree[b];
  const double am0 = S.am[b], bo0 = S.boost[b];
  const float *row = a.lp + b * a.ld;
  int4 rec = make_int4(0, 0, 0, 0);
  if (boost) {
    rec = __ldg(t.clo_rec + st);
    for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
    __syncwarp();
    for (int i = lane; i < rec.y; i += 32) {
      const int tok = __ldg(&t.clo[rec.x + i].x);
      atomicOr(bm + (tok >> 5), 1u << (tok & 31));
    }
    __syncwarp();
  }
  const float acc = __int_as_float(rec.z);
  AgCand best{-INFINITY, -INFINITY, INT_MAX, 0.0f, 0};
  auto consider = [&](int v, float x, float s, int nx) {
    const double amv = __dadd_rn(am0, static_cast<double>(x));
    const double bv = __dadd_rn(bo0, boost ? static_cast<double>(s) : 0.0);
    const AgCand c{__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, v, s, nx};
    if (ag_better(c, best)) best = c;
  };
  auto dense = [&](int v, float x) {
    if (v == eos) return;
    if (boost) {
      if ((bm[v >> 5] >> (v & 31)) & 1u) return;
      consider(v, x, acc + __ldg(t.root_scores + v), __ldg(t.root_next + v));
    } else {
      consider(v, x, 0.0f, 0);
    }
  };
  if (kVec) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    for (int i = lane; i < (V >> 2); i += 32) {
      const float4 x = __ldg(r4 + i);
      dense(4 * i, x.x);
      dense(4 * i + 1, x.y);
      dense(4 * i + 2, x.z);
      dense(4 * i + 3, x.w);
    }
  } else {
    for (int v = lane; v < V; v += 32) dense(v, __ldg(row + v));
  }
  if (boost) {
    for (int i = lane; i < rec.y; i += 32) {
      const int4 e = __ldg(t.clo + rec.x + i);
      if (e.x == eos) continue;
      consider(e.x, __ldg(row + e.x), __int_as_float(e.z), e.y);
    }
  }
  // eos candidate (lane 0): the bump is a double sum of two f32 values
  if (lane == 0) {
    double bump = 0.0;
    if (boost && S.row_max) {
      const float m = __ldg(S.row_max + st);
      bump = m > 0.0f ? static_cast<double>(m) : 0.0;
      bump = __dadd_rn(bump, static_cast<double>(__ldg(S.final_bonus + st)));
    }
    const double amv = __dadd_rn(am0, static_cast<double>(__ldg(row + eos)));
    const double bv = __dadd_rn(bo0, bump);
    const AgCand c{__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, -1, 0.0f, st};
    if (ag_better(c, best)) best = c;
  }
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
  if (lane != 0) return;
  const int64_t tb = b * int64_t(S.max_len + 1);
  if (best.id == -1) {
    double bump = 0.0;
    if (boost && S.row_max) {
      const float m = __ldg(S.row_max + st);
      bump = m > 0.0f ? static_cast<double>(m) : 0.0;
      bump = __dadd_rn(bump, static_cast<double>(__ldg(S.final_bonus + st)));
    }
    S.am[b] = best.am;
    S.boost[b] = __dadd_rn(bo0, bump);
    S.ended[b] = 1;
    S.deltas[tb + pos] = bump;
    S.states[tb + pos] = st;
    S.feed[b] = eos;
    return;
  }
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
  const size_t smem = size_t(kAgWarps) * size_t((V + 31) >> 5) * 4;
  if (smem > 200 * 1024) return fail(PGPB_EINVAL, "vocabulary too large");
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  auto fn = vec ? aed_greedy_kernel<true> : aed_greedy_kernel<false>;
  if (smem > 48 * 1024)
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned grid = unsigned((B + kAgWarps - 1) / kAgWarps);
  fn<<<grid, 32 * kAgWarps, smem, static_cast<cudaStream_t>(stream)>>>(a);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}
