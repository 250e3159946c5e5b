// Fused beam expansion + per-utterance top-k (pgpb_beam_topk).
//
// Replaces the V-wide Python loops of the reference's beam decoders
// (decoding.py:294-321 CTC prefix beam, :473-489 transducer beam,
// :544-583 AED beam).  One CTA per utterance (group of hypotheses):
//   1. each hypothesis' flattened closure tokens are marked in a per-hyp
//      shared-memory bitmap (the explicit first-hit arcs of its chain);
//   2. threads stream the log-prob rows with 16-byte loads and score every
//      (h, v) candidate — dense tokens from the shared-memory root row
//      shifted by the state's backoff total, closure tokens from the closure
//      — keeping a register-resident sorted top-K list per thread;
//   3. k rounds of block-wide argmax merge the per-thread lists, in passes
//      of up to 32 winners (each pass rescans below the previous pass's
//      last winner, so any k is exact);
//   4. the winners' tree score / next state are resolved (binary search in
//      the sorted closure) and written out.
// Never materialises the [H,V] score matrix.  All score arithmetic is fp64,
// unfused, in the reference's operation order.

#include <string>

#include "pgpb_beam.cuh"

namespace pgpb {

struct BeamArgs {
  TableView t;
  const float *lp;
  int64_t ld;
  int64_t hyps;
  int V;
  int group;
  int k;
  const int32_t *states;
  const double *am;
  const double *boost;
  const int32_t *exclude;
  const int32_t *alt_token;
  const double *alt_am;
  const uint8_t *valid;
  double lam;
  int use_boost;
  int skip_neg_inf;
  int smem_root;
  int32_t *out_hyp;
  int32_t *out_token;
  double *out_am;
  double *out_boost;
  int32_t *out_next;
  float *out_delta;
};


template <int K, bool kVec>
__global__ void __launch_bounds__(kBeamThreads) beam_topk_kernel(BeamArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cand s_warp[kBeamThreads / 32];
  __shared__ int s_win[kMaxTopK];
  __shared__ double s_win_key[kMaxTopK];
  __shared__ double s_win_am[kMaxTopK];
  const TableView &t = a.t;
  const int V = a.V;
  const int bm_words = (V + 31) >> 5;
  const float *root = t.root_scores;
  const int32_t *rnext = t.root_next;
  size_t off = 0;
  if (a.use_boost && a.smem_root) {
    float *s_root = reinterpret_cast<float *>(smem);
    int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(t.vocab_padded) * 4);
    stage_root(t, s_root, s_next);
    root = s_root;
    rnext = s_next;
    off = size_t(t.vocab_padded) * 8;
  }
  unsigned *bm = reinterpret_cast<unsigned *>(smem + off);  // [group][bm_words]
  const int64_t g = blockIdx.x;
  const int64_t h0 = g * a.group;
  const int64_t rem = a.hyps - h0;
  const int nh = static_cast<int>(rem < a.group ? rem : a.group);
  if (a.use_boost) {
    for (int i = threadIdx.x; i < nh * bm_words; i += blockDim.x) bm[i] = 0u;
    __syncthreads();
    for (int hl = 0; hl < nh; ++hl) {
      const int64_t h = h0 + hl;
      if (a.valid && !a.valid[h]) continue;
      const int4 rec = __ldg(t.clo_rec + a.states[h]);
      for (int i = threadIdx.x; i < rec.y; i += blockDim.x) {
        const int tok = __ldg(&t.clo[rec.x + i].x);
        atomicOr(bm + hl * bm_words + (tok >> 5), 1u << (tok & 31));
      }
    }
  }
  __syncthreads();

  // Top-k in passes of up to 32 winners: pass p keeps, per thread, the best
  // K candidates strictly below the previous pass's last winner (`floor`;
  // the order (key, am, cid) is total, cid = hl * V + v unique), so the
  // passes enumerate the exact global order for any k.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = a.k;
  bool have_floor = false;
  Cand floor{INFINITY, INFINITY, -1};
  for (int p0 = 0; p0 < k; p0 += kMaxTopK) {
    const int rounds = min(kMaxTopK, k - p0);
    Cand list[K];
#pragma unroll
    for (int i = 0; i < K; ++i) list[i] = Cand{-INFINITY, -INFINITY, INT_MAX};

    for (int hl = 0; hl < nh; ++hl) {
      const int64_t h = h0 + hl;
      if (a.valid && !a.valid[h]) continue;
      const float *row = a.lp + h * a.ld;
      const double am_h = a.am[h], boost_h = a.boost[h];
      const int ex = a.exclude ? a.exclude[h] : -1;
      const int alt = a.alt_token ? a.alt_token[h] : -1;
      const double alt_am = a.alt_am ? a.alt_am[h] : 0.0;
      float acc = 0.0f;
      int4 rec = make_int4(0, 0, 0, 0);
      if (a.use_boost) {
        rec = __ldg(t.clo_rec + a.states[h]);
        acc = __int_as_float(rec.z);
      }
      const unsigned *hbm = bm + hl * bm_words;
      auto consider = [&](int v, float x, float s) {
        if (v == ex) return;
        const double base = (v == alt) ? alt_am : am_h;
        const double amv = __dadd_rn(base, static_cast<double>(x));
        if (a.skip_neg_inf && amv == -INFINITY) return;
        const double bv = __dadd_rn(boost_h, static_cast<double>(s));
        Cand c{__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, hl * V + v};
        if (have_floor && !cand_better(floor, c)) return;
        list_insert<K>(list, c);
      };
      if (kVec) {
        const float4 *row4 = reinterpret_cast<const float4 *>(row);
        for (int i = threadIdx.x; i < (V >> 2); i += blockDim.x) {
          const float4 x4 = __ldg(row4 + i);
          const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int v = 4 * i + j;
            if (a.use_boost) {
              if ((hbm[v >> 5] >> (v & 31)) & 1u) continue;
              consider(v, xs[j], acc + root[v]);
            } else {
              consider(v, xs[j], 0.0f);
            }
          }
        }
      } else {
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
          const float x = __ldg(row + v);
          if (a.use_boost) {
            if ((hbm[v >> 5] >> (v & 31)) & 1u) continue;
            consider(v, x, acc + root[v]);
          } else {
            consider(v, x, 0.0f);
          }
        }
      }
      if (a.use_boost) {
        for (int i = threadIdx.x; i < rec.y; i += blockDim.x) {
          const int4 e = __ldg(t.clo + rec.x + i);
          consider(e.x, __ldg(row + e.x), __int_as_float(e.z));
        }
      }
    }

    // Block merge: `rounds` rounds of argmax over the per-thread list heads.
    for (int r = 0; r < rounds; ++r) {
      const Cand best = cand_warp_best(list[0]);
      if (lane == 0) s_warp[wid] = best;
      __syncthreads();
      if (threadIdx.x == 0) {
        Cand b = s_warp[0];
        for (int w = 1; w < kBeamThreads / 32; ++w)
          if (cand_better(s_warp[w], b)) b = s_warp[w];
        s_win[r] = b.cid;
        s_win_key[r] = b.key;
        s_win_am[r] = b.am;
      }
      __syncthreads();
      if (s_win[r] != INT_MAX && list[0].cid == s_win[r]) list_pop<K>(list);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rounds; r += blockDim.x) {
      const int64_t o = g * k + p0 + r;
      const int cid = s_win[r];
      if (cid == INT_MAX) {
        a.out_hyp[o] = -1;
        a.out_token[o] = -1;
        a.out_am[o] = -INFINITY;
        a.out_boost[o] = 0.0;
        a.out_next[o] = 0;
        a.out_delta[o] = 0.0f;
        continue;
      }
      const int hl = cid / V, v = cid % V;
      const int64_t h = h0 + hl;
      float s = 0.0f;
      int nx = 0;
      if (a.use_boost) resolve_ranked(t, root, bm + hl * bm_words, __ldg(t.clo_rec + a.states[h]), v, s, nx);
      a.out_hyp[o] = static_cast<int32_t>(h);
      a.out_token[o] = v;
      a.out_am[o] = s_win_am[r];
      a.out_boost[o] = __dadd_rn(a.boost[h], static_cast<double>(s));
      a.out_next[o] = nx;
      a.out_delta[o] = s;
    }
    const int last = s_win[rounds - 1];
    floor = Cand{s_win_key[rounds - 1], s_win_am[rounds - 1], last};
    have_floor = true;
    __syncthreads();
    if (last == INT_MAX) {  // fewer candidates than k: the rest stay empty
      for (int r = p0 + rounds + threadIdx.x; r < k; r += blockDim.x) {
        const int64_t o = g * k + r;
        a.out_hyp[o] = -1;
        a.out_token[o] = -1;
        a.out_am[o] = -INFINITY;
        a.out_boost[o] = 0.0;
        a.out_next[o] = 0;
        a.out_delta[o] = 0.0f;
      }
      break;
    }
  }
}

template <int K>
static int launch_k(const BeamArgs &args, bool vec, size_t smem, int64_t groups, cudaStream_t st) {
  auto fn = vec ? beam_topk_kernel<K, true> : beam_topk_kernel<K, false>;
  if (smem > 48 * 1024) {
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  fn<<<static_cast<unsigned>(groups), kBeamThreads, smem, st>>>(args);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

}  // namespace pgpb

extern "C" int pgpb_beam_topk(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t hyps,
                              int32_t V, int32_t group, int32_t k, const int32_t *d_states,
                              const double *d_am, const double *d_boost, const int32_t *d_exclude,
                              const int32_t *d_alt_token, const double *d_alt_am,
                              const uint8_t *d_valid, double lam, int32_t use_boost,
                              int32_t skip_neg_inf, int32_t *d_out_hyp, int32_t *d_out_token,
                              double *d_out_am, double *d_out_boost, int32_t *d_out_next,
                              float *d_out_delta, void *stream) {
  using namespace pgpb;
  if (hyps < 0 || V < 1 || (ld != 0 && ld < V) || group < 1 || k < 1)
    return fail(PGPB_EINVAL, "bad shape");
  if (int64_t(group) * V >= INT_MAX) return fail(PGPB_EINVAL, "group * V too large");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (hyps == 0) return PGPB_OK;
  if (use_boost && !d_states) return fail(PGPB_EINVAL, "states required with use_boost");
  BeamArgs a{};
  a.t = table ? table->view : TableView{};
  if (!table) {
    a.t.vocab_size = V;
    a.t.vocab_padded = (V + 3) & ~3;
  }
  a.lp = d_lp;
  a.ld = ld;
  a.hyps = hyps;
  a.V = V;
  a.group = group;
  a.k = k;
  a.states = d_states;
  a.am = d_am;
  a.boost = d_boost;
  a.exclude = d_exclude;
  a.alt_token = d_alt_token;
  a.alt_am = d_alt_am;
  a.valid = d_valid;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.skip_neg_inf = skip_neg_inf ? 1 : 0;
  a.out_hyp = d_out_hyp;
  a.out_token = d_out_token;
  a.out_am = d_out_am;
  a.out_boost = d_out_boost;
  a.out_next = d_out_next;
  a.out_delta = d_out_delta;
  const size_t bm = use_boost ? size_t(group) * size_t((V + 31) >> 5) * 4 : 0;
  const size_t root = size_t((V + 3) & ~3) * 8;
  a.smem_root = (use_boost && root + bm <= size_t(kMaxSmemRootBytes)) ? 1 : 0;
  const size_t smem = bm + (a.smem_root ? root : 0);
  if (smem > 200 * 1024) return fail(PGPB_EINVAL, "group too large for shared-memory bitmaps");
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  const int64_t groups = (hyps + group - 1) / group;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k <= 4) return launch_k<4>(a, vec, smem, groups, st);
  if (k <= 8) return launch_k<8>(a, vec, smem, groups, st);
  if (k <= 16) return launch_k<16>(a, vec, smem, groups, st);
  return launch_k<32>(a, vec, smem, groups, st);
}
