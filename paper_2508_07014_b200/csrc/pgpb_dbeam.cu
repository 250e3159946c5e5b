// Device-resident batched beam search: transducer waves (pgpb_tbeam_wave)
// and AED label-synchronous steps (pgpb_aed_step).
//
// Reference: transducer_beam_boosted (decoding.py:428-495, R9),
// aed_beam_boosted (decoding.py:502-587, R10), _keep_better / _rank_key
// (decoding.py:396-411, R11).  The reference keeps hypotheses in Python
// dicts keyed by token tuples and loops over V per hypothesis; here one CTA
// per utterance does, per wave / step:
//   1. stage the beam (K slots) in shared memory;
//   2. (transducer) merge every slot's blank extension into the frame's
//      finished pool: a warp compares (length, hash) of the pool entries in
//      parallel and confirms a hash hit by walking both trace chains;
//   3. score every (slot, token) expansion — closure tokens exactly from the
//      flattened closure, all other tokens from the dense root row shifted by
//      the state's backoff total — with fp64 keys in the reference's order,
//      keeping a sorted per-thread top-K list, then K block-wide argmax
//      rounds;
//   4. resolve each winner's (score, next state), append its trace node and
//      write the new beam in place.
// Nothing of the [K, V] score matrix is materialised.

#include <string>

#include <cuda_bf16.h>

#include "pgpb_beam.cuh"

namespace pgpb {

constexpr uint8_t kValid = 1, kEnded = 2;

// Threads per CTA of the device-beam kernels: small lists (K <= 4) run 1024
// threads (4 candidates per thread at beam 4 x V 1024: the scan's fp64 key
// and list-insertion chains are latency-bound, so more warps per SM hide
// them); K = 8 runs 512 and larger lists 256 (register budget: 64 per thread
// at 1024 threads).
template <int K>
constexpr int db_threads() {
  return K <= 4 ? 1024 : (K <= 8 ? 512 : 256);
}
constexpr int kDbMaxWarps = 32;

#ifdef PGPB_TBEAM_PROFILE
// Debug build only: per-phase cycles of the transducer wave (CTA 0,
// thread 0 timeline, summed over launches), read by pgpb_debug_tbeam_profile.
__device__ unsigned long long g_tb_prof[16];
#define TB_MARK(i)                                                                  \
  do {                                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                      \
      const long long now_ = clock64();                                             \
      atomicAdd(&g_tb_prof[i], (unsigned long long)(now_ - tb_last));             \
      tb_last = now_;                                                               \
    }                                                                               \
  } while (0)
// the first expansion thread's timeline (thread 32)
#define TB_MARKW(i)                                                                 \
  do {                                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 32) {                                     \
      const long long now_ = clock64();                                             \
      atomicAdd(&g_tb_prof[i], (unsigned long long)(now_ - tb_lastw));            \
      tb_lastw = now_;                                                              \
    }                                                                               \
  } while (0)
#else
#define TB_MARK(i) \
  do {             \
  } while (0)
#define TB_MARKW(i) \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ uint64_t hash_push(uint64_t h, int v) {
  uint64_t x = h * 0x100000001B3ull + (uint64_t(uint32_t(v)) + 0x9E3779B97F4A7C15ull);
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ double rank_key(double am, double boost, double lam) {
  return __dadd_rn(am, __dmul_rn(lam, boost));
}

// Token sequences ending at trace nodes a and b (same utterance, same
// length) are equal?  Shared prefixes end the walk early (a == b).
__device__ bool same_tokens(const int32_t *parent, const int32_t *token, int a, int b) {
  while (a != b) {
    if (a < 0 || b < 0) return false;
    if (__ldcg(token + a) != __ldcg(token + b)) return false;
    a = __ldcg(parent + a);
    b = __ldcg(parent + b);
  }
  return true;
}

// Beam staged in shared memory.
struct SBeam {
  double am[kMaxTopK], boost[kMaxTopK], extra[kMaxTopK];
  uint64_t hash[kMaxTopK];
  int tree[kMaxTopK], last[kMaxTopK], node[kMaxTopK], len[kMaxTopK], flags[kMaxTopK];
};

__device__ __forceinline__ void stage_beam(const pgpb_beam_hyps &H, int64_t base, int beam, SBeam &s) {
  for (int h = threadIdx.x; h < beam; h += blockDim.x) {
    s.am[h] = H.am[base + h];
    s.boost[h] = H.boost[base + h];
    s.tree[h] = H.tree[base + h];
    s.last[h] = H.last[base + h];
    s.node[h] = H.node[base + h];
    s.len[h] = H.len[base + h];
    s.hash[h] = H.hash[base + h];
    s.flags[h] = H.flags[base + h];
    s.extra[h] = 0.0;
  }
}

// Per-thread candidate scan over the expandable slots: dense tokens from the
// root row shifted by the backoff total, closure tokens exactly.  `skip` is
// the token that is not an expansion (transducer blank), `special` a token
// scored with boost `extra[h]` instead of the tree (AED eos), -1 for none.
template <int K, bool kVec>
__device__ __forceinline__ void scan_candidates(const TableView &t, const float *root, const unsigned *bm,
                                                int bm_words, const float *lp, int64_t ld, int64_t row0, int V,
                                                const SBeam &s, const bool *expand, int beam, int skip, int special,
                                                double lam, bool use_boost, const int4 *s_rec, KCand (&list)[K],
                                                int t0 = 0, bool closure_pass = true) {
  const int tid = int(threadIdx.x) - t0, nt = int(blockDim.x) - t0;
  // candidate (h, v) of token v at log-prob x (per-slot values from shared memory)
  auto dense = [&](int h, int v, float x) {
    if (v == skip) return;
    const double am_h = s.am[h], boost_h = s.boost[h];
    double bv;
    if (v == special) {
      bv = __dadd_rn(boost_h, s.extra[h]);
    } else if (use_boost) {
      if ((bm[h * bm_words + (v >> 5)] >> (v & 31)) & 1u) return;
      bv = __dadd_rn(boost_h, static_cast<double>(__int_as_float(s_rec[h].z) + root[v]));
    } else {
      bv = boost_h;
    }
    const double amv = __dadd_rn(am_h, static_cast<double>(x));
    klist_insert<K>(list, kcand(rank_key(amv, bv, lam), amv, h * V + v));
  };
  if (kVec) {
    // work items (slot, float2 pair) spread over every thread (pairs, not
    // float4s: 2048 items over the 992 worker threads leave at most 6 tokens
    // on a thread instead of 8); up to four items' loads in flight before
    // any is scored
    const int V2 = V >> 1;
    const int n = beam * V2;
    for (int i0 = tid; i0 < n; i0 += 4 * nt) {
      float2 xs[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int it = i0 + g * nt, h = it / V2;
        // generic loads: the rows are global (caller's) or shared (fused log-softmax)
        if (it < n && expand[h]) xs[g] = reinterpret_cast<const float2 *>(lp + (row0 + h) * ld)[it - h * V2];
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int it = i0 + g * nt, h = it / V2, c = it - h * V2;
        if (it < n && expand[h]) {
          // the item's closure-bitmap bits, root pair and slot values read
          // once (dense() re-reads them per token)
          const int v0 = 2 * c;
          const double am_h = s.am[h], boost_h = s.boost[h];
          unsigned cb = 0u;
          float2 q = make_float2(0.f, 0.f);
          float acc = 0.0f;
          if (use_boost) {
            cb = (bm[h * bm_words + (v0 >> 5)] >> (v0 & 31)) & 0x3u;
            q = reinterpret_cast<const float2 *>(root)[c];
            acc = __int_as_float(s_rec[h].z);
          }
          auto one = [&](int k, float x, float r) {
            const int v = v0 + k;
            if (v == skip) return;
            double bv;
            if (v == special) {
              bv = __dadd_rn(boost_h, s.extra[h]);
            } else if (use_boost) {
              if ((cb >> k) & 1u) return;
              bv = __dadd_rn(boost_h, static_cast<double>(acc + r));
            } else {
              bv = boost_h;
            }
            const double amv = __dadd_rn(am_h, static_cast<double>(x));
            klist_insert<K>(list, kcand(rank_key(amv, bv, lam), amv, h * V + v));
          };
          one(0, xs[g].x, q.x);
          one(1, xs[g].y, q.y);
        }
      }
    }
  } else {
    for (int h = 0; h < beam; ++h) {
      if (!expand[h]) continue;
      const float *row = lp + (row0 + h) * ld;
      for (int v = tid; v < V; v += nt) dense(h, v, row[v]);
    }
  }
  // closure arcs of every expandable slot in one flattened pass (their
  // entry and log-prob loads in flight together instead of slot by slot;
  // s_rec[h] is zero for slots that do not expand)
  if (use_boost && closure_pass) {
    int total = 0;
    for (int h = 0; h < beam; ++h) total += s_rec[h].y;
    for (int idx = tid; idx < total; idx += nt) {
      int h = 0, off = idx;
      while (off >= s_rec[h].y) {
        off -= s_rec[h].y;
        ++h;
      }
      const int4 e = __ldg(t.clo + s_rec[h].x + off);
      if (e.x == skip || e.x == special) continue;
      const float x = lp[(row0 + h) * ld + e.x];
      const double amv = __dadd_rn(s.am[h], static_cast<double>(x));
      const double bv = __dadd_rn(s.boost[h], static_cast<double>(__int_as_float(e.z)));
      klist_insert<K>(list, kcand(rank_key(amv, bv, lam), amv, h * V + e.x));
    }
  }
}

// Block top-k in two levels: each warp pops its own top k from its lanes'
// lists with warp reductions, then warp 0 merges the warps' sorted k-lists head by head —
// two block barriers in total instead of two per round.
template <int K>
__device__ __forceinline__ void block_topk(KCand (&list)[K], int k, KCand *s_warp, int *s_win, double *s_key,
                                           double *s_am) {
  (void)s_warp;
  __shared__ KCand s_wl[kDbMaxWarps * kMaxTopK];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = 0; r < k; ++r) {
    const KCand best = kc_warp_best(list[0]);
    if (lane == 0) s_wl[wid * k + r] = best;
    if (best.cid != INT_MAX && list[0].cid == best.cid) klist_pop<K>(list);
  }
  __syncthreads();
  if (wid == 0) kmerge_warp_lists(s_wl, nw, k, lane, s_win, s_key, s_am);
  __syncthreads();
}

// Mark each expandable slot's closure tokens in its bitmap.
// Every slot's closure record is loaded at once into s_rec (reused by the
// candidate scan), then all slots' closure tokens in one flattened pass, so
// the marking costs two dependent round trips whatever the beam width.
// Barrier over the worker threads [t0, blockDim.x): the whole block when
// t0 == 0, else named barrier 1 (warp 0 is busy with the pool merge).
__device__ __forceinline__ void worker_sync(int t0) {
  if (t0 == 0)
    __syncthreads();
  else
    asm volatile("bar.sync 1, %0;" ::"r"(int(blockDim.x) - t0) : "memory");
}

__device__ __forceinline__ void mark_closures(const TableView &t, unsigned *bm, int bm_words, const SBeam &s,
                                              const bool *expand, int beam, int4 *s_rec, int t0 = 0) {
  const int tid = int(threadIdx.x) - t0, nt = int(blockDim.x) - t0;
  for (int i = tid; i < beam * bm_words; i += nt) bm[i] = 0u;
  for (int h = tid; h < beam; h += nt) s_rec[h] = expand[h] ? __ldg(t.clo_rec + s.tree[h]) : make_int4(0, 0, 0, 0);
  worker_sync(t0);
  int total = 0;
  for (int h = 0; h < beam; ++h) total += s_rec[h].y;
  for (int idx = tid; idx < total; idx += nt) {
    int h = 0, off = idx;
    while (off >= s_rec[h].y) {
      off -= s_rec[h].y;
      ++h;
    }
    const int tok = __ldg(&t.clo[s_rec[h].x + off].x);
    atomicOr(bm + h * bm_words + (tok >> 5), 1u << (tok & 31));
  }
  worker_sync(t0);
}

// mark_closures fused with the closure candidates: each thread that loads
// a closure entry (token, next, score) sets its bitmap bit and scores it
// right away (the log-prob gather follows the entry load), so the entries
// are read once; scan_candidates then runs without its closure pass.
template <int K>
__device__ __forceinline__ void mark_and_score_closures(const TableView &t, unsigned *bm, int bm_words,
                                                        const SBeam &s, const bool *expand, int beam, int4 *s_rec,
                                                        const float *lp, int64_t ld, int64_t row0, int V, int skip,
                                                        int special, double lam, KCand (&list)[K], int t0 = 0) {
  const int tid = int(threadIdx.x) - t0, nt = int(blockDim.x) - t0;
  for (int i = tid; i < beam * bm_words; i += nt) bm[i] = 0u;
  for (int h = tid; h < beam; h += nt) s_rec[h] = expand[h] ? __ldg(t.clo_rec + s.tree[h]) : make_int4(0, 0, 0, 0);
  worker_sync(t0);
  int total = 0;
  for (int h = 0; h < beam; ++h) total += s_rec[h].y;
  for (int idx = tid; idx < total; idx += nt) {
    int h = 0, off = idx;
    while (off >= s_rec[h].y) {
      off -= s_rec[h].y;
      ++h;
    }
    const int4 e = __ldg(t.clo + s_rec[h].x + off);
    atomicOr(bm + h * bm_words + (e.x >> 5), 1u << (e.x & 31));
    if (e.x == skip || e.x == special) continue;
    const float x = lp[(row0 + h) * ld + e.x];
    const double amv = __dadd_rn(s.am[h], static_cast<double>(x));
    const double bv = __dadd_rn(s.boost[h], static_cast<double>(__int_as_float(e.z)));
    klist_insert<K>(list, kcand(rank_key(amv, bv, lam), amv, h * V + e.x));
  }
  worker_sync(t0);
}

// Advance blobs (TableView::adv_blob) of the expandable slots in shared
// memory: one cp.async copy per slot brings the closure words (the dense
// scan's exclusion bitmap), their ranks, the accumulator and the closure
// pairs, replacing the record -> entries -> bitmap-marking round trips.
__device__ __forceinline__ void db_cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

// Closure candidates of the expandable slots from their blobs: every set
// bit of a slot's closure words is a first-hit arc, its pair the rank-th.
template <int K>
__device__ __forceinline__ void blob_closure_candidates(const TableView &t, const int4 *blobs, const SBeam &s,
                                                        const bool *expand, int beam, const float *lp, int64_t ld,
                                                        int64_t row0, int V, int skip, int special, double lam,
                                                        KCand (&list)[K], int t0) {
  // items from the last worker thread down: the dense scan gives its extra
  // items to the first worker threads, so the two loads do not stack up
  const int nt = int(blockDim.x) - t0, tid = nt - 1 - (int(threadIdx.x) - t0);
  const int S16 = t.adv_stride16, Vw = t.bits_words, E0 = t.adv_ent0;
  for (int i = tid; i < beam * Vw; i += nt) {
    const int h = i / Vw, w = i - h * Vw;
    if (!expand[h]) continue;
    const int32_t *bl = reinterpret_cast<const int32_t *>(blobs + size_t(h) * S16);
    unsigned word = static_cast<unsigned>(bl[4 + w]);
    if (!word) continue;
    int q = reinterpret_cast<const uint16_t *>(bl + 4 + Vw)[w];
    const int2 *ent = reinterpret_cast<const int2 *>(bl + E0);
    while (word) {
      const int v = 32 * w + __ffs(word) - 1;
      word &= word - 1;
      const int2 e = ent[q++];
      if (v == skip || v == special) continue;
      const float x = lp[(row0 + h) * ld + v];
      const double amv = __dadd_rn(s.am[h], static_cast<double>(x));
      const double bv = __dadd_rn(s.boost[h], static_cast<double>(__int_as_float(e.y)));
      klist_insert<K>(list, kcand(rank_key(amv, bv, lam), amv, h * V + v));
    }
  }
}

// (score, next) of token v at a slot whose blob is in shared memory.
__device__ __forceinline__ void blob_resolve(const TableView &t, const int4 *blob, const float *root, int v, float &sc,
                                             int &nx) {
  const int32_t *bl = reinterpret_cast<const int32_t *>(blob);
  const int Vw = t.bits_words;
  const unsigned w = static_cast<unsigned>(bl[4 + (v >> 5)]);
  if ((w >> (v & 31)) & 1u) {
    const int q = reinterpret_cast<const uint16_t *>(bl + 4 + Vw)[v >> 5] + __popc(w & ((1u << (v & 31)) - 1u));
    const int2 e = reinterpret_cast<const int2 *>(bl + t.adv_ent0)[q];
    sc = __int_as_float(e.y);
    nx = e.x & 0x1FFFFFF;
  } else {
    sc = __int_as_float(bl[0]) + root[v];
    nx = __ldg(t.root_next + v);
  }
}

__device__ __forceinline__ void setup_root(const TableView &t, bool use_boost, int smem_root, unsigned char *smem,
                                           const float *&root, unsigned *&bm) {
  root = t.root_scores;
  size_t off = 0;
  if (use_boost && smem_root) {
    float *s_root = reinterpret_cast<float *>(smem);
    const int n4 = t.vocab_padded >> 2;
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      reinterpret_cast<float4 *>(s_root)[i] = __ldg(reinterpret_cast<const float4 *>(t.root_scores) + i);
    root = s_root;
    off = size_t(t.vocab_padded) * 4;
  }
  bm = reinterpret_cast<unsigned *>(smem + off);
}

// setup_root with the root row brought in by cp.async (the caller waits for
// its group before the barrier that precedes the first read), so no warp
// stalls on it.
__device__ __forceinline__ void setup_root_async(const TableView &t, bool use_boost, int smem_root,
                                                 unsigned char *smem, const float *&root, unsigned *&bm) {
  root = t.root_scores;
  size_t off = 0;
  if (use_boost && smem_root) {
    float *s_root = reinterpret_cast<float *>(smem);
    const int n4 = t.vocab_padded >> 2;
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      db_cp_async16(reinterpret_cast<float4 *>(s_root) + i, reinterpret_cast<const float4 *>(t.root_scores) + i);
    root = s_root;
    off = size_t(t.vocab_padded) * 4;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  bm = reinterpret_cast<unsigned *>(smem + off);
}

// ---------------------------------------------------------------------------
// Transducer wave

struct TBeamArgs {
  TableView t;
  const float *lp;
  int64_t ld;
  int V;
  int blank;
  double lam;
  int use_boost;
  int wave;
  int smem_root;
  pgpb_tbeam_state s;
  // fused joint tail (pgpb_tbeam_wave_fused): the slots' bf16 logits are
  // log-softmaxed here (rows kept in shared memory, written to lp as the
  // record of what was decided on), and the next wave's joint hidden rows
  // z = relu(enc_proj[b, t] + pred_j[last]) are written at the end
  const __nv_bfloat16 *logits;
  int64_t ld_logits;
  const __nv_bfloat16 *enc;
  int64_t enc_ld_b;
  int J;
  const __nv_bfloat16 *pred_j;
  __nv_bfloat16 *z;
  int blob_off;  // byte offset of the slots' advance blobs in dynamic shared memory (0: none)
};

__device__ __forceinline__ void write_hyp(const pgpb_beam_hyps &H, int64_t i, double am, double boost, int tree,
                                          int last, int node, int len, uint64_t hash, uint8_t flags) {
  H.am[i] = am;
  H.boost[i] = boost;
  H.tree[i] = tree;
  H.last[i] = last;
  H.node[i] = node;
  H.len[i] = len;
  H.hash[i] = hash;
  H.flags[i] = flags;
}

// Fused epilogue: the next wave's joint hidden rows of utterance b's slots,
// z[b*K + k] = relu(bf16(enc_proj[b, min(t, len-1)] + pred_j[ctx_k])), ctx
// = the slot's last token (blank at the start), as beam_hidden_kernel.  The
// hypotheses and t were just written by this block (visible after the
// barrier; read through L2).
// tf: the frame the next wave reads (this kernel's S.t[b] after its update);
// s_ctx[k]: slot k's last token as this kernel wrote it, INT_MIN where it
// kept the stored one (read back from global)
__device__ __forceinline__ void tbeam_joint_hidden(const TBeamArgs &a, int b, int64_t hb, int beam, int tf,
                                                   const int *s_ctx) {
  __syncthreads();
  const pgpb_tbeam_state &S = a.s;
  const int len = S.lengths[b];
  const int lim = len > 0 ? len - 1 : 0;
  if (tf > lim) tf = lim;
  const int J = a.J;
  const __nv_bfloat16 *e = a.enc + int64_t(b) * a.enc_ld_b + int64_t(tf) * J;
  for (int i = threadIdx.x; i < beam * J; i += blockDim.x) {
    const int k = i / J, j = i - k * J;
    const int lst = s_ctx[k] != INT_MIN ? s_ctx[k] : __ldcg(S.hyps.last + hb + k);
    const int ctx = lst < 0 ? a.blank : lst;
    const float sv = __bfloat162float(__float2bfloat16_rn(__bfloat162float(e[j]) +
                                                          __bfloat162float(a.pred_j[int64_t(ctx) * J + j])));
    a.z[(hb + k) * J + j] = __float2bfloat16_rn(sv > 0.0f ? sv : 0.0f);
  }
}

// Fused log-softmax split: warps per row, values per warp.
constexpr int kLsParts = 7, kLsPart = 160;

template <int K, bool kVec>
__global__ void __launch_bounds__(db_threads<K>()) tbeam_wave_kernel(TBeamArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
#ifdef PGPB_TBEAM_PROFILE
  long long tb_last = clock64(), tb_lastw = tb_last;
#endif
  __shared__ SBeam s;
  __shared__ bool s_expand[kMaxTopK];
  __shared__ int4 s_rec[kMaxTopK];
  __shared__ KCand s_warp[kDbMaxWarps];
  __shared__ int s_win[kMaxTopK];
  __shared__ double s_key[kMaxTopK], s_am[kMaxTopK];
  __shared__ int s_node_base;
  __shared__ int s_ctx[kMaxTopK];
  const pgpb_tbeam_state &S = a.s;
  const int b = blockIdx.x;
  const int t = S.t[b];
  if (t >= S.lengths[b]) return;
  const TableView &tv = a.t;
  const int V = a.V, beam = S.beam;
  const bool use_boost = a.use_boost != 0;
  const int64_t hb = int64_t(b) * beam;
  const int64_t nb = int64_t(b) * S.trace.nmax;
  const int32_t *np = S.trace.parent + nb, *nt = S.trace.token + nb;
  const float *root;
  unsigned *bm;
  setup_root_async(tv, use_boost, a.smem_root, smem, root, bm);
  // the beam's slots staged by the last warp, off the log-softmax warps'
  // path (their global round trips overlap)
  const bool expand_wave = a.wave < S.cap;
  {
    const int w0 = int(blockDim.x) - 32;
    if (int(threadIdx.x) >= w0) {
      const int l = int(threadIdx.x) - w0;
      for (int h = l; h < beam; h += 32) {
        s.am[h] = S.hyps.am[hb + h];
        s.boost[h] = S.hyps.boost[hb + h];
        s.tree[h] = S.hyps.tree[hb + h];
        s.last[h] = S.hyps.last[hb + h];
        s.node[h] = S.hyps.node[hb + h];
        s.len[h] = S.hyps.len[hb + h];
        s.hash[h] = S.hyps.hash[hb + h];
        const uint8_t f = S.hyps.flags[hb + h];
        s.flags[h] = f;
        s.extra[h] = 0.0;
        s_expand[h] = expand_wave && (f & kValid);
      }
      if (l == 0) s_node_base = S.trace.count[b];
      if (use_boost && a.blob_off && expand_wave) {
        // the expandable slots' advance blobs, copied while warps 0.. run
        // the log-softmax; their headers give the closure records
        __syncwarp();
        int4 *bl = reinterpret_cast<int4 *>(smem + a.blob_off);
        const int S16 = tv.adv_stride16;
        for (int i = l; i < beam * S16; i += 32) {
          const int h = i / S16;
          if (s_expand[h]) db_cp_async16(bl + i, tv.adv_blob + int64_t(s.tree[h]) * S16 + (i - h * S16));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // waited for before the stage barrier
      }
    }
  }
  const bool staged_blobs = use_boost && a.blob_off && expand_wave;
  // log-prob rows of the beam slots: the caller's f32 rows, or (fused) the
  // slots' logits log-softmaxed into shared memory after the bitmaps with
  // torch's formula, (x - max) - log(sum exp(x - max)): 7 warps per row
  // (partial maxima and sums through shared memory, summed in part order)
  // for V <= 1120 and beams <= 4, else one warp per row in the order of
  // log_softmax_bf16_kernel.  Either way the rows are written to lp as the
  // record of what was decided on (the replay tests decode those rows).
  const float *LP = a.lp;
  int64_t LD = a.ld, R0 = hb;
  if (a.logits) {
    const int Vp4 = (V + 3) & ~3;
    float *lrows = reinterpret_cast<float *>(
        (reinterpret_cast<uintptr_t>(bm + size_t(beam) * ((V + 31) >> 5)) + 15) & ~uintptr_t(15));
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (V <= kLsParts * kLsPart && beam * kLsParts <= nw - 1) {
      // each row over kLsParts warps (kLsPart values each, 5 per lane):
      // partial maxima and sums through shared memory, summed in part
      // order; the last warp stays free for the slot staging
      __shared__ float s_pmax[kMaxTopK * kLsParts], s_psum[kMaxTopK * kLsParts];
      const int w = threadIdx.x >> 5, r = w / kLsParts, part = w - r * kLsParts;
      const bool mine = r < beam;
      float xv[kLsPart / 32];
      const __nv_bfloat16 *xr = a.logits + (hb + (mine ? r : 0)) * a.ld_logits;
      if (mine) {
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < kLsPart / 32; ++k) {
          const int v = part * kLsPart + 32 * k + lane;
          xv[k] = v < V ? __bfloat162float(xr[v]) : -INFINITY;
          m = fmaxf(m, xv[k]);
        }
        float mr;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
        if (lane == 0) s_pmax[w] = mr;
      }
      __syncthreads();
      float rmax = -INFINITY;
      if (mine) {
        for (int q = 0; q < kLsParts; ++q) rmax = fmaxf(rmax, s_pmax[r * kLsParts + q]);
        float sm = 0.0f;
#pragma unroll
        for (int k = 0; k < kLsPart / 32; ++k)
          if (part * kLsPart + 32 * k + lane < V) sm += expf(xv[k] - rmax);
#pragma unroll
        for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(kFull, sm, o);
        if (lane == 0) s_psum[w] = sm;
      }
      __syncthreads();
      if (mine) {
        float tot = 0.0f;
        for (int q = 0; q < kLsParts; ++q) tot += s_psum[r * kLsParts + q];
        const float ls = logf(tot);
        float *yr = lrows + size_t(r) * Vp4;
        float *gr = const_cast<float *>(a.lp) + (hb + r) * a.ld;
#pragma unroll
        for (int k = 0; k < kLsPart / 32; ++k) {
          const int v = part * kLsPart + 32 * k + lane;
          if (v < V) {
            const float y = (xv[k] - rmax) - ls;
            yr[v] = y;
            gr[v] = y;
          }
        }
      }
    } else
    for (int r = threadIdx.x >> 5; r < beam; r += nw) {
      const __nv_bfloat16 *xr = a.logits + (hb + r) * a.ld_logits;
      float *yr = lrows + size_t(r) * Vp4;
      float *gr = const_cast<float *>(a.lp) + (hb + r) * a.ld;
      if (V <= 1024) {
        // the row's 32 values per lane loaded once, all in flight together;
        // same per-lane order (v = lane + 32 k) and reductions as below
        float xv[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int v = lane + 32 * k;
          xv[k] = v < V ? __bfloat162float(xr[v]) : -INFINITY;
        }
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < 32; ++k) m = fmaxf(m, xv[k]);
        float mr;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
        float sm = 0.0f;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (lane + 32 * k < V) sm += expf(xv[k] - mr);
#pragma unroll
        for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(kFull, sm, o);
        const float ls = logf(sm);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int v = lane + 32 * k;
          if (v < V) {
            const float y = (xv[k] - mr) - ls;
            yr[v] = y;
            gr[v] = y;
          }
        }
        continue;
      }
      float m = -INFINITY;
      for (int v = lane; v < V; v += 32) m = fmaxf(m, __bfloat162float(xr[v]));
      float mr;
      asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(m));
      float sm = 0.0f;
      for (int v = lane; v < V; v += 32) sm += expf(__bfloat162float(xr[v]) - mr);
#pragma unroll
      for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(kFull, sm, o);
      const float ls = logf(sm);
      for (int v = lane; v < V; v += 32) {
        const float y = (__bfloat162float(xr[v]) - mr) - ls;
        yr[v] = y;
        gr[v] = y;
      }
    }
    LP = lrows;
    LD = Vp4;
    R0 = 0;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // the root row (and the staging warp's blobs)
  if (staged_blobs && int(threadIdx.x) >= int(blockDim.x) - 32) {
    __syncwarp();
    const int4 *bl = reinterpret_cast<const int4 *>(smem + a.blob_off);
    for (int h = int(threadIdx.x) - (int(blockDim.x) - 32); h < beam; h += 32) {
      const int32_t *hd = reinterpret_cast<const int32_t *>(bl + size_t(h) * tv.adv_stride16);
      s_rec[h] = s_expand[h] ? make_int4(0, hd[1], hd[0], 0) : make_int4(0, 0, 0, 0);
    }
  }
  __syncthreads();

  TB_MARK(0);
  // 1. blank extensions -> finished pool, in rank (slot) order (warp 0).
  // Pools of <= 32 entries live in the warp's registers (lane j = entry j,
  // loaded once), so each slot's merge is a ballot instead of a global round
  // trip; larger pools take the general loop below.
  if (threadIdx.x < 32 && S.pool_cap <= 32) {
    const int lane = threadIdx.x;
    const int64_t pb = int64_t(b) * S.pool_cap;
    int cnt = S.pool_count[b];
    int e_len = -1;
    uint64_t e_hash = 0;
    double e_am = 0.0, e_bo = 0.0;
    int e_node = -1;
    // every slot's blank log-prob in flight at once (lane h holds slot h's)
    const float blank_lp = lane < beam ? LP[(R0 + lane) * LD + a.blank] : 0.0f;
    if (lane < cnt) {
      e_len = S.pool.len[pb + lane];
      e_hash = S.pool.hash[pb + lane];
      e_am = S.pool.am[pb + lane];
      e_bo = S.pool.boost[pb + lane];
      e_node = S.pool.node[pb + lane];
    }
    for (int h = 0; h < beam; ++h) {
      const float blp = __shfl_sync(kFull, blank_lp, h);
      if (!(s.flags[h] & kValid)) continue;
      const double am_e = __dadd_rn(s.am[h], static_cast<double>(blp));
      const double bo_e = s.boost[h];
      bool eq = false;
      if (lane < cnt && e_len == s.len[h] && e_hash == s.hash[h]) eq = same_tokens(np, nt, e_node, s.node[h]);
      const unsigned m = __ballot_sync(kFull, eq);
      const int match = m ? __ffs(m) - 1 : -1;
      int dst = -1;
      if (match >= 0) {
        const double oa = __shfl_sync(kFull, e_am, match), ob = __shfl_sync(kFull, e_bo, match);
        const double ok = rank_key(oa, ob, a.lam);
        const double ck = rank_key(am_e, bo_e, a.lam);
        if (ck > ok || (ck == ok && am_e > oa)) dst = match;  // decoding.py:396-404
      } else if (cnt < S.pool_cap) {
        dst = cnt;
      }
      if (dst >= 0) {
        if (lane == dst) {
          e_len = s.len[h];
          e_hash = s.hash[h];
          e_am = am_e;
          e_bo = bo_e;
          e_node = s.node[h];
        }
        if (lane == 0)
          write_hyp(S.pool, pb + dst, am_e, bo_e, s.tree[h], s.last[h], s.node[h], s.len[h], s.hash[h], kValid);
      }
      if (match < 0 && cnt < S.pool_cap) ++cnt;
    }
    if (lane == 0) S.pool_count[b] = cnt;
  } else if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int64_t pb = int64_t(b) * S.pool_cap;
    int cnt = S.pool_count[b];
    for (int h = 0; h < beam; ++h) {
      if (!(s.flags[h] & kValid)) continue;
      const double am_e = __dadd_rn(s.am[h], static_cast<double>(LP[(R0 + h) * LD + a.blank]));
      const double bo_e = s.boost[h];
      int match = -1;
      for (int j0 = 0; j0 < cnt && match < 0; j0 += 32) {
        const int j = j0 + lane;
        bool eq = false;
        if (j < cnt && S.pool.len[pb + j] == s.len[h] && S.pool.hash[pb + j] == s.hash[h])
          eq = same_tokens(np, nt, S.pool.node[pb + j], s.node[h]);
        const unsigned m = __ballot_sync(kFull, eq);
        if (m) match = j0 + __ffs(m) - 1;
      }
      if (lane == 0) {
        int dst = -1;
        if (match >= 0) {
          const double oa = S.pool.am[pb + match];
          const double ok = rank_key(oa, S.pool.boost[pb + match], a.lam);
          const double ck = rank_key(am_e, bo_e, a.lam);
          if (ck > ok || (ck == ok && am_e > oa)) dst = match;  // decoding.py:396-404
        } else if (cnt < S.pool_cap) {
          dst = cnt;
        }
        if (dst >= 0)
          write_hyp(S.pool, pb + dst, am_e, bo_e, s.tree[h], s.last[h], s.node[h], s.len[h], s.hash[h], kValid);
      }
      if (match < 0 && cnt < S.pool_cap) ++cnt;
      __syncwarp();
    }
    if (lane == 0) S.pool_count[b] = cnt;
  }

  TB_MARK(1);
  if (expand_wave) {
    // 2. top-beam non-blank expansions -> next wave, on warps 1.. while warp
    // 0 merges the blank extensions (independent work; they meet at the
    // top-k barrier)
    const int bm_words = (V + 31) >> 5;
    const int t0 = blockDim.x > 32 ? 32 : 0;
    KCand list[K];
#pragma unroll
    for (int i = 0; i < K; ++i) list[i] = kcand_none();
    int4 *blobs = (use_boost && a.blob_off) ? reinterpret_cast<int4 *>(smem + a.blob_off) : nullptr;
    if (int(threadIdx.x) >= t0) {
      if (blobs) {
        TB_MARKW(7);
        TB_MARKW(8);  // blobs and their records staged before the block barrier
        blob_closure_candidates<K>(tv, blobs, s, s_expand, beam, LP, LD, R0, V, a.blank, -1, a.lam, list, t0);
        TB_MARK(2);
        TB_MARKW(9);
        // the blobs' closure words are the dense scan's exclusion bitmaps
        scan_candidates<K, kVec>(tv, root, reinterpret_cast<const unsigned *>(blobs) + 4, tv.adv_stride16 * 4, LP,
                                 LD, R0, V, s, s_expand, beam, a.blank, -1, a.lam, use_boost, s_rec, list, t0, false);
        TB_MARKW(10);
      } else {
        if (use_boost)
          mark_and_score_closures<K>(tv, bm, bm_words, s, s_expand, beam, s_rec, LP, LD, R0, V, a.blank, -1, a.lam,
                                     list, t0);
        TB_MARK(2);
        TB_MARKW(7);
        TB_MARKW(8);
        TB_MARKW(9);
        scan_candidates<K, kVec>(tv, root, bm, bm_words, LP, LD, R0, V, s, s_expand, beam, a.blank, -1, a.lam,
                                 use_boost, s_rec, list, t0, false);
        TB_MARKW(10);
      }
    }
    TB_MARK(3);
    block_topk<K>(list, beam, s_warp, s_win, s_key, s_am);
    TB_MARK(4);
    TB_MARKW(11);
    for (int r = threadIdx.x; r < beam; r += blockDim.x) {
      const int cid = s_win[r];
      const int64_t o = hb + r;
      s_ctx[r] = INT_MIN;
      if (cid == INT_MAX) {
        S.hyps.flags[o] = 0;
        continue;
      }
      const int h = cid / V, v = cid % V;
      float sc = 0.0f;
      int nx = 0;
      if (blobs)
        blob_resolve(tv, blobs + size_t(h) * tv.adv_stride16, root, v, sc, nx);
      else if (use_boost)
        resolve_ranked(tv, root, bm + h * ((V + 31) >> 5), s_rec[h], v, sc, nx);
      const int node = s_node_base + r;  // winners fill slots 0.. contiguously
      if (node >= S.trace.nmax) {
        *S.trace.overflow = 1;
        S.hyps.flags[o] = 0;
        continue;
      }
      S.trace.parent[nb + node] = s.node[h];
      S.trace.token[nb + node] = v;
      S.trace.state[nb + node] = nx;
      S.trace.delta[nb + node] = static_cast<double>(sc);
      write_hyp(S.hyps, o, s_am[r], __dadd_rn(s.boost[h], static_cast<double>(sc)), nx, v, node, s.len[h] + 1,
                hash_push(s.hash[h], v), kValid);
      s_ctx[r] = v;
    }
    if (threadIdx.x == 0) {
      int n = 0;
      while (n < beam && s_win[n] != INT_MAX) ++n;
      const int64_t lim = S.trace.nmax;
      S.trace.count[b] = int(s_node_base + n < lim ? s_node_base + n : lim);
    }
    TB_MARK(5);
    if (a.z) tbeam_joint_hidden(a, b, hb, beam, t, s_ctx);
    return;
  }

  // 3. last wave: the pool's top-beam becomes the next frame's beam
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int64_t pb = int64_t(b) * S.pool_cap;
    const int cnt = S.pool_count[b];
    const bool final_frame = (t + 1 == S.lengths[b]);
    if (final_frame && S.rollback && use_boost) {
      for (int j = lane; j < cnt; j += 32) {
        const float accv = __int_as_float(__ldg(&tv.clo_rec[S.pool.tree[pb + j]].z));
        S.pool.boost[pb + j] = __dadd_rn(S.pool.boost[pb + j], static_cast<double>(accv));
      }
      __syncwarp();
    }
    unsigned long long taken = 0ull;  // entries lane + 32*i already selected
    for (int r = 0; r < beam; ++r) {
      double bk = -INFINITY, ba = -INFINITY;
      int bj = INT_MAX;
      for (int i = 0, j = lane; j < cnt; ++i, j += 32) {
        if ((taken >> i) & 1ull) continue;
        const double am = S.pool.am[pb + j];
        const double k = rank_key(am, S.pool.boost[pb + j], a.lam);
        if (k > bk || (k == bk && (am > ba || (am == ba && j < bj)))) {
          bk = k;
          ba = am;
          bj = j;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ok = __shfl_xor_sync(kFull, bk, o), oa = __shfl_xor_sync(kFull, ba, o);
        const int oj = __shfl_xor_sync(kFull, bj, o);
        if (ok > bk || (ok == bk && (oa > ba || (oa == ba && oj < bj)))) {
          bk = ok;
          ba = oa;
          bj = oj;
        }
      }
      if (bj != INT_MAX && (bj & 31) == lane) taken |= 1ull << (bj >> 5);
      if (lane == 0) {
        const int64_t o = hb + r;
        s_ctx[r] = INT_MIN;
        if (bj == INT_MAX) {
          S.hyps.flags[o] = 0;
        } else {
          const int64_t q = pb + bj;
          const int lq = S.pool.last[q];
          write_hyp(S.hyps, o, S.pool.am[q], S.pool.boost[q], S.pool.tree[q], lq, S.pool.node[q],
                    S.pool.len[q], S.pool.hash[q], kValid);
          s_ctx[r] = lq;
        }
      }
    }
    if (lane == 0) {
      S.pool_count[b] = 0;
      S.t[b] = t + 1;
    }
  }
  if (a.z) tbeam_joint_hidden(a, b, hb, beam, t + 1, s_ctx);
}

// ---------------------------------------------------------------------------
// AED step

struct AedArgs {
  TableView t;
  const float *lp;
  int64_t ld;
  int V;
  double lam;
  int use_boost;
  int smem_root;
  pgpb_aed_state s;
};

template <int K, bool kVec>
__global__ void __launch_bounds__(db_threads<K>()) aed_step_kernel(AedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SBeam s;
  __shared__ bool s_expand[kMaxTopK];
  __shared__ int4 s_rec[kMaxTopK];
  __shared__ KCand s_warp[kDbMaxWarps];
  __shared__ int s_win[kMaxTopK];
  __shared__ double s_key[kMaxTopK], s_am[kMaxTopK];
  __shared__ int s_node_base, s_any;
  const pgpb_aed_state &S = a.s;
  const int b = blockIdx.x;
  const TableView &tv = a.t;
  const int V = a.V, beam = S.beam, eos = S.eos;
  const bool use_boost = a.use_boost != 0;
  const int64_t hb = int64_t(b) * beam;
  const int64_t nb = int64_t(b) * S.trace.nmax;
  const float *root;
  unsigned *bm;
  setup_root(tv, use_boost, a.smem_root, smem, root, bm);
  stage_beam(S.hyps, hb, beam, s);
  if (threadIdx.x == 0) {
    s_node_base = S.trace.count[b];
    s_any = 0;
  }
  __syncthreads();
  for (int h = threadIdx.x; h < beam; h += blockDim.x) {
    const bool ex = (s.flags[h] & kValid) && !(s.flags[h] & kEnded) && s.len[h] < S.max_len;
    s_expand[h] = ex;
    if (ex) atomicOr(&s_any, 1);
    // eos bump (decoding.py:546-552): max(0, max_v srow) + final score
    double bump = 0.0;
    if (ex && use_boost && S.eos_bump) {
      const float best = __ldg(S.row_max + s.tree[h]);
      bump = best > 0.0f ? static_cast<double>(best) : 0.0;
      const int4 rec = __ldg(tv.clo_rec + s.tree[h]);
      if (rec.w) bump = __dadd_rn(bump, static_cast<double>(__ldg(tv.final_score + s.tree[h])));
    }
    if (ex && use_boost && S.rollback)  // extension: the unfinished phrase's credit goes back at eos
      bump = __dadd_rn(bump, static_cast<double>(__int_as_float(__ldg(&tv.clo_rec[s.tree[h]].z))));
    s.extra[h] = bump;
  }
  __syncthreads();
  if (!s_any) {  // nothing left to expand: the beam stays as it is
    for (int r = threadIdx.x; r < beam; r += blockDim.x) S.hyps.parent[hb + r] = r;
    return;
  }
  const int bm_words = (V + 31) >> 5;
  KCand list[K];
#pragma unroll
  for (int i = 0; i < K; ++i) list[i] = kcand_none();
  if (use_boost)
    mark_and_score_closures<K>(tv, bm, bm_words, s, s_expand, beam, s_rec, a.lp, a.ld, hb, V, -1, eos, a.lam, list);
  scan_candidates<K, kVec>(tv, root, bm, bm_words, a.lp, a.ld, hb, V, s, s_expand, beam, -1, eos, a.lam, use_boost,
                           s_rec, list, 0, false);
  // carried hypotheses (ended or at max_len), ranked unchanged
  for (int h = threadIdx.x; h < beam; h += blockDim.x)
    if ((s.flags[h] & kValid) && !s_expand[h])
      klist_insert<K>(list, kcand(rank_key(s.am[h], s.boost[h], a.lam), s.am[h], beam * V + h));
  block_topk<K>(list, beam, s_warp, s_win, s_key, s_am);
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  // Winners that create a trace node get consecutive node ids in rank order.
  for (int r = threadIdx.x; r < beam; r += blockDim.x) {
    const int cid = s_win[r];
    const int64_t o = hb + r;
    if (cid == INT_MAX) {
      S.hyps.flags[o] = 0;
      S.hyps.parent[o] = r;
      continue;
    }
    if (cid >= beam * V) {  // carried
      const int h = cid - beam * V;
      write_hyp(S.hyps, o, s.am[h], s.boost[h], s.tree[h], s.last[h], s.node[h], s.len[h], s.hash[h],
                static_cast<uint8_t>(s.flags[h]));
      S.hyps.parent[o] = h;
      continue;
    }
    int node = s_node_base;
    for (int q = 0; q < r; ++q) node += (s_win[q] != INT_MAX && s_win[q] < beam * V);
    const int h = cid / V, v = cid % V;
    S.hyps.parent[o] = h;
    if (node >= S.trace.nmax) {
      *S.trace.overflow = 1;
      S.hyps.flags[o] = 0;
      continue;
    }
    S.trace.parent[nb + node] = s.node[h];
    S.trace.token[nb + node] = v;
    if (v == eos) {  // ended, tokens / state / last unchanged; trace gets (eos, bump, state)
      S.trace.state[nb + node] = s.tree[h];
      S.trace.delta[nb + node] = s.extra[h];
      write_hyp(S.hyps, o, s_am[r], __dadd_rn(s.boost[h], s.extra[h]), s.tree[h], s.last[h], node, s.len[h],
                s.hash[h], kValid | kEnded);
    } else {
      float sc = 0.0f;
      int nx = 0;
      if (use_boost) resolve_ranked(tv, root, bm + h * bm_words, s_rec[h], v, sc, nx);
      S.trace.state[nb + node] = nx;
      S.trace.delta[nb + node] = static_cast<double>(sc);
      write_hyp(S.hyps, o, s_am[r], __dadd_rn(s.boost[h], static_cast<double>(sc)), nx, v, node, s.len[h] + 1,
                hash_push(s.hash[h], v), kValid);
      if (s.len[h] + 1 < S.max_len) atomicOr(&s_any, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int q = 0; q < beam; ++q) n += (s_win[q] != INT_MAX && s_win[q] < beam * V);
    const int64_t lim = S.trace.nmax;
    S.trace.count[b] = int(s_node_base + n < lim ? s_node_base + n : lim);
    if (s_any) atomicOr(S.any_active, 1);
  }
}

static size_t beam_smem(const TableView &t, bool use_boost, int beam, int &smem_root) {
  const size_t bm = use_boost ? size_t(beam) * size_t((t.vocab_size + 31) >> 5) * 4 : 0;
  const size_t root = size_t(t.vocab_padded) * 4;
  smem_root = (use_boost && root + bm <= size_t(kMaxSmemRootBytes)) ? 1 : 0;
  return bm + (smem_root ? root : 0);
}

template <int K, typename Fn, typename Args>
static int launch_beam(Fn fn, const Args &args, size_t smem, int64_t grid, cudaStream_t st) {
  // static + dynamic shared memory above 48 KB needs the opt-in; the kernels'
  // static part is ~27 KB, so opt in for any sizeable dynamic part (once per
  // size for each kernel)
  static thread_local size_t set_for[2] = {0, 0};
  static thread_local const void *fn_for[2] = {nullptr, nullptr};
  const void *f = reinterpret_cast<const void *>(fn);
  const int slot = fn_for[0] == f ? 0 : (fn_for[1] == f ? 1 : (fn_for[0] ? 1 : 0));
  if (smem > 16 * 1024 && (fn_for[slot] != f || set_for[slot] < smem)) {
    PGPB_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    fn_for[slot] = f;
    set_for[slot] = smem;
  }
  fn<<<static_cast<unsigned>(grid), db_threads<K>(), smem, st>>>(args);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

static int check_common(const pgpb_table *table, int64_t ld, int64_t batch, int V, int beam, int use_boost) {
  if (batch < 0 || V < 2 || ld < V) return fail(PGPB_EINVAL, "bad shape");
  if (beam < 1 || beam > kMaxTopK) return fail(PGPB_EINVAL, "beam must be in [1, 32]");
  if (int64_t(beam) * V + beam >= INT_MAX) return fail(PGPB_EINVAL, "beam * V too large");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  return PGPB_OK;
}

static TableView view_or_empty(const pgpb_table *table, int V) {
  TableView v{};
  if (table) return table->view;
  v.vocab_size = V;
  v.vocab_padded = (V + 3) & ~3;
  return v;
}

}  // namespace pgpb

extern "C" {

int pgpb_tbeam_wave(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t batch, int32_t V,
                    int32_t blank, double lam, int32_t use_boost, int32_t wave, const pgpb_tbeam_state *state,
                    void *stream) {
  using namespace pgpb;
  if (!state) return fail(PGPB_EINVAL, "NULL state");
  int rc = check_common(table, ld, batch, V, state->beam, use_boost);
  if (rc) return rc;
  if (blank < 0 || blank >= V) return fail(PGPB_EINVAL, "blank out of range");
  if (wave < 0 || wave > state->cap || state->cap < 1) return fail(PGPB_EINVAL, "bad wave index");
  if (state->pool_cap < state->beam * (state->cap + 1) || state->pool_cap > 64 * 32)
    return fail(PGPB_EINVAL, "pool_cap must be in [beam*(cap+1), 2048]");
  if (batch == 0) return PGPB_OK;
  TBeamArgs a{};
  a.t = view_or_empty(table, V);
  a.lp = d_lp;
  a.ld = ld;
  a.V = V;
  a.blank = blank;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.wave = wave;
  a.s = *state;
  size_t smem = beam_smem(a.t, use_boost, state->beam, a.smem_root);
  if (use_boost && a.t.adv_blob && tuning().beam_blobs != 1) {
    smem = (smem + 15) & ~size_t(15);
    a.blob_off = int(smem);
    smem += size_t(state->beam) * size_t(a.t.adv_stride16) * 16;
  }
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int k = state->beam;
#define PGPB_TB(KK) \
  return vec ? launch_beam<KK>(tbeam_wave_kernel<KK, true>, a, smem, batch, st) \
             : launch_beam<KK>(tbeam_wave_kernel<KK, false>, a, smem, batch, st)
  if (k <= 4) PGPB_TB(4);
  if (k <= 8) PGPB_TB(8);
  if (k <= 16) PGPB_TB(16);
  PGPB_TB(32);
#undef PGPB_TB
}

int pgpb_tbeam_wave_fused(const pgpb_table *table, const void *d_logits_bf16, int64_t ld_logits, float *d_lp_out,
                          int64_t ld, int64_t batch, int32_t V, int32_t blank, double lam, int32_t use_boost,
                          int32_t wave, const pgpb_tbeam_state *state, const void *d_enc_proj, int64_t enc_ld_b,
                          int32_t J, const void *d_pred_j, void *d_z_out, void *stream) {
  using namespace pgpb;
  if (!state || !d_logits_bf16 || !d_lp_out || !d_enc_proj || !d_pred_j || !d_z_out)
    return fail(PGPB_EINVAL, "NULL argument");
  int rc = check_common(table, ld, batch, V, state->beam, use_boost);
  if (rc) return rc;
  if (ld_logits < V || J < 1 || enc_ld_b < J) return fail(PGPB_EINVAL, "bad shape");
  if (blank < 0 || blank >= V) return fail(PGPB_EINVAL, "blank out of range");
  if (wave < 0 || wave > state->cap || state->cap < 1) return fail(PGPB_EINVAL, "bad wave index");
  if (state->pool_cap < state->beam * (state->cap + 1) || state->pool_cap > 64 * 32)
    return fail(PGPB_EINVAL, "pool_cap must be in [beam*(cap+1), 2048]");
  if (batch == 0) return PGPB_OK;
  TBeamArgs a{};
  a.t = view_or_empty(table, V);
  a.lp = d_lp_out;
  a.ld = ld;
  a.V = V;
  a.blank = blank;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.wave = wave;
  a.s = *state;
  a.logits = static_cast<const __nv_bfloat16 *>(d_logits_bf16);
  a.ld_logits = ld_logits;
  a.enc = static_cast<const __nv_bfloat16 *>(d_enc_proj);
  a.enc_ld_b = enc_ld_b;
  a.J = J;
  a.pred_j = static_cast<const __nv_bfloat16 *>(d_pred_j);
  a.z = static_cast<__nv_bfloat16 *>(d_z_out);
  // shared memory: root row | bitmaps (always, the rows follow them) | rows
  int smem_root = 0;
  beam_smem(a.t, use_boost, state->beam, smem_root);
  a.smem_root = smem_root;
  const size_t bm_bytes = size_t(state->beam) * size_t((V + 31) >> 5) * 4;
  size_t smem = (smem_root ? size_t(a.t.vocab_padded) * 4 : 0) + bm_bytes + 16 +
                size_t(state->beam) * size_t((V + 3) & ~3) * 4;
  if (use_boost && a.t.adv_blob && tuning().beam_blobs != 1) {
    smem = (smem + 15) & ~size_t(15);
    a.blob_off = int(smem);
    smem += size_t(state->beam) * size_t(a.t.adv_stride16) * 16;
  }
  if (smem > 200 * 1024) return fail(PGPB_EINVAL, "beam x vocabulary too large for the fused wave");
  const bool vec = (V % 4) == 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int k = state->beam;
#define PGPB_TB(KK) \
  return vec ? launch_beam<KK>(tbeam_wave_kernel<KK, true>, a, smem, batch, st) \
             : launch_beam<KK>(tbeam_wave_kernel<KK, false>, a, smem, batch, st)
  if (k <= 4) PGPB_TB(4);
  if (k <= 8) PGPB_TB(8);
  if (k <= 16) PGPB_TB(16);
  PGPB_TB(32);
#undef PGPB_TB
}

int pgpb_aed_step(const pgpb_table *table, const float *d_lp, int64_t ld, int64_t batch, int32_t V, double lam,
                  int32_t use_boost, const pgpb_aed_state *state, void *stream) {
  using namespace pgpb;
  if (!state) return fail(PGPB_EINVAL, "NULL state");
  int rc = check_common(table, ld, batch, V, state->beam, use_boost);
  if (rc) return rc;
  if (state->eos < 0 || state->eos >= V) return fail(PGPB_EINVAL, "eos out of range");
  if (state->max_len < 1) return fail(PGPB_EINVAL, "max_len must be >= 1");
  if (use_boost && state->eos_bump && !state->row_max) return fail(PGPB_EINVAL, "row_max required for the eos bump");
  if (batch == 0) return PGPB_OK;
  AedArgs a{};
  a.t = view_or_empty(table, V);
  a.lp = d_lp;
  a.ld = ld;
  a.V = V;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.s = *state;
  const size_t smem = beam_smem(a.t, use_boost, state->beam, a.smem_root);
  const bool vec = (V % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int k = state->beam;
#define PGPB_AE(KK) \
  return vec ? launch_beam<KK>(aed_step_kernel<KK, true>, a, smem, batch, st) \
             : launch_beam<KK>(aed_step_kernel<KK, false>, a, smem, batch, st)
  if (k <= 4) PGPB_AE(4);
  if (k <= 8) PGPB_AE(8);
  if (k <= 16) PGPB_AE(16);
  PGPB_AE(32);
#undef PGPB_AE
}

#ifdef PGPB_TBEAM_PROFILE
int pgpb_debug_tbeam_profile(unsigned long long *h_out, int reset) {
  cudaMemcpyFromSymbol(h_out, pgpb::g_tb_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(pgpb::g_tb_prof, z, sizeof(z));
  }
  return 0;
}
#endif

}  // extern "C"
