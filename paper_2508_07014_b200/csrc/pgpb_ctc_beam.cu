// Batched boosted CTC prefix beam search, device resident (pgpb_ctc_beam).
//
// Reference: ctc_beam_boosted (decoding.py:232-343, R8), _logaddexp
// (:94-100).  One CTA per utterance runs every frame of the utterance in one
// launch; the beam (<= 32 prefixes) lives in shared memory.  Per frame:
//   1. the frame's log-prob row is staged in shared memory (the next frame's
//      row is prefetched into the other buffer while this one is decided);
//   2. every live prefix j finds its parent among the live prefixes
//      (length, prefix hash, confirmed on the trace chains) and computes its
//      carries: pb' = tot_j + lp[blank], pnb' = pnb_j + lp[last_j] (+) the
//      parent's extension mass — at most two terms, so the reference's
//      accumulation order does not matter;
//   3. every (prefix i, token v != blank) that does not land on a live prefix
//      is scored as a new prefix: am = (v == last_i ? pb_i : tot_i) + lp[v],
//      boost = boost_i + score(state_i, v) (closure tokens exactly from the
//      flattened closure, all others from the dense root row shifted by the
//      state's backoff total), key = am + lam * boost; per-thread top-K
//      lists plus the carried prefixes, then `beam` block-wide argmax rounds
//      (the reference's ranking: key, then am; exact ties between different
//      prefixes fall back to (slot, token) order — DESIGN.md §2);
//   4. winners become the next beam; new prefixes append a trace node
//      (TraceStep(v, delta, next), decoding.py:63-69).
// Scores: fp64 in the reference's operation order; logaddexp uses the
// device exp / log1p (within 1 ulp of the host's libm), so am values match
// the reference within ~1e-15 relative, boost and tree states exactly.

#include <string>

#include "pgpb_beam.cuh"

namespace pgpb {

namespace {

// Threads per CTA by list size (the per-thread top-K lists' registers):
// 1024 for K <= 4, 512 for K = 8, 256 beyond.
template <int K>
constexpr int cb_threads() {
  return K <= 4 ? 1024 : (K <= 8 ? 512 : 256);
}
constexpr int kCbMaxWarps = 32;

__device__ __forceinline__ double logaddexp(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double m = a > b ? a : b;
  return __dadd_rn(m, log1p(exp(-fabs(__dadd_rn(a, -b)))));
}

__device__ __forceinline__ uint64_t cb_hash_push(uint64_t h, int v) {
  uint64_t x = h * 0x100000001B3ull + (uint64_t(uint32_t(v)) + 0x9E3779B97F4A7C15ull);
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// Token sequences ending at trace nodes a and b (-1 = empty) are equal?
__device__ bool cb_same_tokens(const int32_t *parent, const int32_t *token, int a, int b) {
  while (a != b) {
    if (a < 0 || b < 0) return false;
    if (token[a] != token[b]) return false;
    a = parent[a];
    b = parent[b];
  }
  return true;
}

// One beam.  tot = logaddexp(pb, pnb), known when the slot is filled (the
// winner's am: a carried prefix's am is that very logaddexp, a new prefix
// has pb = -inf), so no frame recomputes it; pnode = the trace node the
// prefix's last token was appended to (its parent's node), so the parent
// search confirms the usual case without reading the trace.
struct Slots {
  double pb[kMaxTopK], pnb[kMaxTopK], tot[kMaxTopK], boost[kMaxTopK];
  uint64_t hash[kMaxTopK], phash[kMaxTopK];
  int tree[kMaxTopK], last[kMaxTopK], node[kMaxTopK], pnode[kMaxTopK], len[kMaxTopK];
};

struct CbArgs {
  TableView t;
  const float *lp;  // [B, T, V]
  int64_t B, T;
  int V;
  const int32_t *lengths;
  int blank;
  int beam;
  double lam;
  int use_boost;
  // trace (per utterance b: nodes b*nmax ..)
  int32_t *tr_parent, *tr_token, *tr_state;
  double *tr_delta;
  int64_t nmax;
  // final beams [B, beam]
  double *o_pb, *o_pnb, *o_boost;
  int32_t *o_node, *o_len, *o_tree;
  int32_t *o_count;
  int32_t *overflow;
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

#ifdef PGPB_CB_PROFILE
// Debug-only CTA-0 phase timeline (pgpb_debug_cb_profile): [i] cycles spent
// in phase i summed over frames (thread 0, measured after each barrier),
// [15] frames.
__device__ unsigned long long g_cb_prof[16];
#define CB_MARK(i)                                                      \
  do {                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                          \
      const long long n_ = clock64();                                   \
      g_cb_prof[i] += (unsigned long long)(n_ - t_mark);                \
      t_mark = n_;                                                      \
    }                                                                   \
  } while (0)
#else
#define CB_MARK(i) \
  do {             \
  } while (0)
#endif

template <int K, bool kVec>
__global__ void __launch_bounds__(cb_threads<K>()) ctc_beam_kernel(CbArgs a) {
#ifdef PGPB_CB_PROFILE
  long long t_mark = clock64();
#endif
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Slots sl[2];  // this frame's beam and the next (swapped by frame parity)
  __shared__ int s_par[kMaxTopK];
  __shared__ double s_cpb[kMaxTopK], s_cpnb[kMaxTopK], s_amj[kMaxTopK];
  // closure records of the live prefixes' states, double-buffered: the next
  // frame's are fetched (cp.async, own commit group) as soon as the winners'
  // states are known, and waited for only after the next frame's carries
  __shared__ __align__(16) int4 s_rec2[2][kMaxTopK];
  __shared__ KCand s_wl[kCbMaxWarps * kMaxTopK];
  __shared__ int s_win[kMaxTopK];
  __shared__ double s_key[kMaxTopK], s_am[kMaxTopK];
  const TableView &t = a.t;
  const int V = a.V, Vp = (V + 3) & ~3, Vw = (V + 31) >> 5, beam = a.beam;
  const bool boost = a.use_boost != 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // shared layout: row[2][Vp] f32 | root[Vp] f32 | rnext[Vp] i32 | bm[K][Vw] | ex[K][Vw]
  float *rows = reinterpret_cast<float *>(smem);
  float *root = rows + 2 * Vp;
  int32_t *rnext = reinterpret_cast<int32_t *>(root + Vp);
  unsigned *bm = reinterpret_cast<unsigned *>(rnext + Vp);
  unsigned *ex = bm + size_t(kMaxTopK) * Vw;
  if (boost) {
    for (int i = threadIdx.x; i < Vp; i += blockDim.x) {
      root[i] = __ldg(t.root_scores + i);
      rnext[i] = __ldg(t.root_next + i);
    }
  }
  for (int64_t b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int64_t Tb = a.lengths ? min(max(int64_t(__ldg(a.lengths + b)), int64_t(0)), a.T) : a.T;
    const int64_t nb = b * a.nmax;
    int32_t *np = a.tr_parent + nb, *nt = a.tr_token + nb;
    __syncthreads();
    if (threadIdx.x == 0) {
      sl[0].pb[0] = 0.0;
      sl[0].pnb[0] = -INFINITY;
      sl[0].tot[0] = 0.0;  // logaddexp(0, -inf)
      sl[0].boost[0] = 0.0;
      sl[0].hash[0] = 0ull;
      sl[0].phash[0] = 0ull;
      sl[0].tree[0] = 0;
      sl[0].last[0] = -1;
      sl[0].node[0] = -1;
      sl[0].pnode[0] = -1;
      sl[0].len[0] = 0;
    }
    // live prefixes and trace nodes used: block-uniform registers, every
    // thread counts the winners itself
    int n = 1, nodes = 0;
    // frame 0's row and the root's closure record
    const float *lpb = a.lp + b * a.T * int64_t(V);
    if (Tb > 0)
      for (int i = threadIdx.x; i < V; i += blockDim.x) rows[i] = __ldg(lpb + i);
    if (boost && threadIdx.x == 0) cp_async16(&s_rec2[0][0], t.clo_rec);
    asm volatile("cp.async.commit_group;" ::: "memory");
    __syncthreads();
    for (int64_t tf = 0; tf < Tb; ++tf) {
      Slots &cur = sl[tf & 1], &nxt = sl[(tf + 1) & 1];
      const float *row = rows + (tf & 1) * Vp;
      int4 *s_rec = s_rec2[tf & 1];
      // prefetch the next frame's row into the other buffer (consumed after
      // this frame's barriers)
      if (tf + 1 < Tb) {
        float *nrow = rows + ((tf + 1) & 1) * Vp;
        const float *src = lpb + (tf + 1) * int64_t(V);
        if (kVec) {  // asynchronous copies (cp.async): the loads overlap this frame's work
          for (int i = threadIdx.x; i < (V >> 2); i += blockDim.x) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(nrow + 4 * i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + 4 * i) : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        } else {
          for (int i = threadIdx.x; i < V; i += blockDim.x) nrow[i] = __ldg(src + i);
        }
      }
      // 2. parents, carries and the carried prefixes' am (one thread per
      // live prefix)
      if (threadIdx.x < n) {
        const int j = threadIdx.x;
        const double tot = cur.tot[j];
        int par = -1;
        if (cur.len[j] > 0) {
          const int pn = cur.pnode[j];
          for (int i = 0; i < n && par < 0; ++i)
            if (cur.len[i] == cur.len[j] - 1 && cur.hash[i] == cur.phash[j] &&
                (pn == cur.node[i] || cb_same_tokens(np, nt, pn, cur.node[i])))
              par = i;
        }
        s_par[j] = par;
        const double cpb = __dadd_rn(tot, static_cast<double>(row[a.blank]));
        s_cpb[j] = cpb;
        double pnb = -INFINITY;
        if (cur.len[j] > 0) pnb = logaddexp(pnb, __dadd_rn(cur.pnb[j], static_cast<double>(row[cur.last[j]])));
        if (par >= 0) {
          // the parent's iteration (decoding.py:303-321): v = last_j
          const int v = cur.last[j];
          const double contrib =
              __dadd_rn(v == cur.last[par] ? cur.pb[par] : cur.tot[par], static_cast<double>(row[v]));
          if (contrib != -INFINITY) pnb = logaddexp(pnb, contrib);
        }
        s_cpnb[j] = pnb;
        s_amj[j] = logaddexp(cpb, pnb);
      }
      // exclusion bitmaps (extensions landing on a live prefix) and
      // closure records
      for (int i = threadIdx.x; i < n * Vw; i += blockDim.x) ex[i] = 0u;
      if (boost)
        for (int i = threadIdx.x; i < n * Vw; i += blockDim.x) bm[i] = 0u;
      // this frame's closure records (issued last frame); the next row's
      // group, the newest when one was issued this frame, may pend
      if (kVec && tf + 1 < Tb)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      CB_MARK(0);
      if (threadIdx.x < n && s_par[threadIdx.x] >= 0) {
        const int v = cur.last[threadIdx.x];
        atomicOr(ex + s_par[threadIdx.x] * Vw + (v >> 5), 1u << (v & 31));
      }
      int total = 0;
      // the thread's first closure entry stays in registers for the
      // candidate pass (one load per entry when total <= blockDim.x)
      int4 my_e = make_int4(0, 0, 0, 0);
      int my_h = 0;
      if (boost) {
        for (int h = 0; h < n; ++h) total += s_rec[h].y;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
          int h = 0, off = idx;
          while (off >= s_rec[h].y) {
            off -= s_rec[h].y;
            ++h;
          }
          const int4 e = __ldg(t.clo + s_rec[h].x + off);
          atomicOr(bm + h * Vw + (e.x >> 5), 1u << (e.x & 31));
          if (idx == int(threadIdx.x)) {
            my_e = e;
            my_h = h;
          }
        }
      }
      __syncthreads();
      CB_MARK(1);
      // 3. new-prefix candidates
      KCand list[K];
#pragma unroll
      for (int i = 0; i < K; ++i) list[i] = kcand_none();
      {
        // candidate (h, v): per-prefix values from shared memory
        auto dense = [&](int h, int v, float x) {
          if (v == a.blank || ((ex[h * Vw + (v >> 5)] >> (v & 31)) & 1u)) return;
          double bv;
          if (boost) {
            if ((bm[h * Vw + (v >> 5)] >> (v & 31)) & 1u) return;
            bv = __dadd_rn(cur.boost[h], static_cast<double>(__int_as_float(s_rec[h].z) + root[v]));
          } else {
            bv = __dadd_rn(cur.boost[h], 0.0);
          }
          const double amv = __dadd_rn(v == cur.last[h] ? cur.pb[h] : cur.tot[h], static_cast<double>(x));
          if (amv == -INFINITY) return;
          klist_insert<K>(list, kcand(__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, h * V + v));
        };
        // work items (prefix, float4 chunk) spread over every thread; the
        // prefix's values, the exclusion / closure bitmap nibbles and the
        // root row's float4 are read once per item.  Float prefilter: each
        // candidate's key is first estimated in fp32 (|error| <= 2^-21 M,
        // M = the sum of the operands' magnitudes); a candidate whose estimate
        // is below the warp's beam-th largest lane maximum by more than
        // 2^-18 max M is strictly worse than `beam` candidates of its own
        // warp, so it cannot be a winner and skips the exact fp64 key and the
        // list insertion.  The survivors (a few per warp) are ranked exactly.
        if (kVec) {
          const int V4 = V >> 2, ni = n * V4;
          const float4 *r4 = reinterpret_cast<const float4 *>(row);
          const float4 *q4 = reinterpret_cast<const float4 *>(root);
          const float lamf = static_cast<float>(a.lam), alam = fabsf(lamf);
          for (int it0 = threadIdx.x - lane; it0 < ni; it0 += blockDim.x) {  // warp-uniform trip count
            const int it = it0 + lane;
            const bool valid = it < ni;
            const int h = valid ? it / V4 : 0, c = valid ? it - h * V4 : 0, v0 = 4 * c;
            const float4 x = r4[c];
            unsigned skip = valid ? (ex[h * Vw + (v0 >> 5)] >> (v0 & 31)) & 0xFu : 0xFu;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            float acc = 0.0f;
            if (boost) {
              skip |= (bm[h * Vw + (v0 >> 5)] >> (v0 & 31)) & 0xFu;
              q = q4[c];
              acc = __int_as_float(s_rec[h].z);
            }
            const double pbh = cur.pb[h], toth = cur.tot[h], bh = cur.boost[h];
            const int lasth = cur.last[h];
            const float pbf = static_cast<float>(pbh), totf = static_cast<float>(toth), bf = static_cast<float>(bh);
            float f[4], lmax = -INFINITY, mmax = 0.0f;
            auto est = [&](int k, float xv, float qv) {
              const int v = v0 + k;
              const float base = v == lasth ? pbf : totf, s = acc + qv;
              float fk = (base + xv) + lamf * (bf + s);
              const float mk = (fabsf(base) + fabsf(xv)) + alam * (fabsf(bf) + fabsf(s));
              if (((skip >> k) & 1u) || v == a.blank) fk = -INFINITY;
              f[k] = fk;
              lmax = fmaxf(lmax, fk);
              if (fk > -INFINITY) mmax = fmaxf(mmax, mk);
            };
            est(0, x.x, q.x);
            est(1, x.y, q.y);
            est(2, x.z, q.z);
            est(3, x.w, q.w);
            const float thr = warp_kth_max(lmax, beam);
            const float mw = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mmax)));
            const float cut = thr - mw * 0x1p-18f;
            auto one = [&](int k, float xv, float qv) {
              const int v = v0 + k;
              if (((skip >> k) & 1u) || v == a.blank || f[k] < cut) return;
              const double bv = __dadd_rn(bh, boost ? static_cast<double>(acc + qv) : 0.0);
              const double amv = __dadd_rn(v == lasth ? pbh : toth, static_cast<double>(xv));
              if (amv == -INFINITY) return;
              klist_insert<K>(list, kcand(__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, h * V + v));
            };
            one(0, x.x, q.x);
            one(1, x.y, q.y);
            one(2, x.z, q.z);
            one(3, x.w, q.w);
          }
        } else {
          for (int it = threadIdx.x; it < n * V; it += blockDim.x) {
            const int h = it / V, v = it - h * V;
            dense(h, v, row[v]);
          }
        }
      }
      CB_MARK(7);
      if (boost) {
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
          int h = my_h;
          int4 e = my_e;
          if (idx != int(threadIdx.x)) {
            int off = idx;
            h = 0;
            while (off >= s_rec[h].y) {
              off -= s_rec[h].y;
              ++h;
            }
            e = __ldg(t.clo + s_rec[h].x + off);
          }
          const int v = e.x;
          if (v == a.blank || ((ex[h * Vw + (v >> 5)] >> (v & 31)) & 1u)) continue;
          const double amv = __dadd_rn(v == cur.last[h] ? cur.pb[h] : cur.tot[h], static_cast<double>(row[v]));
          if (amv == -INFINITY) continue;
          const double bv = __dadd_rn(cur.boost[h], static_cast<double>(__int_as_float(e.z)));
          klist_insert<K>(list, kcand(__dadd_rn(amv, __dmul_rn(a.lam, bv)), amv, h * V + v));
        }
      }
      CB_MARK(8);
      // carried prefixes (cid past the extension range)
      if (threadIdx.x < n) {
        const int j = threadIdx.x;
        const double amj = s_amj[j];
        klist_insert<K>(list, kcand(__dadd_rn(amj, __dmul_rn(a.lam, cur.boost[j])), amj, kMaxTopK * V + j));
      }
      CB_MARK(2);
      // 4. top `beam` in two levels: each warp pops its own top from its
      // lanes' lists (shuffles only), then warp 0 merges the warps' lists
      for (int r = 0; r < beam; ++r) {
        const KCand best = kc_warp_best(list[0]);
        if (lane == 0) s_wl[wid * beam + r] = best;
        if (best.cid != INT_MAX && list[0].cid == best.cid) klist_pop<K>(list);
      }
      __syncthreads();
      CB_MARK(3);
      if (wid == 0) kmerge_warp_lists(s_wl, int(blockDim.x >> 5), beam, lane, s_win, s_key, s_am);
      __syncthreads();
      CB_MARK(4);
      // 5. the next beam
      if (threadIdx.x < beam) {
        const int r = threadIdx.x;
        const int cid = s_win[r];
        if (cid != INT_MAX) {
          if (cid >= kMaxTopK * V) {  // carried prefix
            const int j = cid - kMaxTopK * V;
            if (boost) cp_async16(&s_rec2[(tf + 1) & 1][r], t.clo_rec + cur.tree[j]);
            nxt.pb[r] = s_cpb[j];
            nxt.pnb[r] = s_cpnb[j];
            nxt.tot[r] = s_am[r];  // = logaddexp(pb, pnb) (the candidate's am)
            nxt.boost[r] = cur.boost[j];
            nxt.hash[r] = cur.hash[j];
            nxt.phash[r] = cur.phash[j];
            nxt.tree[r] = cur.tree[j];
            nxt.last[r] = cur.last[j];
            nxt.node[r] = cur.node[j];
            nxt.pnode[r] = cur.pnode[j];
            nxt.len[r] = cur.len[j];
          } else {
            const int h = cid / V, v = cid - h * V;
            float sc = 0.0f;
            int nx = 0;
            if (boost) {
              resolve_ranked(t, root, bm + h * Vw, s_rec[h], v, sc, nx);
              cp_async16(&s_rec2[(tf + 1) & 1][r], t.clo_rec + nx);
            }
            // trace node: winners of this frame take consecutive nodes in
            // rank order among the new prefixes
            int rank = 0;
            for (int q = 0; q < r; ++q) rank += s_win[q] != INT_MAX && s_win[q] < kMaxTopK * V;
            const int node = nodes + rank;
            if (node < a.nmax) {
              a.tr_parent[nb + node] = cur.node[h];
              a.tr_token[nb + node] = v;
              a.tr_state[nb + node] = nx;
              a.tr_delta[nb + node] = static_cast<double>(sc);
            } else {
              *a.overflow = 1;
            }
            nxt.pb[r] = -INFINITY;
            nxt.pnb[r] = s_am[r];
            nxt.tot[r] = s_am[r];  // logaddexp(-inf, pnb)
            nxt.boost[r] = __dadd_rn(cur.boost[h], static_cast<double>(sc));
            nxt.hash[r] = cb_hash_push(cur.hash[h], v);
            nxt.phash[r] = cur.hash[h];
            nxt.tree[r] = nx;
            nxt.last[r] = v;
            nxt.node[r] = node < a.nmax ? node : -1;
            nxt.pnode[r] = cur.node[h];
            nxt.len[r] = cur.len[h] + 1;
          }
        }
      }
      {  // every thread: the next beam's size and the trace nodes used
        int m = 0, e = 0;
        while (m < beam && s_win[m] != INT_MAX) {
          e += s_win[m] < kMaxTopK * V;
          ++m;
        }
        n = m;
        nodes += e;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // the next frame's records
      // the next row has landed (the records' group may still pend)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncthreads();
      CB_MARK(5);
#ifdef PGPB_CB_PROFILE
      if (blockIdx.x == 0 && threadIdx.x == 0) g_cb_prof[15] += 1;
      __syncthreads();  // one bare barrier, for scale
      CB_MARK(9);
#endif
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    // final beam (rank order)
    const Slots &cur = sl[Tb & 1];
    if (threadIdx.x < beam) {
      const int r = threadIdx.x;
      const int64_t o = b * beam + r;
      if (r < n) {
        a.o_pb[o] = cur.pb[r];
        a.o_pnb[o] = cur.pnb[r];
        a.o_boost[o] = cur.boost[r];
        a.o_node[o] = cur.node[r];
        a.o_len[o] = cur.len[r];
        a.o_tree[o] = cur.tree[r];
      }
    }
    if (threadIdx.x == 0) a.o_count[b] = n;
  }
}

}  // namespace

}  // namespace pgpb

#ifdef PGPB_CB_PROFILE
extern "C" int pgpb_debug_cb_profile(unsigned long long *out, int reset) {
  PGPB_CUDA_TRY(cudaMemcpyFromSymbol(out, pgpb::g_cb_prof, sizeof(pgpb::g_cb_prof)));
  if (reset) {
    unsigned long long z[16] = {};
    PGPB_CUDA_TRY(cudaMemcpyToSymbol(pgpb::g_cb_prof, z, sizeof(z)));
  }
  return PGPB_OK;
}
#endif

extern "C" int pgpb_ctc_beam(const pgpb_table *table, const float *d_lp, int64_t B, int64_t T, int32_t V,
                             const int32_t *d_lengths, int32_t blank, int32_t beam, double lam, int32_t use_boost,
                             const pgpb_ctc_beam_out *out, void *stream) {
  using namespace pgpb;
  if (!out) return fail(PGPB_EINVAL, "out is NULL");
  if (B < 0 || T < 0 || V < 1) return fail(PGPB_EINVAL, "bad shape");
  if (beam < 1 || beam > kMaxTopK) return fail(PGPB_EINVAL, "beam must be in [1, 32]");
  if (blank < 0 || blank >= V) return fail(PGPB_EINVAL, "blank out of range");
  if (use_boost && !table) return fail(PGPB_EINVAL, "use_boost requires a table");
  if (table && table->view.vocab_size != V)
    return fail(PGPB_EINVAL, "emission vocab size " + std::to_string(V) + " != table vocab size " +
                                 std::to_string(table->view.vocab_size));
  if (int64_t(kMaxTopK + 1) * V >= INT_MAX) return fail(PGPB_EINVAL, "vocabulary too large");
  if (out->trace_nmax < T * int64_t(beam) + 1) return fail(PGPB_EINVAL, "trace_nmax must be >= T * beam + 1");
  if (B == 0) return PGPB_OK;
  CbArgs a{};
  if (table) {
    a.t = table->view;
  } else {
    a.t.vocab_size = V;
    a.t.vocab_padded = (V + 3) & ~3;
  }
  a.lp = d_lp;
  a.B = B;
  a.T = T;
  a.V = V;
  a.lengths = d_lengths;
  a.blank = blank;
  a.beam = beam;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.tr_parent = out->trace_parent;
  a.tr_token = out->trace_token;
  a.tr_state = out->trace_state;
  a.tr_delta = out->trace_delta;
  a.nmax = out->trace_nmax;
  a.o_pb = out->pb;
  a.o_pnb = out->pnb;
  a.o_boost = out->boost;
  a.o_node = out->node;
  a.o_len = out->len;
  a.o_tree = out->tree;
  a.o_count = out->count;
  a.overflow = out->overflow;
  const int Vp = (V + 3) & ~3, Vw = (V + 31) >> 5;
  const size_t smem = size_t(Vp) * 4 * 4 + size_t(2) * kMaxTopK * Vw * 4;
  if (smem > 200 * 1024) return fail(PGPB_EINVAL, "vocabulary too large for the shared-memory rows");
  const bool vec = (V % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  using Fn = void (*)(CbArgs);
  Fn fn;
  if (beam <= 4) fn = vec ? ctc_beam_kernel<4, true> : ctc_beam_kernel<4, false>;
  else if (beam <= 8) fn = vec ? ctc_beam_kernel<8, true> : ctc_beam_kernel<8, false>;
  else if (beam <= 16) fn = vec ? ctc_beam_kernel<16, true> : ctc_beam_kernel<16, false>;
  else fn = vec ? ctc_beam_kernel<32, true> : ctc_beam_kernel<32, false>;
  PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
  const int64_t cap = int64_t(sm_count(current_device())) * 2;
  const unsigned grid = unsigned(B < cap ? B : cap);
  int threads = beam <= 4 ? cb_threads<4>() : (beam <= 8 ? cb_threads<8>() : cb_threads<16>());
  if (tuning().cb_threads >= 32 && tuning().cb_threads <= threads) threads = tuning().cb_threads & ~31;
  fn<<<grid, threads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}
