// Batched fused greedy CTC with shallow-fusion boosting (pgpb_ctc_greedy).
//
// Reference: _kernels.ctc_greedy (_kernels.pyx:75-225) and
// ctc_greedy_boosted (decoding.py:156-229), R6 in SURVEY.md.  Two kernels:
//
//  Phase A  frame_topm_kernel — embarrassingly parallel over all (b, t)
//           frames, HBM-bound: one warp streams a log-prob row with 16-byte
//           loads and reduces it to its top-M tokens by (logprob desc, id
//           asc).  Entry 0 is the stage-1 argmax (first max).  M = 1 when
//           boosting is off.
//
//  Phase B  ctc_seq_kernel — one warp per utterance, sequential over its
//           frames, touching rows only at *emitting* frames (argmax neither
//           blank nor the previous symbol).  The boosted rerank there uses:
//             * the state's blob (header + flattened first-hit arcs, one
//               contiguous load; each arc carries its target's blob offset);
//             * the row prefetched into shared memory with cp.async while
//               the previous emitting frame was being decided;
//             * an exact pruning bound: closure tokens are scored exactly,
//               dense tokens only among the frame's top-M, and any dense
//               token outside the top-M scores at most
//                 fl(lp_M + fl(lam * fl32(acc + max_root)))
//               (every rounded op is monotone), so a winner strictly above
//               that bound is final; otherwise a full-row rescan decides.
//             * speculative L1 prefetch of every candidate's successor blob
//               during the reduction, so the next emission's state is warm.
//           The [B,V] score matrix is never written.
//
// Bit-exact with the reference per utterance: argmax first-max semantics,
// fp64 fusion lp + lam*s with two separately rounded ops, ties broken by
// higher raw logprob then lower token id.

#include <cstdlib>
#include <string>

#include "pgpb_rerank.cuh"

namespace pgpb {

// Production path (pgpb_ctc_spec.cu).
int ctc_spec_launch(const pgpb_table *table, const float *d_lp, int64_t B, int64_t T, int32_t V,
                     const int32_t *d_lengths, int32_t blank, double lam, int32_t use_boost, int32_t *d_tokens,
                     double *d_deltas, int32_t *d_states, int32_t *d_num_out, double *d_am, double *d_boost,
                     cudaStream_t st);

constexpr int kTopM = 4;

#ifdef PGPB_SEQ_PROFILE
// Debug-only phase timing of the sequential kernel (utterance 0, lane 0):
// accumulated cycles between checkpoints, read by pgpb_debug_seq_profile.
__device__ unsigned long long g_seq_prof[16];
#define SEQ_MARK(i)                                                        \
  do {                                                                     \
    if (b == 0 && lane == 0) {                                             \
      const long long _now = clock64();                                    \
      atomicAdd(&g_seq_prof[i], (unsigned long long)(_now - _prof_last));  \
      _prof_last = _now;                                                   \
    }                                                                      \
  } while (0)
#else
#define SEQ_MARK(i) \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// Phase A

// Register-resident variant for V <= 32 * 4 * NC (16-byte rows): the row
// stays in registers; top-M via a threshold: the M-th largest lane maximum
// bounds the row's M-th largest value from below, so only elements >= it
// (normally exactly M) are gathered into shared memory and ranked.  Falls
// back to the insertion network when ties produce more than 32 survivors.
template <int M, int NC>
__global__ void __launch_bounds__(kThreads)
    frame_topm_reg_kernel(const float *__restrict__ lp, int64_t B, int64_t T, int V,
                          const int32_t *__restrict__ lengths, int32_t *__restrict__ top_idx,
                          float *__restrict__ top_lp) {
  __shared__ float s_val[kWarpsPerBlock][32];
  __shared__ int s_idx[kWarpsPerBlock][32];
  __shared__ int s_cnt[kWarpsPerBlock];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int V4 = V >> 2;
  for (int64_t f = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < B * T; f += nwarps) {
    if (lengths) {
      const int64_t b = f / T;
      if (f - b * T >= __ldg(lengths + b)) continue;
    }
    const float4 *row4 = reinterpret_cast<const float4 *>(lp + f * V);
    float4 x[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      x[k] = c < V4 ? __ldcs(row4 + c) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
    // lane maximum (first index among equals)
    float lm = -INFINITY;
    int li = INT_MAX;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int v = 4 * (lane + 32 * k);
      if (argmax_better(x[k].x, v, lm, li)) { lm = x[k].x; li = v; }
      if (argmax_better(x[k].y, v + 1, lm, li)) { lm = x[k].y; li = v + 1; }
      if (argmax_better(x[k].z, v + 2, lm, li)) { lm = x[k].z; li = v + 2; }
      if (argmax_better(x[k].w, v + 3, lm, li)) { lm = x[k].w; li = v + 3; }
    }
    if (M == 1) {
      warp_argmax(lm, li);
      if (lane == 0) {
        top_idx[f] = li < V ? li : INT_MAX;
        top_lp[f] = lm;
      }
      continue;
    }
    // threshold = M-th largest lane maximum
    float thr = -INFINITY;
    {
      float v = lm;
      int id = li;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        float bx = v;
        int bi = id;
        warp_argmax(bx, bi);
        thr = bx;
        if (id == bi) {
          v = -INFINITY;
          id = INT_MAX;
        }
      }
    }
    // gather survivors >= thr
    if (lane == 0) s_cnt[wib] = 0;
    __syncwarp();
    int mine = 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) mine += (x[k].x >= thr) + (x[k].y >= thr) + (x[k].z >= thr) + (x[k].w >= thr);
    int pos = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, pos, o);
      if (lane >= o) pos += y;
    }
    const int total = __shfl_sync(kFull, pos, 31);
    pos -= mine;
    if (total <= 32) {
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int v = 4 * (lane + 32 * k);
        if (x[k].x >= thr) { s_val[wib][pos] = x[k].x; s_idx[wib][pos++] = v; }
        if (x[k].y >= thr) { s_val[wib][pos] = x[k].y; s_idx[wib][pos++] = v + 1; }
        if (x[k].z >= thr) { s_val[wib][pos] = x[k].z; s_idx[wib][pos++] = v + 2; }
        if (x[k].w >= thr) { s_val[wib][pos] = x[k].w; s_idx[wib][pos++] = v + 3; }
      }
      __syncwarp();
      float cv = lane < total ? s_val[wib][lane] : -INFINITY;
      int ci = lane < total ? s_idx[wib][lane] : INT_MAX;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        float bx = cv;
        int bi = ci;
        warp_argmax(bx, bi);
        if (ci == bi) {
          cv = -INFINITY;
          ci = INT_MAX;
        }
        if (lane == 0) {
          top_idx[f * M + r] = bi < V ? bi : INT_MAX;
          top_lp[f * M + r] = bx;
        }
      }
      __syncwarp();
    } else {  // heavy ties: insertion network over the registers
      float lv[M];
      int lix[M];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        lv[i] = -INFINITY;
        lix[i] = INT_MAX;
      }
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int v = 4 * (lane + 32 * k);
        if (v < V) {
          topm_insert<M>(lv, lix, x[k].x, v);
          topm_insert<M>(lv, lix, x[k].y, v + 1);
          topm_insert<M>(lv, lix, x[k].z, v + 2);
          topm_insert<M>(lv, lix, x[k].w, v + 3);
        }
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
        float bx = lv[0];
        int bi = lix[0];
        warp_argmax(bx, bi);
        if (lix[0] == bi && bi != INT_MAX) {
#pragma unroll
          for (int i = 0; i < M - 1; ++i) {
            lv[i] = lv[i + 1];
            lix[i] = lix[i + 1];
          }
          lv[M - 1] = -INFINITY;
          lix[M - 1] = INT_MAX;
        }
        if (lane == 0) {
          top_idx[f * M + r] = bi < V ? bi : INT_MAX;
          top_lp[f * M + r] = bx;
        }
      }
    }
  }
}

template <int M, bool kVec>
__global__ void __launch_bounds__(kThreads)
    frame_topm_kernel(const float *__restrict__ lp, int64_t B, int64_t T, int V,
                      const int32_t *__restrict__ lengths, int32_t *__restrict__ top_idx,
                      float *__restrict__ top_lp) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t F = B * T;
  for (int64_t f = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < F; f += nwarps) {
    if (lengths) {
      const int64_t b = f / T;
      if (f - b * T >= __ldg(lengths + b)) continue;
    }
    const float *row = lp + f * V;
    float lv[M];
    int li[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      lv[i] = -INFINITY;
      li[i] = INT_MAX;
    }
    if (kVec) {
      const float4 *row4 = reinterpret_cast<const float4 *>(row);
#pragma unroll 4
      for (int c = lane; c < (V >> 2); c += 32) {
        const float4 x = __ldcs(row4 + c);  // streamed once
        topm_insert<M>(lv, li, x.x, 4 * c);
        topm_insert<M>(lv, li, x.y, 4 * c + 1);
        topm_insert<M>(lv, li, x.z, 4 * c + 2);
        topm_insert<M>(lv, li, x.w, 4 * c + 3);
      }
    } else {
      for (int v = lane; v < V; v += 32) topm_insert<M>(lv, li, __ldcs(row + v), v);
    }
    // M rounds of warp argmax over the lanes' list heads.
#pragma unroll
    for (int r = 0; r < M; ++r) {
      float bx = lv[0];
      int bi = li[0];
      warp_argmax(bx, bi);
      if (li[0] == bi && bi != INT_MAX) {
#pragma unroll
        for (int i = 0; i < M - 1; ++i) {
          lv[i] = lv[i + 1];
          li[i] = li[i + 1];
        }
        lv[M - 1] = -INFINITY;
        li[M - 1] = INT_MAX;
      }
      if (lane == 0) {
        top_idx[f * M + r] = bi;
        top_lp[f * M + r] = bx;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Phase B helpers: L1 row prefetch (default) or a TMA bulk ring of shared
// buffers with one mbarrier per slot (PGPB_CTC_RING=P, experimental).

__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint32_t saddr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_row_g2s(float *dst, const float *src, uint32_t bytes, uint64_t *bar) {
  // (the slot's previous contents were consumed into registers before the
  // warp-converged issue point, so no proxy fence is needed for the WAR)
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
  }
}

// Ring of prefetched rows for one warp (all fields warp-uniform).
struct RowRing {
  float *buf;        // [P+1][Vp] (slot P = synchronous spare)
  uint64_t *bar;     // [P+1]
  int32_t *frame;    // [P] frame held by each slot
  int P, Vp;
  uint32_t phase;    // parity bit per slot
  int head, count;   // FIFO of in-flight / ready slots
  int64_t scan_pos;   // predictor: first frame not yet loaded into scan_mask
  int64_t scan_base;  // frame of bit 0 of scan_mask
  unsigned scan_mask; // predicted emitting frames of the current chunk not yet issued
  int scan_prev;      // stage-1 argmax of frame scan_pos - 1 (-1 before frame 0)
};

// Predicted emitting frames assume the boosted choice equals the stage-1
// argmax (the common case): frame f emits iff a[f] != blank and
// a[f] != a[f-1].  Fill the ring up to P in-flight rows.  The predictor
// keeps the candidate mask of its current 32-frame chunk in registers.
__device__ __forceinline__ void ring_refill(RowRing &r, const int32_t *ti, int M, int64_t Tb, int blank,
                                            const float *rows, int V, int lane) {
  while (r.count < r.P) {
    if (r.scan_mask == 0u) {  // load the next chunk of stage-1 argmaxes
      if (r.scan_pos >= Tb) break;
      const int64_t f = r.scan_pos + lane;
      const int af = f < Tb ? __ldg(ti + f * M) : blank;
      int prev = __shfl_up_sync(kFull, af, 1);
      if (lane == 0) prev = r.scan_prev;
      r.scan_mask = __ballot_sync(kFull, f < Tb && af != blank && af != prev);
      const int nvalid = int(Tb - r.scan_pos < 32 ? Tb - r.scan_pos : 32);
      r.scan_prev = __shfl_sync(kFull, af, nvalid - 1);
      r.scan_base = r.scan_pos;
      r.scan_pos += nvalid;
      continue;
    }
    const int k = __ffs(r.scan_mask) - 1;
    r.scan_mask &= r.scan_mask - 1;
    int slot = r.head + r.count;
    if (slot >= r.P) slot -= r.P;
    const int64_t fr = r.scan_base + k;
    if (lane == 0) {
      r.frame[slot] = static_cast<int32_t>(fr);
      bulk_row_g2s(r.buf + size_t(slot) * r.Vp, rows + fr * V, uint32_t(V) * 4, r.bar + slot);
    }
    ++r.count;
  }
  __syncwarp();
}

// Row of frame `tt` in shared memory: the ring head if predicted, otherwise a
// synchronous bulk load into the spare slot.  Stale (mispredicted) slots
// are retired on the way.
__device__ __forceinline__ const float *ring_get(RowRing &r, int64_t tt, const float *grow, int V, int lane) {
  while (r.count > 0) {
    const int h = r.head;
    const int fr = r.frame[h];
    if (fr > tt) break;
    mbar_wait(r.bar + h, (r.phase >> h) & 1u);
    r.phase ^= 1u << h;
    if (fr == tt) return r.buf + size_t(h) * r.Vp;  // popped by ring_pop
    if (++r.head == r.P) r.head = 0;
    --r.count;
  }
  if (lane == 0) bulk_row_g2s(r.buf + size_t(r.P) * r.Vp, grow, uint32_t(V) * 4, r.bar + r.P);
  mbar_wait(r.bar + r.P, (r.phase >> r.P) & 1u);
  r.phase ^= 1u << r.P;
  return r.buf + size_t(r.P) * r.Vp;
}

__device__ __forceinline__ void ring_pop_if(RowRing &r, int64_t tt) {
  if (r.count > 0 && r.frame[r.head] == tt) {
    __syncwarp();
    if (++r.head == r.P) r.head = 0;
    --r.count;
  }
}

struct SeqArgs {
  TableView t;
  const float *lp;
  int64_t B, T;
  int V;
  const int32_t *lengths;
  const int32_t *top_idx;  // [B,T,M]
  const float *top_lp;
  int M;
  int blank;
  double lam;
  int use_boost;
  int ring;  // P rows prefetched per warp (0: read rows from global memory)
  int32_t *tokens;
  double *deltas;
  int32_t *ostates;
  int32_t *nout;
  double *am_out;
  double *boost_out;
};

__global__ void __launch_bounds__(kThreads) ctc_seq_kernel(SeqArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const TableView &t = a.t;
  const int V = a.V, Vp = t.vocab_padded, Vw = (V + 31) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int P = a.ring;
  // shared: root scores | root next | root next blob offsets | per warp:
  //         [P+1] rows | [P+1] mbarriers | [P] frame ids | bitmap
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_rnext = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  int32_t *s_rnoff = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 8);
  const size_t base = (size_t(Vp) * 12 + 127) & ~size_t(127);
  const size_t rows_bytes = P ? size_t(P + 1) * Vp * 4 : 0;
  const size_t bm_bytes = (size_t(Vw) * 4 + 15) & ~size_t(15);
  const size_t per_warp = ((rows_bytes + size_t(P + 1) * 8 + size_t(P) * 4 + bm_bytes + 127) & ~size_t(127));
  unsigned char *wb = smem + base + size_t(wib) * per_warp;
  RowRing ring;
  ring.buf = reinterpret_cast<float *>(wb);
  ring.bar = reinterpret_cast<uint64_t *>(wb + rows_bytes);
  ring.frame = reinterpret_cast<int32_t *>(wb + rows_bytes + size_t(P + 1) * 8);
  unsigned *bm = reinterpret_cast<unsigned *>(wb + rows_bytes + size_t(P + 1) * 8 + size_t(P) * 4);
  ring.P = P;
  ring.Vp = Vp;
  ring.phase = 0;
  if (a.use_boost) {
    for (int i = threadIdx.x; i < Vp; i += blockDim.x) {
      s_root[i] = __ldg(t.root_scores + i);
      s_rnext[i] = __ldg(t.root_next + i);
      s_rnoff[i] = __ldg(t.root_next_off + i);
    }
    for (int i = lane; i < Vw; i += 32) bm[i] = 0u;
    if (P && lane == 0)
      for (int i = 0; i <= P; ++i) mbar_init(ring.bar + i);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int M = a.M;
  const float max_root = t.max_root_score;
  for (int64_t b = int64_t(blockIdx.x) * W + wib; b < a.B; b += int64_t(gridDim.x) * W) {
    const int64_t Tb = a.lengths ? int64_t(__ldg(a.lengths + b)) : a.T;
    const int32_t *ti = a.top_idx + b * a.T * M;
    const float *tl = a.top_lp + b * a.T * M;
    const float *urows = a.lp + b * a.T * V;
    double am = 0.0, boost = 0.0;
    int last = -1;
    BlobRegs cur;
    if (a.use_boost) cur = load_blob(t, __ldg(t.blob_off), lane);
    int64_t n = 0;
    ring.head = 0;
    ring.count = 0;
    ring.scan_pos = 0;
    ring.scan_base = 0;
    ring.scan_mask = 0u;
    ring.scan_prev = -1;
    const bool use_ring = a.use_boost && P > 0;
#ifdef PGPB_SEQ_PROFILE
    long long _prof_last = clock64();
#endif
    if (use_ring) ring_refill(ring, ti, M, Tb, a.blank, urows, V, lane);
    for (int64_t t0 = 0; t0 < Tb; t0 += 32) {
      const int cnt = int(Tb - t0 < 32 ? Tb - t0 : 32);
      const int ca = lane < cnt ? __ldg(ti + (t0 + lane) * M) : a.blank;
      const float cl = lane < cnt ? __ldg(tl + (t0 + lane) * M) : 0.0f;
      int ctv[kTopM];
      float ctx[kTopM];
      if (a.use_boost) {
#pragma unroll
        for (int j = 0; j < kTopM; ++j) {
          ctv[j] = lane < cnt ? __ldg(ti + (t0 + lane) * M + j) : INT_MAX;
          ctx[j] = lane < cnt ? __ldg(tl + (t0 + lane) * M + j) : -INFINITY;
        }
      }
      for (int i = 0; i < cnt; ++i) {
        const int av = __shfl_sync(kFull, ca, i);
        const float lp1 = __shfl_sync(kFull, cl, i);
        if (av == a.blank || av == last) {  // blank / repeat pass through (R6)
          am += static_cast<double>(lp1);
          last = av;
          continue;
        }
        const int64_t tt = t0 + i;
        SEQ_MARK(0);  // non-emitting frames since the last mark
        BCand w;
        if (!a.use_boost) {
          w.v = av;
          w.lp = lp1;
          w.s = 0.0f;
          w.nx = 0;
          w.noff = 0;
        } else {
          const float *grow = urows + tt * V;
          const float *row = use_ring ? ring_get(ring, tt, grow, V, lane) : grow;
          if (!use_ring) {
            // L1 prefetch of the next predicted emitting frame's row (frame j
            // emits iff its argmax is neither blank nor frame j-1's argmax,
            // assuming the argmax survives this rerank); one 128-byte line
            // per lane covers 4 KB
            const int prev = __shfl_up_sync(kFull, ca, 1);
            const unsigned m = __ballot_sync(kFull, lane > i && lane < cnt && ca != a.blank && ca != prev);
            if (m) {
              const float *nrow = urows + (t0 + __ffs(m) - 1) * V;
              for (int c = lane * 32; c < V; c += 32 * 32) prefetch_l1(nrow + c);
            }
          }
          SEQ_MARK(1);
          int tv[kTopM];
          float tx[kTopM];
#pragma unroll
          for (int j = 0; j < kTopM; ++j) {
            tv[j] = __shfl_sync(kFull, ctv[j], i);
            tx[j] = __shfl_sync(kFull, ctx[j], i);
          }
          // software pipelining: start loading the successor blob for the
          // stage-1 argmax (the usual winner) before the rerank runs
          const int count = __shfl_sync(kFull, cur.b0.x, 0);
          const int pred_off = blob_next_off(cur, count, s_rnoff, av, lane);
          const BlobRegs pred = load_blob(t, pred_off, lane);
          SEQ_MARK(2);
          w = blob_rerank_regs<kTopM>(t, cur, s_root, s_rnext, s_rnoff, bm, row, V, tv, tx, a.blank, last, a.lam,
                                      max_root, lane);
          SEQ_MARK(3);
          cur = (w.noff == pred_off) ? pred : load_blob(t, w.noff, lane);
          if (use_ring) {
            ring_pop_if(ring, tt);
            ring_refill(ring, ti, M, Tb, a.blank, urows, V, lane);
          }
          SEQ_MARK(4);
        }
        if (lane == 0) {
          a.tokens[b * a.T + n] = w.v;
          a.deltas[b * a.T + n] = static_cast<double>(w.s);
          a.ostates[b * a.T + n] = w.nx;
        }
        ++n;
        am += static_cast<double>(w.lp);
        boost += static_cast<double>(w.s);
        last = w.v;
        SEQ_MARK(5);
      }
    }
    if (use_ring) {  // drain rows still in flight before the slots are reused
      while (ring.count > 0) {
        const int h = ring.head;
        mbar_wait(ring.bar + h, (ring.phase >> h) & 1u);
        ring.phase ^= 1u << h;
        if (++ring.head == ring.P) ring.head = 0;
        --ring.count;
      }
      __syncwarp();
    }
    if (lane == 0) {
      a.nout[b] = static_cast<int32_t>(n);
      a.am_out[b] = am;
      a.boost_out[b] = boost;
    }
  }
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // The two-phase kernels below (parallel top-M + one warp per utterance)
  // stay reachable for A/B measurements: PGPB_CTC_TWOPHASE=1.
  const bool two_phase = getenv("PGPB_CTC_TWOPHASE") && atoi(getenv("PGPB_CTC_TWOPHASE")) != 0;
  if (!two_phase)
    return ctc_spec_launch(table, d_lp, B, T, V, d_lengths, blank, lam, use_boost, d_tokens, d_deltas, d_states,
                            d_num_out, d_am, d_boost, st);
  retain_pool(current_device());
  const int M = use_boost ? kTopM : 1;
  const int64_t F = B * (T > 0 ? T : 1);
  const size_t idx_bytes = ((size_t(F) * M * 4 + 255) / 256) * 256;
  char *ws = nullptr;
  PGPB_CUDA_TRY(cudaMallocAsync(&ws, 2 * idx_bytes, st));
  int32_t *top_idx = reinterpret_cast<int32_t *>(ws);
  float *top_lp = reinterpret_cast<float *>(ws + idx_bytes);
  const bool vec = (V % 4) == 0 && (reinterpret_cast<uintptr_t>(d_lp) % 16) == 0;
  if (T > 0) {
    const unsigned grid = warp_grid(B * T, 8);
    const int nc = (V + 127) / 128;
    if (vec && nc <= 8) {
      using KF = void (*)(const float *, int64_t, int64_t, int, const int32_t *, int32_t *, float *);
      static const KF k1[8] = {frame_topm_reg_kernel<1, 1>, frame_topm_reg_kernel<1, 2>, frame_topm_reg_kernel<1, 3>,
                               frame_topm_reg_kernel<1, 4>, frame_topm_reg_kernel<1, 5>, frame_topm_reg_kernel<1, 6>,
                               frame_topm_reg_kernel<1, 7>, frame_topm_reg_kernel<1, 8>};
      static const KF k4[8] = {frame_topm_reg_kernel<kTopM, 1>, frame_topm_reg_kernel<kTopM, 2>,
                               frame_topm_reg_kernel<kTopM, 3>, frame_topm_reg_kernel<kTopM, 4>,
                               frame_topm_reg_kernel<kTopM, 5>, frame_topm_reg_kernel<kTopM, 6>,
                               frame_topm_reg_kernel<kTopM, 7>, frame_topm_reg_kernel<kTopM, 8>};
      (M == 1 ? k1 : k4)[nc - 1]<<<grid, kThreads, 0, st>>>(d_lp, B, T, V, d_lengths, top_idx, top_lp);
    } else if (M == 1) {
      auto fa = vec ? frame_topm_kernel<1, true> : frame_topm_kernel<1, false>;
      fa<<<grid, kThreads, 0, st>>>(d_lp, B, T, V, d_lengths, top_idx, top_lp);
    } else {
      auto fa = vec ? frame_topm_kernel<kTopM, true> : frame_topm_kernel<kTopM, false>;
      fa<<<grid, kThreads, 0, st>>>(d_lp, B, T, V, d_lengths, top_idx, top_lp);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFreeAsync(ws, st);
      return fail(PGPB_ECUDA, std::string("frame_topm_kernel: ") + cudaGetErrorString(e));
    }
  }
  SeqArgs a{};
  a.t = table ? table->view : empty_view(V);
  a.lp = d_lp;
  a.B = B;
  a.T = T;
  a.V = V;
  a.lengths = d_lengths;
  a.top_idx = top_idx;
  a.top_lp = top_lp;
  a.M = M;
  a.blank = blank;
  a.lam = lam;
  a.use_boost = use_boost ? 1 : 0;
  a.tokens = d_tokens;
  a.deltas = d_deltas;
  a.ostates = d_states;
  a.nout = d_num_out;
  a.am_out = d_am;
  a.boost_out = d_boost;
  const int Vp = (V + 3) & ~3, Vw = (V + 31) >> 5;
  const size_t bm_bytes = (size_t(Vw) * 4 + 15) & ~size_t(15);
  size_t smem = 0;
  int W = kWarpsPerBlock;
  a.ring = 0;
  if (use_boost) {
    // ring depth P and warps per CTA W within ~200 KB of shared memory
    const size_t base = (size_t(Vp) * 12 + 127) & ~size_t(127);
    auto per_warp = [&](int P) {
      const size_t rows = P ? size_t(P + 1) * Vp * 4 : 0;
      return (rows + size_t(P + 1) * 8 + size_t(P) * 4 + bm_bytes + 127) & ~size_t(127);
    };
    const char *e = getenv("PGPB_CTC_RING");
    int P = (vec && (size_t(V) * 4) % 16 == 0) ? (e ? atoi(e) : 8) : 0;
    for (;;) {
      W = kWarpsPerBlock;
      while (W > 1 && base + W * per_warp(P) > 200 * 1024) --W;
      if (base + W * per_warp(P) <= 200 * 1024 || P == 0) break;
      P /= 2;
    }
    a.ring = P;
    smem = base + W * per_warp(P);
    if (smem > 220 * 1024) {
      cudaFreeAsync(ws, st);
      return fail(PGPB_EINVAL, "vocabulary too large for the shared-memory root row");
    }
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(ctc_seq_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) {
      cudaFreeAsync(ws, st);
      return fail(PGPB_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
  }
  const int64_t blocks = (B + W - 1) / W;
  ctc_seq_kernel<<<unsigned(blocks), 32 * W, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(ws, st);
  if (e != cudaSuccess) return fail(PGPB_ECUDA, std::string("ctc_seq_kernel: ") + cudaGetErrorString(e));
  return PGPB_OK;
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

#ifdef PGPB_SEQ_PROFILE
int pgpb_debug_seq_profile(unsigned long long *h_out, int reset) {
  cudaMemcpyFromSymbol(h_out, pgpb::g_seq_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(pgpb::g_seq_prof, z, sizeof(z));
  }
  return 0;
}
#endif

}  // extern "C"
