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

#include <string>

#include "pgpb_rerank.cuh"

namespace pgpb {

constexpr int kTopM = 4;

// ---------------------------------------------------------------------------
// Phase A

template <int M>
__device__ __forceinline__ void topm_insert(float (&lv)[M], int (&li)[M], float x, int v) {
  if (!argmax_better(x, v, lv[M - 1], li[M - 1])) return;
  lv[M - 1] = x;
  li[M - 1] = v;
#pragma unroll
  for (int i = M - 1; i > 0; --i) {
    if (argmax_better(lv[i], li[i], lv[i - 1], li[i - 1])) {
      const float tx = lv[i];
      lv[i] = lv[i - 1];
      lv[i - 1] = tx;
      const int ti = li[i];
      li[i] = li[i - 1];
      li[i - 1] = ti;
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
    if (lengths && (f % T) >= __ldg(lengths + f / T)) continue;
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
// Phase B helpers

__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Row -> shared buffer with 16-byte cp.async (V % 4 == 0).
__device__ __forceinline__ void issue_row(float *dst, const float *src, int V, int lane) {
  for (int c = lane; c < (V >> 2); c += 32) cp_async16(dst + 4 * c, src + 4 * c);
  cp_async_commit();
}

struct Cand {
  double c;
  float lp;
  int v;
  float s;
  int nx;
  int noff;
};

__device__ __forceinline__ void cand_consider(Cand &b, double c, float x, int v, float s, int nx, int noff) {
  if (rerank_better(c, x, v, b.c, b.lp, b.v)) b = Cand{c, x, v, s, nx, noff};
}

// Warp reduction on (c, lp, v); returns the winner with (s, nx, noff) from
// its owning lane.
__device__ __forceinline__ Cand warp_best(const Cand &mine) {
  double rc = mine.c;
  float rlp = mine.lp;
  int rv = mine.v;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(kFull, rc, o);
    const float olp = __shfl_xor_sync(kFull, rlp, o);
    const int ov = __shfl_xor_sync(kFull, rv, o);
    if (rerank_better(oc, olp, ov, rc, rlp, rv)) {
      rc = oc;
      rlp = olp;
      rv = ov;
    }
  }
  const unsigned owner = __ballot_sync(kFull, mine.v == rv);
  const int src = owner ? __ffs(owner) - 1 : 0;
  Cand w;
  w.c = rc;
  w.lp = rlp;
  w.v = rv;
  w.s = __shfl_sync(kFull, mine.s, src);
  w.nx = __shfl_sync(kFull, mine.nx, src);
  w.noff = __shfl_sync(kFull, mine.noff, src);
  return w;
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
  int prefetch;  // rows staged in shared memory (V % 4 == 0)
  int32_t *tokens;
  double *deltas;
  int32_t *ostates;
  int32_t *nout;
  double *am_out;
  double *boost_out;
};

__global__ void __launch_bounds__(kThreads) ctc_seq_kernel(SeqArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const TableView &t = a.t;
  const int V = a.V, Vp = t.vocab_padded, Vw = (V + 31) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, W = blockDim.x >> 5;
  // shared: root scores | root next | root next blob offsets | per warp: bitmap, 2 rows
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_rnext = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  int32_t *s_rnoff = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 8);
  const size_t base = size_t(Vp) * 12;
  const size_t bm_bytes = (size_t(Vw) * 4 + 15) & ~size_t(15);
  const size_t per_warp = bm_bytes + (a.prefetch ? size_t(Vp) * 8 : 0);
  unsigned *bm = reinterpret_cast<unsigned *>(smem + base + size_t(wib) * per_warp);
  float *rowbuf = reinterpret_cast<float *>(smem + base + size_t(wib) * per_warp + bm_bytes);
  if (a.use_boost) {
    for (int i = threadIdx.x; i < Vp; i += blockDim.x) {
      s_root[i] = __ldg(t.root_scores + i);
      s_rnext[i] = __ldg(t.root_next + i);
      s_rnoff[i] = __ldg(t.root_next_off + i);
    }
    for (int i = lane; i < Vw; i += 32) bm[i] = 0u;
  }
  __syncthreads();
  const int M = a.M;
  const float max_root = t.max_root_score;
  for (int64_t b = int64_t(blockIdx.x) * W + wib; b < a.B; b += int64_t(gridDim.x) * W) {
    const int64_t Tb = a.lengths ? int64_t(__ldg(a.lengths + b)) : a.T;
    const int32_t *ti = a.top_idx + b * a.T * M;
    const float *tl = a.top_lp + b * a.T * M;
    double am = 0.0, boost = 0.0;
    int last = -1, soff = a.use_boost ? __ldg(t.blob_off) : 0;
    int64_t n = 0;
    int64_t pf_frame = -1;
    int pf_buf = 0;
    for (int64_t t0 = 0; t0 < Tb; t0 += 32) {
      const int cnt = int(Tb - t0 < 32 ? Tb - t0 : 32);
      const int ca = lane < cnt ? __ldg(ti + (t0 + lane) * M) : a.blank;
      const float cl = lane < cnt ? __ldg(tl + (t0 + lane) * M) : 0.0f;
      for (int i = 0; i < cnt; ++i) {
        const int av = __shfl_sync(kFull, ca, i);
        const float lp1 = __shfl_sync(kFull, cl, i);
        if (av == a.blank || av == last) {  // blank / repeat pass through (R6)
          am += static_cast<double>(lp1);
          last = av;
          continue;
        }
        const int64_t tt = t0 + i;
        Cand w;
        if (!a.use_boost) {
          w.v = av;
          w.lp = lp1;
          w.s = 0.0f;
          w.nx = 0;
          w.noff = 0;
        } else {
          const float *grow = a.lp + (b * a.T + tt) * V;
          const float *row = grow;
          if (a.prefetch) {
            int cur;
            if (pf_frame == tt) {
              cur = pf_buf;
            } else {
              if (pf_frame >= 0) cp_async_wait_all();  // retire a stale prefetch first
              cur = pf_buf ^ 1;
              issue_row(rowbuf + cur * Vp, grow, V, lane);
            }
            // speculative prefetch of the next emitting frame, assuming the
            // argmax survives the rerank (the common case): frame j emits iff
            // its argmax is neither blank nor frame j-1's argmax
            const int prev = __shfl_up_sync(kFull, ca, 1);
            const bool cand = lane > i && lane < cnt && ca != a.blank && ca != prev;
            const unsigned m = __ballot_sync(kFull, cand);
            if (m) {
              const int64_t t2 = t0 + __ffs(m) - 1;
              issue_row(rowbuf + (cur ^ 1) * Vp, a.lp + (b * a.T + t2) * V, V, lane);
              pf_frame = t2;
              pf_buf = cur ^ 1;
              cp_async_wait_1();
            } else {
              pf_frame = -1;
              cp_async_wait_all();
            }
            __syncwarp();
            row = rowbuf + cur * Vp;
          }
          const int4 hdr = __ldg(t.blob + soff);
          const float acc = __int_as_float(hdr.y);
          const int ccount = hdr.x;
          // closure tokens -> bitmap
          for (int k = lane; k < ccount; k += 32) {
            const int tok = __ldg(&t.blob[soff + 1 + k].x);
            atomicOr(bm + (tok >> 5), 1u << (tok & 31));
          }
          __syncwarp();
          Cand mine{-INFINITY, -INFINITY, INT_MAX, 0.0f, 0, 0};
          for (int k = lane; k < ccount; k += 32) {
            const int4 e = __ldg(t.blob + soff + 1 + k);
            if (e.x == a.blank || e.x == last) continue;
            const float x = row[e.x];
            cand_consider(mine, fuse(x, a.lam, __int_as_float(e.z)), x, e.x, __int_as_float(e.z), e.y, e.w);
          }
          if (lane < M) {
            const int v = __ldg(ti + tt * M + lane);
            const float x = __ldg(tl + tt * M + lane);
            if (v < V && v != a.blank && v != last && !((bm[v >> 5] >> (v & 31)) & 1u)) {
              const float s = acc + s_root[v];
              cand_consider(mine, fuse(x, a.lam, s), x, v, s, s_rnext[v], s_rnoff[v]);
            }
          }
          if (mine.v != INT_MAX) prefetch_l1(t.blob + mine.noff);
          w = warp_best(mine);
          // exact pruning bound for dense tokens outside the top-M
          bool exact = V <= M;
          if (!exact) {
            const float lpM = __ldg(tl + tt * M + (M - 1));
            const double bound = fuse(lpM, a.lam, acc + max_root);
            exact = w.c > bound;
          }
          if (!exact) {  // full rescan of the row (rare)
            Cand full{-INFINITY, -INFINITY, INT_MAX, 0.0f, 0, 0};
            for (int v = lane; v < V; v += 32) {
              if (v == a.blank || v == last || ((bm[v >> 5] >> (v & 31)) & 1u)) continue;
              const float x = row[v];
              const float s = acc + s_root[v];
              cand_consider(full, fuse(x, a.lam, s), x, v, s, s_rnext[v], s_rnoff[v]);
            }
            for (int k = lane; k < ccount; k += 32) {
              const int4 e = __ldg(t.blob + soff + 1 + k);
              if (e.x == a.blank || e.x == last) continue;
              const float x = row[e.x];
              cand_consider(full, fuse(x, a.lam, __int_as_float(e.z)), x, e.x, __int_as_float(e.z), e.y, e.w);
            }
            w = warp_best(full);
          }
          __syncwarp();
          for (int k = lane; k < ccount; k += 32) bm[__ldg(&t.blob[soff + 1 + k].x) >> 5] = 0u;
          __syncwarp();
        }
        if (lane == 0) {
          a.tokens[b * a.T + n] = w.v;
          a.deltas[b * a.T + n] = static_cast<double>(w.s);
          a.ostates[b * a.T + n] = w.nx;
        }
        ++n;
        am += static_cast<double>(w.lp);
        boost += static_cast<double>(w.s);
        soff = w.noff;
        last = w.v;
      }
    }
    if (a.prefetch && a.use_boost) {
      cp_async_wait_all();
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
    if (M == 1) {
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
  a.prefetch = (use_boost && vec) ? 1 : 0;
  size_t smem = 0;
  int W = kWarpsPerBlock;
  if (use_boost) {
    for (;; a.prefetch = 0) {
      const size_t per_warp = bm_bytes + (a.prefetch ? size_t(Vp) * 8 : 0);
      W = kWarpsPerBlock;
      while (W > 1 && size_t(Vp) * 12 + W * per_warp > 200 * 1024) --W;
      smem = size_t(Vp) * 12 + W * per_warp;
      if (smem <= 200 * 1024 || !a.prefetch) break;
    }
    if (smem > 200 * 1024) {
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
