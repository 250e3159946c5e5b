// Advance kernel: scores[B,V], next[B,V] for a batch of tree states.
//
// Reference: _kernels.score_batch (_kernels.pyx:30-72), R5 in SURVEY.md.
// HBM-write-bound (8 B written per cell).  Kernels:
//  * advance_v6_kernel: one launch = one advance (pgpb_advance), single-pass
//    full-line stores with closure overrides patched in by bitmap rank;
//  * advance_steps_blob_kernel / advance_steps_compact_kernel: R chained
//    advances per launch (config 5, pgpb_advance_steps), rows split into
//    column parts so small batches fill the GPU, next-step operands fetched
//    behind the stores; the first reads per-state advance blobs into shared
//    memory (latency-bound launches), the second the compact advance arrays
//    (bandwidth-bound launches); V <= 1024;
//  * advance_steps_kernel: the same on the ranked bitmap rows (any V);
//  * advance_closure_kernel: generic fallback (any V, unaligned outputs);
//  * advance_chain_kernel: the reference's chain walk (pgpb_advance_chain),
//    a cross-check that does not use the flattened closure.
// Superseded variants (v1-v5, v7) and their measurements: profiles/r1_summary.md.

#include <algorithm>
#include <cstdlib>
#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

static int g_sm_count[64] = {0};

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// Keep stream-ordered allocations of the *_host entry points cached in the
// device's default memory pool across synchronizations (the default release
// threshold of 0 would hand the memory back at every sync and re-map it on
// the next call).
void retain_pool(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

int sm_count(int device) {
  if (device < 0 || device >= 64) return 148;
  if (!g_sm_count[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n < 1)
      n = 148;
    g_sm_count[device] = n;
  }
  return g_sm_count[device];
}

// Dense fill of one row: score = acc + root[v], next = root_next[v].
template <bool kVec>
__device__ __forceinline__ void write_dense_row(float *__restrict__ srow, int32_t *__restrict__ nrow,
                                                const float *root, const int32_t *rnext, float acc,
                                                int V, int lane) {
  if (kVec) {
    const int V4 = V >> 2;
    float4 *s4 = reinterpret_cast<float4 *>(srow);
    int4 *n4 = reinterpret_cast<int4 *>(nrow);
    const float4 *r4 = reinterpret_cast<const float4 *>(root);
    const int4 *q4 = reinterpret_cast<const int4 *>(rnext);
#pragma unroll 4
    for (int i = lane; i < V4; i += 32) {
      float4 r = r4[i];
      r.x = acc + r.x;  // fp32 add, operand order as _kernels.pyx:70
      r.y = acc + r.y;
      r.z = acc + r.z;
      r.w = acc + r.w;
      __stcs(s4 + i, r);
      __stcs(n4 + i, q4[i]);
    }
  } else {
    for (int v = lane; v < V; v += 32) {
      __stcs(srow + v, acc + root[v]);
      __stcs(nrow + v, rnext[v]);
    }
  }
}

template <bool kVec, bool kSmemRoot>
__global__ void __launch_bounds__(kThreads)
    advance_closure_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                           float *__restrict__ scores, int32_t *__restrict__ next) {
  extern __shared__ __align__(16) unsigned char smem[];
  const float *root = t.root_scores;
  const int32_t *rnext = t.root_next;
  if (kSmemRoot) {
    float *s_root = reinterpret_cast<float *>(smem);
    int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(t.vocab_padded) * 4);
    stage_root(t, s_root, s_next);
    __syncthreads();
    root = s_root;
    rnext = s_next;
  }
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int V = t.vocab_size;
  for (int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < B; row += nwarps) {
    const int32_t s = __ldg(states + row);
    const int4 rec = __ldg(t.clo_rec + s);
    float *srow = scores + row * V;
    int32_t *nrow = next + row * V;
    write_dense_row<kVec>(srow, nrow, root, rnext, __int_as_float(rec.z), V, lane);
    __syncwarp();
    for (int i = lane; i < rec.y; i += 32) {
      const int4 e = __ldg(t.clo + rec.x + i);
      srow[e.x] = __int_as_float(e.z);
      nrow[e.x] = e.y;
    }
  }
}

// Chain-walk variant: the reference's per-row algorithm without the
// precomputed closure.  Levels are scattered deepest-first so the level
// nearest the query state (the first hit) is written last.
constexpr int kMaxCachedLevels = 32;

template <bool kVec, bool kSmemRoot>
__global__ void __launch_bounds__(kThreads)
    advance_chain_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                         float *__restrict__ scores, int32_t *__restrict__ next) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int4 lvl[kWarpsPerBlock][kMaxCachedLevels];  // {start, end, bits(acc), state}
  const float *root = t.root_scores;
  const int32_t *rnext = t.root_next;
  if (kSmemRoot) {
    float *s_root = reinterpret_cast<float *>(smem);
    int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(t.vocab_padded) * 4);
    stage_root(t, s_root, s_next);
    __syncthreads();
    root = s_root;
    rnext = s_next;
  }
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int V = t.vocab_size;
  for (int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < B; row += nwarps) {
    // Walk the chain (uniform across the warp): acc in fp32, chain order.
    int32_t s = __ldg(states + row);
    float acc = 0.0f;
    int L = 0;
    while (s != 0) {
      const int4 r = __ldg(t.state_rec + s);
      if (L < kMaxCachedLevels && lane == 0) lvl[wib][L] = make_int4(r.x, r.y, __float_as_int(acc), s);
      acc = acc + __int_as_float(r.w);
      s = r.z;
      ++L;
    }
    __syncwarp();
    float *srow = scores + row * V;
    int32_t *nrow = next + row * V;
    write_dense_row<kVec>(srow, nrow, root, rnext, acc, V, lane);
    for (int k = L - 1; k >= 0; --k) {
      int4 lv;
      if (k < kMaxCachedLevels) {
        lv = lvl[wib][k];
      } else {  // deep chain: re-walk from the last cached level
        int4 c = lvl[wib][kMaxCachedLevels - 1];
        float a = __int_as_float(c.z);
        int32_t st = c.w;
        for (int q = kMaxCachedLevels - 1; q < k; ++q) {
          const int4 r = __ldg(t.state_rec + st);
          a = a + __int_as_float(r.w);
          st = r.z;
        }
        const int4 r = __ldg(t.state_rec + st);
        lv = make_int4(r.x, r.y, __float_as_int(a), st);
      }
      __syncwarp();
      const float a = __int_as_float(lv.z);
      for (int j = lv.x + lane; j < lv.y; j += 32) {
        const int4 e = __ldg(t.arcs + j);
        srow[e.x] = a + __int_as_float(e.z);
        nrow[e.x] = e.y;
      }
    }
    __syncwarp();
  }
}

// v6 output stores: L1::no_allocate + L2::evict_first policy (default, 2;
// 65536 rows: 80.7% of the HBM peak vs 79.1% with st.global.cs, equal at
// 8192); PGPB_ADV_STORE=0 builds st.global.cs, 1 plain stores (70%).
#ifndef PGPB_ADV_STORE
#define PGPB_ADV_STORE 2
#endif
__device__ __forceinline__ uint64_t ef_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <typename T>
__device__ __forceinline__ void adv_store(T *p, const T &v) {
#if PGPB_ADV_STORE == 1
  *p = v;
#elif PGPB_ADV_STORE == 2
  static_assert(sizeof(T) == 16, "16-byte stores");
  const int4 w = *reinterpret_cast<const int4 *>(&v);
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(w.x),
               "r"(w.y), "r"(w.z), "r"(w.w), "l"(ef_policy())
               : "memory");
#else
  __stcs(p, v);
#endif
}

// ---------------------------------------------------------------------------
// v6: v5 without the per-warp scratch row.  A row's closure arcs are sorted
// by token, so the arc overriding token v is the rank(v)-th one: per row the
// warp sets the arcs' bits in a bitmap and takes an exclusive prefix
// popcount over its words; the streaming pass finds each override's arc
// (an L1 hit: the row's arcs were just loaded) by rank.  Shared memory per
// warp drops from V*8 B to Vw*8 B, so more CTAs fit per SM.
__global__ void __launch_bounds__(kThreads, 4)
    advance_v6_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                      float *__restrict__ scores, int32_t *__restrict__ next, int rows_per_cta, int strided,
                      int tbits) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vp = t.vocab_padded, Vw = (V + 31) >> 5;
  // Row map.  Blocked: CTA c owns rows [c*rows_per_cta, ...), local row i.
  // Strided: local row i = (warp w = i % W, step j = i / W) is global row
  // (j * gridDim + c) * W + w, so at step j every warp of the grid writes
  // one contiguous block of gridDim * W rows (two write fronts per launch).
  const int64_t r0 = strided ? 0 : int64_t(blockIdx.x) * rows_per_cta;
  const int Wb = blockDim.x >> 5;
  const int64_t gstride = int64_t(gridDim.x) * Wb;
  auto grow = [&](int i) -> int64_t {
    return strided ? (int64_t(i / Wb) * gridDim.x + blockIdx.x) * Wb + (i % Wb) : r0 + i;
  };
  int n;
  if (strided) {
    const int64_t J = (B + gstride - 1) / gstride;  // steps
    const int64_t mine = int64_t(blockIdx.x) * Wb;
    // rows of this CTA: J - 1 full steps plus the valid part of the last
    const int64_t last_base = (J - 1) * gstride + mine;
    const int64_t tail = min(int64_t(Wb), max(int64_t(0), B - last_base));
    n = static_cast<int>((J - 1) * Wb + tail);
  } else {
    n = static_cast<int>(min(int64_t(rows_per_cta), B - r0));
  }
  const size_t rec_bytes = (size_t(rows_per_cta) * 16 + 255) & ~size_t(255);
  int4 *s_rec = reinterpret_cast<int4 *>(smem);
  float *s_root = reinterpret_cast<float *>(smem + rec_bytes);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + rec_bytes + size_t(Vp) * 4);
  const size_t wbytes = (size_t(Vw) * 8 + 15) & ~size_t(15);
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned *bm = reinterpret_cast<unsigned *>(smem + rec_bytes + size_t(Vp) * 8 + size_t(wib) * wbytes);
  int *pre = reinterpret_cast<int *>(bm + Vw);
  stage_root(t, s_root, s_next);
  for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int st = __ldg(states + grow(i));
    int4 rc = __ldg(t.clo_rec + st);
    rc.w = st;  // (is_final is not needed here) the state id, for its bitmap row
    s_rec[i] = rc;
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  const int V4 = V >> 2;
  const int W = blockDim.x >> 5;
  int j = wib;
  int4 rec = j < n ? s_rec[j] : make_int4(0, 0, 0, 0);
  int4 e = (lane < rec.y) ? __ldg(t.clo + rec.x + lane) : make_int4(0, 0, 0, 0);
  // tbits: the table's ranked closure bitmap row of the state (word w =
  // {bits, closure tokens in words < w}) replaces the per-row bitmap build
  // and prefix popcount; lane l holds word l (V <= 1024)
  uint2 wb = (tbits && j < n && lane < Vw) ? __ldg(t.clo_bits + int64_t(rec.w) * Vw + lane) : make_uint2(0u, 0u);
  for (; j < n; j += W) {
    if (!tbits) {
      if (lane < rec.y) atomicOr(bm + (e.x >> 5), 1u << (e.x & 31));
      for (int i = lane + 32; i < rec.y; i += 32) {
        const int tok = __ldg(&t.clo[rec.x + i].x);
        atomicOr(bm + (tok >> 5), 1u << (tok & 31));
      }
    }
    const int jn = j + W;
    const int4 nrec = jn < n ? s_rec[jn] : make_int4(0, 0, 0, 0);
    const int4 ne = (lane < nrec.y) ? __ldg(t.clo + nrec.x + lane) : make_int4(0, 0, 0, 0);
    const uint2 nwb = (tbits && jn < n && lane < Vw) ? __ldg(t.clo_bits + int64_t(nrec.w) * Vw + lane)
                                                    : make_uint2(0u, 0u);
    if (!tbits) __syncwarp();
    // exclusive prefix popcount over the bitmap words (lane-contiguous words)
    if (!tbits) {
      const int per = (Vw + 31) >> 5, w0 = lane * per;
      int cnt = 0;
      for (int k = 0; k < per; ++k)
        if (w0 + k < Vw) cnt += __popc(bm[w0 + k]);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - cnt;
      for (int k = 0; k < per; ++k)
        if (w0 + k < Vw) {
          pre[w0 + k] = run;
          run += __popc(bm[w0 + k]);
        }
    }
    if (!tbits) __syncwarp();
    const float acc = __int_as_float(rec.z);
    const int64_t row = grow(j);
    float4 *s4 = reinterpret_cast<float4 *>(scores + row * V);
    int4 *n4 = reinterpret_cast<int4 *>(next + row * V);
    const int4 *arcs = t.clo + rec.x;
#pragma unroll 4
    for (int c = lane; c < V4; c += 32) {
      float4 r = r4[c];
      int4 qv = q4[c];
      r.x = acc + r.x;
      r.y = acc + r.y;
      r.z = acc + r.z;
      r.w = acc + r.w;
      unsigned word;
      int base;
      if (tbits) {
        word = __shfl_sync(0xffffffffu, wb.x, c >> 3);
        base = int(__shfl_sync(0xffffffffu, wb.y, c >> 3));
      } else {
        word = bm[c >> 3];
        base = pre[c >> 3];
      }
      const int sh = (c & 7) * 4;
      const unsigned bits = (word >> sh) & 0xFu;
      if (bits) {
        int k = base + __popc(word & ((1u << sh) - 1u));
        if (bits & 1u) { const int4 a = __ldg(arcs + k++); r.x = __int_as_float(a.z); qv.x = a.y; }
        if (bits & 2u) { const int4 a = __ldg(arcs + k++); r.y = __int_as_float(a.z); qv.y = a.y; }
        if (bits & 4u) { const int4 a = __ldg(arcs + k++); r.z = __int_as_float(a.z); qv.z = a.y; }
        if (bits & 8u) { const int4 a = __ldg(arcs + k); r.w = __int_as_float(a.z); qv.w = a.y; }
      }
      adv_store(s4 + c, r);
      adv_store(n4 + c, qv);
    }
    if (!tbits) {
      __syncwarp();
      for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
      __syncwarp();
    }
    rec = nrec;
    e = ne;
    wb = nwb;
  }
}


// ---------------------------------------------------------------------------
// Chained R-step advance (BASELINE config 5): row b advances
// s_0 = states[b] R times, s_{k+1} = next_k[b, tok[k*B + b]], writing step
// k's rows at scores/next + (k*B + b)*V.  Per-step semantics are exactly
// one advance (_kernels.pyx:56-71) of the step's states; the successor is
// the same closure lookup the row's output holds at column tok.
//
// A work item is (row, part): the row's V/4 float4 chunks split into P
// equal parts (64 chunks each by default), so a batch smaller than the
// grid's warps (B=1024 on one of 8 GPUs) still keeps every warp streaming
// and every warp has several items to overlap.  A warp runs all R steps of its
// item with a one-step lookahead: step k+1's closure record, its part of
// the table's ranked closure bitmap row and the bitmap word of tok_{k+1}
// are loaded before step k's row is streamed, so their latency hides behind
// the stores and the per-launch dependent prologue is paid once per R steps.
// Requires the ranked bitmap rows (t.clo_bits), V % (128 P) == 0 and
// Vw <= 32 P (lane l of the warp holds word l of its part).
__global__ void __launch_bounds__(kThreads, 4)
    advance_steps_kernel(TableView t, const int32_t *__restrict__ states, const int32_t *__restrict__ tokens,
                         int R, int64_t B, int P, float *__restrict__ scores, int32_t *__restrict__ next,
                         int32_t *__restrict__ trace, int32_t *__restrict__ final_states) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vp = t.vocab_padded, Vw = t.bits_words;
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  stage_root(t, s_root, s_next);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int W = blockDim.x >> 5;
  const int64_t G = int64_t(gridDim.x) * W;
  const int CP = (V >> 2) / P;  // float4 chunks per part (multiple of 32)
  const int WP = Vw / P;        // bitmap words per part (<= 32)
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  const int64_t items = B * P;
  const int64_t cells = B * int64_t(V);
  bool triggered = false;
  for (int64_t it = int64_t(blockIdx.x) * W + (threadIdx.x >> 5); it < items; it += G) {
    const int64_t b = it / P;
    const int p = int(it - b * P);
    const int c0 = p * CP;
    int s = __ldg(states + b);
    int4 rec = __ldg(t.clo_rec + s);
    uint2 wb = lane < WP ? __ldg(t.clo_bits + int64_t(s) * Vw + p * WP + lane) : make_uint2(0u, 0u);
    // tokens == NULL: a single advance (R = 1), no successor
    int tok = tokens ? __ldg(tokens + b) : 0;
    uint2 tw = tokens ? __ldg(t.clo_bits + int64_t(s) * Vw + (tok >> 5)) : make_uint2(0u, 0u);
    if (!triggered) {
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      triggered = true;
    }
    for (int k = 0; k < R; ++k) {
      // successor of this step (uniform across the warp): closure entry by
      // rank when tok is a first-hit arc of s, else the dense root row
      const unsigned bp = unsigned(tok) & 31u;
      int sn = s;
      if (!tokens)
        ;
      else if ((tw.x >> bp) & 1u)
        sn = __ldg(&t.clo[rec.x + int(tw.y) + __popc(tw.x & ((1u << bp) - 1u))].y);
      else
        sn = s_next[tok];
      int4 nrec = make_int4(0, 0, 0, 0);
      uint2 nwb = make_uint2(0u, 0u), ntw = make_uint2(0u, 0u);
      int ntok = 0;
      if (k + 1 < R) {
        ntok = __ldg(tokens + int64_t(k + 1) * B + b);
        nrec = __ldg(t.clo_rec + sn);
        if (lane < WP) nwb = __ldg(t.clo_bits + int64_t(sn) * Vw + p * WP + lane);
        ntw = __ldg(t.clo_bits + int64_t(sn) * Vw + (ntok >> 5));
      }
      const float acc = __int_as_float(rec.z);
      const int64_t rowoff = int64_t(k) * cells + b * V;
      float4 *s4 = reinterpret_cast<float4 *>(scores + rowoff);
      int4 *n4 = reinterpret_cast<int4 *>(next + rowoff);
      const int4 *arcs = t.clo + rec.x;
#pragma unroll 2
      for (int c = c0 + lane; c < c0 + CP; c += 32) {
        float4 r = r4[c];
        int4 qv = q4[c];
        r.x = acc + r.x;  // fp32 add, operand order as _kernels.pyx:70
        r.y = acc + r.y;
        r.z = acc + r.z;
        r.w = acc + r.w;
        const int wl = (c >> 3) - p * WP;
        const unsigned word = __shfl_sync(kFull, wb.x, wl);
        const int base = int(__shfl_sync(kFull, wb.y, wl));
        const int sh = (c & 7) * 4;
        const unsigned bits = (word >> sh) & 0xFu;
        if (bits) {
          int q = base + __popc(word & ((1u << sh) - 1u));
          if (bits & 1u) { const int4 a = __ldg(arcs + q++); r.x = __int_as_float(a.z); qv.x = a.y; }
          if (bits & 2u) { const int4 a = __ldg(arcs + q++); r.y = __int_as_float(a.z); qv.y = a.y; }
          if (bits & 4u) { const int4 a = __ldg(arcs + q++); r.z = __int_as_float(a.z); qv.z = a.y; }
          if (bits & 8u) { const int4 a = __ldg(arcs + q); r.w = __int_as_float(a.z); qv.w = a.y; }
        }
        adv_store(s4 + c, r);
        adv_store(n4 + c, qv);
      }
      if (trace && p == 0 && lane == 0) trace[int64_t(k) * B + b] = s;
      s = sn;
      rec = nrec;
      wb = nwb;
      tok = ntok;
      tw = ntw;
    }
    if (final_states && p == 0 && lane == 0) final_states[b] = s;
  }
  if (!triggered) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// advance_steps_kernel on the compact arrays (t.adv_bits, V <= 1024): the
// warp loads the state's whole bitmap line (lane l = word l) and derives
// each word's rank with an exclusive popc scan, so the successor's token
// word comes from registers and the closure entries are 8-byte
// {next, score} pairs: about half the table bytes per random row.
__device__ __forceinline__ unsigned excl_popc_scan(unsigned w, int lane) {
  const unsigned c = __popc(w);
  unsigned x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x - c;
}

__global__ void __launch_bounds__(kThreads, 4)
    advance_steps_compact_kernel(TableView t, const int32_t *__restrict__ states, const int32_t *__restrict__ tokens,
                                 int R, int64_t B, int P, float *__restrict__ scores, int32_t *__restrict__ next,
                                 int32_t *__restrict__ trace, int32_t *__restrict__ final_states) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vp = t.vocab_padded, Vw = t.bits_words;
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  stage_root(t, s_root, s_next);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int W = blockDim.x >> 5;
  const int64_t G = int64_t(gridDim.x) * W;
  const int CP = (V >> 2) / P;  // float4 chunks per part (multiple of 32)
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  const int64_t items = B * P;
  const int64_t cells = B * int64_t(V);
  bool triggered = false;
  for (int64_t it = int64_t(blockIdx.x) * W + (threadIdx.x >> 5); it < items; it += G) {
    const int64_t b = it / P;
    const int p = int(it - b * P);
    const int c0 = p * CP;
    int s = __ldg(states + b);
    const int4 r0 = __ldg(t.clo_rec + s);
    int2 rec = make_int2(r0.x, r0.y);  // {clo_start, clo_count}
    float acc = __int_as_float(r0.z);
    unsigned w = lane < Vw ? __ldg(t.adv_bits + int64_t(s) * Vw + lane) : 0u;
    int tok = tokens ? __ldg(tokens + b) : 0;
    if (!triggered) {
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      triggered = true;
    }
    for (int k = 0; k < R; ++k) {
      // successor (warp-uniform) first, it heads the dependent chain: the
      // token's word from registers, its rank by one reduction
      int sn = s;
      if (tokens) {
        const int wt = tok >> 5;
        const unsigned tw = __shfl_sync(kFull, w, wt);
        const unsigned tr = __reduce_add_sync(kFull, lane < wt ? unsigned(__popc(w)) : 0u);
        const unsigned bp = unsigned(tok) & 31u;
        sn = ((tw >> bp) & 1u) ? __ldg(&t.adv_clo[rec.x + int(tr) + __popc(tw & ((1u << bp) - 1u))].x)
                               : s_next[tok];
      }
      int2 nrec = make_int2(0, 0);
      float nacc = 0.0f;
      unsigned nw = 0u;
      int ntok = 0;
      if (k + 1 < R) {
        ntok = __ldg(tokens + int64_t(k + 1) * B + b);
        const int4 r = __ldg(t.clo_rec + sn);
        nrec = make_int2(r.x, r.y);
        nacc = __int_as_float(r.z);
        if (lane < Vw) nw = __ldg(t.adv_bits + int64_t(sn) * Vw + lane);
      }
      // word ranks for the row stream, while the lookahead loads are in flight
      const unsigned rank = excl_popc_scan(w, lane);
      const int64_t rowoff = int64_t(k) * cells + b * V;
      float4 *s4 = reinterpret_cast<float4 *>(scores + rowoff);
      int4 *n4 = reinterpret_cast<int4 *>(next + rowoff);
      const int2 *arcs = t.adv_clo + rec.x;
#pragma unroll 2
      for (int c = c0 + lane; c < c0 + CP; c += 32) {
        float4 r = r4[c];
        int4 qv = q4[c];
        r.x = acc + r.x;  // fp32 add, operand order as _kernels.pyx:70
        r.y = acc + r.y;
        r.z = acc + r.z;
        r.w = acc + r.w;
        const unsigned word = __shfl_sync(kFull, w, c >> 3);
        const int base = int(__shfl_sync(kFull, rank, c >> 3));
        const int sh = (c & 7) * 4;
        const unsigned bits = (word >> sh) & 0xFu;
        if (bits) {
          int q = base + __popc(word & ((1u << sh) - 1u));
          if (bits & 1u) { const int2 a = __ldg(arcs + q++); r.x = __int_as_float(a.y); qv.x = a.x; }
          if (bits & 2u) { const int2 a = __ldg(arcs + q++); r.y = __int_as_float(a.y); qv.y = a.x; }
          if (bits & 4u) { const int2 a = __ldg(arcs + q++); r.z = __int_as_float(a.y); qv.z = a.x; }
          if (bits & 8u) { const int2 a = __ldg(arcs + q); r.w = __int_as_float(a.y); qv.w = a.x; }
        }
        adv_store(s4 + c, r);
        adv_store(n4 + c, qv);
      }
      if (trace && p == 0 && lane == 0) trace[int64_t(k) * B + b] = s;
      s = sn;
      rec = nrec;
      acc = nacc;
      w = nw;
      tok = ntok;
    }
    if (final_states && p == 0 && lane == 0) final_states[b] = s;
  }
  if (!triggered) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// advance_steps on the per-state advance blobs (t.adv_blob): a warp copies
// the next state's whole blob (closure accumulator, bitmap words, word ranks,
// {next, score} pairs) into its shared-memory buffer with one 16-B cp.async
// per lane, one step ahead, so a step resolves its successor, ranks and
// every override from shared memory: no dependent global load on the step's
// path (the closure-override loads inside the stream were its largest
// stall, profiles/r2_summary.md §4).
__device__ __forceinline__ void adv_cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 4)
    advance_steps_blob_kernel(TableView t, const int32_t *__restrict__ states, const int32_t *__restrict__ tokens,
                              int R, int64_t B, int P, float *__restrict__ scores, int32_t *__restrict__ next,
                              int32_t *__restrict__ trace, int32_t *__restrict__ final_states) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vp = t.vocab_padded, Vw = t.bits_words;
  const int S16 = t.adv_stride16, E0 = t.adv_ent0;
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int4 *bufs = reinterpret_cast<int4 *>(smem + size_t(Vp) * 8) + size_t(wid) * 2 * S16;  // 2 blobs per warp
  // closure counts of the root row's successors (sizes the copy of a dense successor's blob)
  unsigned char *s_cnt = reinterpret_cast<unsigned char *>(smem + size_t(Vp) * 8 + size_t(blockDim.x >> 5) * 2 * S16 * 16);
  stage_root(t, s_root, s_next);
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) s_cnt[v] = __ldg(t.adv_root_cnt + v);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int W = blockDim.x >> 5;
  const int64_t G = int64_t(gridDim.x) * W;
  const int CP = (V >> 2) / P;
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  const int64_t items = B * P;
  const int64_t cells = B * int64_t(V);
  // copy the used prefix of a blob: header, words, ranks and cnt pairs
  auto fetch = [&](int st, int cnt, int slot) {
    const int4 *src = t.adv_blob + int64_t(st) * S16;
    int4 *dst = bufs + slot * S16;
    const int n16 = min(S16, (E0 + 2 * cnt + 3) >> 2);
    for (int i = lane; i < n16; i += 32) adv_cp_async16(dst + i, src + i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  bool triggered = false;
  for (int64_t it = int64_t(blockIdx.x) * W + wid; it < items; it += G) {
    const int64_t b = it / P;
    const int p = int(it - b * P);
    const int c0 = p * CP;
    int s = __ldg(states + b);
    int tok = tokens ? __ldg(tokens + b) : 0;
    __syncwarp();  // the previous item's reads of both buffers are done
    fetch(s, 64, 0);  // count unknown: the whole blob
    if (!triggered) {
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      triggered = true;
    }
    for (int k = 0; k < R; ++k) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      const int32_t *cur = reinterpret_cast<const int32_t *>(bufs + (k & 1) * S16);
      const unsigned *wds = reinterpret_cast<const unsigned *>(cur + 4);
      const uint16_t *rks = reinterpret_cast<const uint16_t *>(cur + 4 + Vw);
      const int2 *ent = reinterpret_cast<const int2 *>(cur + E0);
      const float acc = __int_as_float(cur[0]);
      // successor from the blob, then the next blob's copy behind this step's stream
      int sn = s, cn = 64;
      int ntok = 0;
      if (tokens) {
        const unsigned tw = wds[tok >> 5];
        const unsigned bp = unsigned(tok) & 31u;
        if ((tw >> bp) & 1u) {
          const int e = ent[int(rks[tok >> 5]) + __popc(tw & ((1u << bp) - 1u))].x;
          sn = e & 0x1FFFFFF;
          cn = int(unsigned(e) >> 25);
        } else {
          sn = s_next[tok];
          cn = s_cnt[tok];
        }
      }
      if (k + 1 < R) {
        ntok = __ldg(tokens + int64_t(k + 1) * B + b);
        fetch(sn, cn, (k + 1) & 1);
      }
      const int64_t rowoff = int64_t(k) * cells + b * V;
      float4 *s4 = reinterpret_cast<float4 *>(scores + rowoff);
      int4 *n4 = reinterpret_cast<int4 *>(next + rowoff);
#pragma unroll 2
      for (int c = c0 + lane; c < c0 + CP; c += 32) {
        float4 r = r4[c];
        int4 qv = q4[c];
        r.x = acc + r.x;  // fp32 add, operand order as _kernels.pyx:70
        r.y = acc + r.y;
        r.z = acc + r.z;
        r.w = acc + r.w;
        const unsigned word = wds[c >> 3];
        const int sh = (c & 7) * 4;
        const unsigned bits = (word >> sh) & 0xFu;
        if (bits) {
          int q = int(rks[c >> 3]) + __popc(word & ((1u << sh) - 1u));
          if (bits & 1u) { const int2 a = ent[q++]; r.x = __int_as_float(a.y); qv.x = a.x & 0x1FFFFFF; }
          if (bits & 2u) { const int2 a = ent[q++]; r.y = __int_as_float(a.y); qv.y = a.x & 0x1FFFFFF; }
          if (bits & 4u) { const int2 a = ent[q++]; r.z = __int_as_float(a.y); qv.z = a.x & 0x1FFFFFF; }
          if (bits & 8u) { const int2 a = ent[q]; r.w = __int_as_float(a.y); qv.w = a.x & 0x1FFFFFF; }
        }
        adv_store(s4 + c, r);
        adv_store(n4 + c, qv);
      }
      if (trace && p == 0 && lane == 0) trace[int64_t(k) * B + b] = s;
      s = sn;
      tok = ntok;
      __syncwarp();  // this buffer is refilled two steps on
    }
    if (final_states && p == 0 && lane == 0) final_states[b] = s;
  }
  if (!triggered) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Successor gather for the generic chained path: s'[b] = next[b, tok[b]].
__global__ void __launch_bounds__(256)
    gather_next_kernel(const int32_t *__restrict__ next, const int32_t *__restrict__ tok, int64_t B, int V,
                       int32_t *__restrict__ out) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b < B) out[b] = next[b * V + tok[b]];
}

using AdvFn = void (*)(TableView, const int32_t *, int64_t, float *, int32_t *);

static cudaLaunchConfig_t pdl_config(dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     cudaLaunchAttribute *attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

static int steps_parts(const TableView &t);
static int launch_advance_steps(const pgpb_table *table, const int32_t *d_states, const int32_t *d_tokens,
                                int32_t R, int64_t B, float *d_scores, int32_t *d_next, int32_t *d_trace,
                                int32_t *d_final, int32_t parts, void *stream);

static int launch_advance(const pgpb_table *table, const int32_t *d_states, int64_t B,
                          float *d_scores, int32_t *d_next, void *stream, bool chain) {
  if (!table) return fail(PGPB_EINVAL, "table is NULL");
  if (B < 0) return fail(PGPB_EINVAL, "batch must be >= 0");
  if (B == 0) return PGPB_OK;
  if (!d_states || !d_scores || !d_next) return fail(PGPB_EINVAL, "NULL buffer");
  const TableView &t = table->view;
  const bool vec = (t.vocab_size % 4) == 0 && (reinterpret_cast<uintptr_t>(d_scores) % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(d_next) % 16) == 0;
  const size_t root_bytes = size_t(t.vocab_padded) * 8;
  const bool smem_root = root_bytes <= size_t(kMaxSmemRootBytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nsm = sm_count(current_device());
  // Small batches: one step of the blob kernel (rows split into column parts,
  // operands from shared memory) beats the single-advance kernel's dependent
  // startup (1024 rows 34% vs 30% of the HBM peak, 128 rows 6% vs 4%; from
  // 8192 rows the single-advance kernel is faster, 75% vs 62%)
  if (!chain && vec && t.adv_blob && B <= 2048 && tuning().adv_compact == 0 && steps_parts(t) > 0 &&
      root_bytes <= 64 * 1024)
    return launch_advance_steps(table, d_states, nullptr, 1, B, d_scores, d_next, nullptr, nullptr, 0, stream);
  if (!chain && vec && smem_root) {
    const int Vw = (t.vocab_size + 31) >> 5;
    const size_t wbytes = (size_t(Vw) * 8 + 15) & ~size_t(15);
    // Geometry: 4 CTAs per SM (64 registers per thread); rows go to warps
    // round-robin inside a CTA, so pick the warp count (4..8) that divides
    // the CTA's rows most evenly (8192 rows: 14 per CTA on 7 warps, measured
    // best of the 3..6 x 4..8 grid).
    const int per_sm = 4;
    int W = kWarpsPerBlock;
    {
      const int64_t c = int64_t(nsm) * per_sm;
      const int64_t r = std::max<int64_t>(1, (B + c - 1) / c);
      double best = 1e30;
      for (int w = kWarpsPerBlock; w >= 4; --w) {
        const double cost = double((r + w - 1) / w) / (double(r) / double(w));
        if (cost < best - 1e-9) {
          best = cost;
          W = w;
        }
      }
    }
    int64_t ctas = int64_t(nsm) * per_sm;
    int rows = int((B + ctas - 1) / ctas);
    if (rows < 1) rows = 1;
    ctas = (B + rows - 1) / rows;
    // Row map: strided (every step of the grid writes one contiguous block
    // of rows) once each warp has >= 4 rows (65536 rows: 79.1% vs 77.2% of
    // the measured HBM peak); blocked below (8192 rows: equal within noise).
    const int64_t J = (B + ctas * W - 1) / (ctas * W);  // rows per warp, strided
    const int strided = J >= 4 ? 1 : 0;
    if (strided) rows = int(J * W);  // capacity per CTA: J steps of W rows
    const size_t rec_bytes = (size_t(rows) * 16 + 255) & ~size_t(255);
    const size_t smem6 = rec_bytes + root_bytes + size_t(kWarpsPerBlock) * wbytes;
    if (smem6 <= 200 * 1024) {
      if (smem6 > 48 * 1024)
        PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(advance_v6_kernel),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem6)));
      cudaLaunchAttribute attr[1];
      cudaLaunchConfig_t cfg = pdl_config(dim3(unsigned(ctas)), dim3(32 * W), smem6, st, attr);
      // The table's ranked bitmap rows (when built, V <= 1024) instead of a
      // per-row bitmap build, for batches where a warp has at most one row:
      // it takes the build off the dependent startup chain (B=128: 4.35% vs
      // 3.87% of the HBM peak, B=1024: 29.4% vs 27.4%); with more rows per
      // warp the build overlaps the previous row's stream and the per-chunk
      // word shuffles cost more than the shared-memory reads (B=8192: 73.6%
      // vs 74.5%, 65536: 78.2% vs 80.0%).  V % 128 == 0: every lane runs
      // every chunk iteration, so the shuffles are warp-uniform.
      const bool tb_ok = t.clo_bits && Vw <= 32 && t.vocab_size % 128 == 0;
      const int tbits = (tb_ok && rows <= W) ? 1 : 0;
      PGPB_CUDA_TRY(cudaLaunchKernelEx(&cfg, advance_v6_kernel, t, d_states, B, d_scores, d_next, rows, strided,
                                       tbits));
      PGPB_CUDA_TRY(cudaGetLastError());
      return PGPB_OK;
    }
  }
  // Generic paths: any V / alignment / root size (closure kernel), and the
  // reference chain walk (pgpb_advance_chain).
  const size_t smem = smem_root ? root_bytes : 0;
  AdvFn fn;
  if (chain) {
    fn = vec ? (smem_root ? advance_chain_kernel<true, true> : advance_chain_kernel<true, false>)
             : (smem_root ? advance_chain_kernel<false, true> : advance_chain_kernel<false, false>);
  } else {
    fn = vec ? (smem_root ? advance_closure_kernel<true, true> : advance_closure_kernel<true, false>)
             : (smem_root ? advance_closure_kernel<false, true> : advance_closure_kernel<false, false>);
  }
  if (smem > 48 * 1024) {
    PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  const int per_sm = smem <= 16 * 1024 ? 8 : (smem <= 48 * 1024 ? 4 : 1);
  const unsigned grid = warp_grid(B, per_sm);
  fn<<<grid, kThreads, smem, st>>>(t, d_states, B, d_scores, d_next);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}

// Parts per row for the chained kernel: 64 float4 chunks per part (two per
// lane), the measured best at every batch (scripts/advance_steps_sweep.py,
// V=1024: P=4 gives 74% / 90% / 91% of the HBM peak at B=1024 / 8192 / 65536
// against 50% / 84% / 85% for whole rows and 54-67% for P=8), or the
// nearest valid P.  0 when no P is valid.
static int steps_parts(const TableView &t) {
  const int want = std::max(1, t.vocab_size / 256);
  int best = 0, dist = 1 << 30;
  for (int P = 1; P <= 32; P <<= 1) {
    if (t.vocab_size % (128 * P) != 0 || t.bits_words > 32 * P) continue;
    const int d = P > want ? P - want : want - P;
    if (d < dist) {
      dist = d;
      best = P;
    }
  }
  return best;
}

static int launch_advance_steps(const pgpb_table *table, const int32_t *d_states, const int32_t *d_tokens,
                                int32_t R, int64_t B, float *d_scores, int32_t *d_next, int32_t *d_trace,
                                int32_t *d_final, int32_t parts, void *stream) {
  if (!table) return fail(PGPB_EINVAL, "table is NULL");
  if (B < 0 || R < 0) return fail(PGPB_EINVAL, "batch and steps must be >= 0");
  if (B == 0 || R == 0) return PGPB_OK;
  if (!d_states || !d_scores || !d_next) return fail(PGPB_EINVAL, "NULL buffer");
  if (!d_tokens && R != 1) return fail(PGPB_EINVAL, "tokens are required for more than one step");
  const TableView &t = table->view;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nsm = sm_count(current_device());
  const size_t root_bytes = size_t(t.vocab_padded) * 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(d_scores) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(d_next) % 16) == 0;
  const int per_sm = 4;
  int P = parts > 0 ? parts : steps_parts(t);
  const bool ok = P > 0 && t.clo_bits && aligned && root_bytes <= 64 * 1024 &&
                  t.vocab_size % (128 * P) == 0 && t.bits_words <= 32 * P;
  if (ok) {
    const int64_t items = B * P;
    const int64_t ctas = std::min<int64_t>(int64_t(nsm) * per_sm, (items + kWarpsPerBlock - 1) / kWarpsPerBlock);
    // the compact arrays when built (V <= 1024): with uniformly random states
    // 89.0% vs 86.7% of the HBM peak at 8192 rows, 92.8% vs 89.1% at 65536,
    // equal at 1024 (profiles/r2_summary.md §4); the ranked-bitmap kernel
    // otherwise (tuning adv.compact = 1 forces it, for its tests)
    // Kernel by regime (uniformly random states, profiles/r2_summary.md §4):
    // up to R*B = 131072 rows per launch (<= 1 GiB of output) the launch is
    // latency-bound and the advance blobs win (1024 rows x 32 steps: 87.6% vs
    // 78.3% of the HBM peak, 8192 x 8: 91.9% vs 89.0%); above it the stream
    // is bandwidth-bound and the compact arrays' smaller table footprint wins
    // (8192 x 32: 93.1% vs 91.0%).  Tuning adv.compact: 1 ranked-bitmap
    // kernel, 2 compact arrays, 3 blobs (tests).
    const int lay = tuning().adv_compact;
    auto fn = (t.adv_bits && lay != 1) ? advance_steps_compact_kernel : advance_steps_kernel;
    size_t smem = root_bytes;
    const bool blob = t.adv_blob && (lay == 3 || (lay == 0 && int64_t(R) * B <= 131072));
    if (blob) {
      fn = advance_steps_blob_kernel;
      smem += size_t(kWarpsPerBlock) * 2 * size_t(t.adv_stride16) * 16 + size_t(t.vocab_padded);
    }
    if (smem > 48 * 1024)
      PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = pdl_config(dim3(unsigned(ctas)), dim3(kThreads), smem, st, attr);
    PGPB_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, t, d_states, d_tokens, int(R), B, P, d_scores, d_next, d_trace,
                                     d_final));
    PGPB_CUDA_TRY(cudaGetLastError());
    return PGPB_OK;
  }
  if (parts > 0) return fail(PGPB_EINVAL, "parts does not divide the row for this table");
  // Generic: R single-step advances, the successor gathered from each
  // step's next-state rows.
  int32_t *cur = nullptr;
  PGPB_CUDA_TRY(cudaMallocAsync(&cur, size_t(2 * B) * 4, st));
  int32_t *bufs[2] = {cur, cur + B};
  const int64_t cells = B * int64_t(t.vocab_size);
  const unsigned g = unsigned((B + 255) / 256);
  int rc = PGPB_OK;
  const int32_t *src = d_states;
  for (int k = 0; k < R && rc == PGPB_OK; ++k) {
    if (d_trace) {
      if (cudaMemcpyAsync(d_trace + int64_t(k) * B, src, size_t(B) * 4, cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess) {
        rc = fail(PGPB_ECUDA, "trace copy failed");
        break;
      }
    }
    rc = launch_advance(table, src, B, d_scores + k * cells, d_next + k * cells, stream, false);
    if (rc != PGPB_OK) break;
    if (!d_tokens) break;  // single advance, no successor
    int32_t *dst = (k + 1 == R && d_final) ? d_final : bufs[k & 1];
    gather_next_kernel<<<g, 256, 0, st>>>(d_next + k * cells, d_tokens + int64_t(k) * B, B, t.vocab_size, dst);
    if (cudaGetLastError() != cudaSuccess) rc = fail(PGPB_ECUDA, "gather_next_kernel launch failed");
    src = dst;
  }
  cudaFreeAsync(cur, st);
  return rc;
}

}  // namespace pgpb

extern "C" {

int pgpb_advance(const pgpb_table *table, const int32_t *d_states, int64_t B, float *d_scores,
                 int32_t *d_next, void *stream) {
  return pgpb::launch_advance(table, d_states, B, d_scores, d_next, stream, false);
}

int pgpb_advance_chain(const pgpb_table *table, const int32_t *d_states, int64_t B,
                       float *d_scores, int32_t *d_next, void *stream) {
  return pgpb::launch_advance(table, d_states, B, d_scores, d_next, stream, true);
}

int pgpb_advance_steps(const pgpb_table *table, const int32_t *d_states, const int32_t *d_tokens, int32_t steps,
                       int64_t B, float *d_scores, int32_t *d_next, int32_t *d_trace, int32_t *d_final_states,
                       int32_t parts, void *stream) {
  return pgpb::launch_advance_steps(table, d_states, d_tokens, steps, B, d_scores, d_next, d_trace,
                                    d_final_states, parts, stream);
}

int pgpb_advance_host(const pgpb_table *table, const int32_t *h_states, int64_t B,
                      float *h_scores, int32_t *h_next, void *stream) {
  using pgpb::fail;
  if (!table) return fail(PGPB_EINVAL, "table is NULL");
  if (B < 0) return fail(PGPB_EINVAL, "batch must be >= 0");
  if (B == 0) return PGPB_OK;
  const int32_t S = table->view.num_states;
  for (int64_t i = 0; i < B; ++i)
    if (h_states[i] < 0 || h_states[i] >= S)
      return fail(PGPB_ERANGE, "state id out of range [0, " + std::to_string(S) + ")");
  const int64_t V = table->view.vocab_size;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int prev = 0;
  PGPB_CUDA_TRY(cudaGetDevice(&prev));
  PGPB_CUDA_TRY(cudaSetDevice(table->device));
  pgpb::retain_pool(table->device);
  const size_t cells = size_t(B) * size_t(V);
  const size_t o_sc = 0, o_nx = ((cells * 4 + 255) / 256) * 256,
               o_st = o_nx + ((cells * 4 + 255) / 256) * 256;
  char *buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, o_st + size_t(B) * 4, st);
  int rc = PGPB_OK;
  if (e != cudaSuccess) {
    cudaSetDevice(prev);
    return fail(PGPB_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  }
  int32_t *d_states = reinterpret_cast<int32_t *>(buf + o_st);
  float *d_scores = reinterpret_cast<float *>(buf + o_sc);
  int32_t *d_next = reinterpret_cast<int32_t *>(buf + o_nx);
  e = cudaMemcpyAsync(d_states, h_states, size_t(B) * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) rc = pgpb_advance(table, d_states, B, d_scores, d_next, stream);
  if (e == cudaSuccess && rc == PGPB_OK)
    e = cudaMemcpyAsync(h_scores, d_scores, cells * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && rc == PGPB_OK)
    e = cudaMemcpyAsync(h_next, d_next, cells * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(buf, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  cudaSetDevice(prev);
  if (rc != PGPB_OK) return rc;
  if (e != cudaSuccess) return fail(PGPB_ECUDA, std::string("advance_host: ") + cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(PGPB_ECUDA, std::string("advance_host sync: ") + cudaGetErrorString(e2));
  return PGPB_OK;
}

}  // extern "C"
