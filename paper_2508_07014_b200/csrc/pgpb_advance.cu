// Advance kernel: scores[B,V], next[B,V] for a batch of tree states.
//
// Reference: _kernels.score_batch (_kernels.pyx:30-72), R5 in SURVEY.md.
// HBM-write-bound (8 B written per cell).  The production
// kernel is advance_v5_kernel (single-pass full-line stores, ~80% of the
// measured HBM copy bandwidth at 8192 x 1024, profiles/); v1 (warp per row,
// dense stores then scattered overrides), v2 (chunked CTAs), v3 (TMA bulk
// stores from shared memory) and the chain-walk kernel are kept selectable
// through PGPB_ADVANCE_VARIANT for measurement and as cross-checks.

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

// ---------------------------------------------------------------------------
// v2: chunked persistent CTAs.  Each CTA owns a contiguous run of rows; its
// prologue loads every row's state and closure record into shared memory
// (overlapping the root-row staging), and each warp prefetches its row's
// closure entries before issuing the dense stores, so the dependent-load
// latency hides behind the store stream.
template <bool kVec, bool kSmemRoot>
__global__ void __launch_bounds__(kThreads, 4)
    advance_v2_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                      float *__restrict__ scores, int32_t *__restrict__ next, int rows_per_cta) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int n = static_cast<int>(min(int64_t(rows_per_cta), B - r0));
  int4 *s_rec = reinterpret_cast<int4 *>(smem);
  const size_t rec_bytes = (size_t(rows_per_cta) * 16 + 255) & ~size_t(255);
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_rec[i] = __ldg(t.clo_rec + __ldg(states + r0 + i));
  const float *root = t.root_scores;
  const int32_t *rnext = t.root_next;
  if (kSmemRoot) {
    float *s_root = reinterpret_cast<float *>(smem + rec_bytes);
    int32_t *s_next = reinterpret_cast<int32_t *>(smem + rec_bytes + size_t(t.vocab_padded) * 4);
    stage_root(t, s_root, s_next);
    root = s_root;
    rnext = s_next;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int V = t.vocab_size;
  for (int j = threadIdx.x >> 5; j < n; j += kWarpsPerBlock) {
    const int4 rec = s_rec[j];
    int4 e0 = make_int4(0, 0, 0, 0);
    if (lane < rec.y) e0 = __ldg(t.clo + rec.x + lane);
    const int64_t row = r0 + j;
    float *srow = scores + row * V;
    int32_t *nrow = next + row * V;
    write_dense_row<kVec>(srow, nrow, root, rnext, __int_as_float(rec.z), V, lane);
    __syncwarp();
    if (lane < rec.y) {
      srow[e0.x] = __int_as_float(e0.z);
      nrow[e0.x] = e0.y;
    }
    for (int i = lane + 32; i < rec.y; i += 32) {
      const int4 e = __ldg(t.clo + rec.x + i);
      srow[e.x] = __int_as_float(e.z);
      nrow[e.x] = e.y;
    }
  }
}

// ---------------------------------------------------------------------------
// v3: rows assembled in shared memory and written by the TMA engine with
// bulk async copies (cp.async.bulk.global.shared::cta, SASS UBLKCP), double
// buffered per warp.  Requires V % 4 == 0 (16-byte aligned rows).
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads)
    advance_v3_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                      float *__restrict__ scores, int32_t *__restrict__ next, int warps) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size;
  const int Vp = t.vocab_padded;
  float *s_root = reinterpret_cast<float *>(smem);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + size_t(Vp) * 4);
  stage_root(t, s_root, s_next);
  __syncthreads();
  const int wib = threadIdx.x >> 5;
  if (wib >= warps) return;
  const int lane = threadIdx.x & 31;
  // per-warp double buffer: [2][scores Vp | next Vp]
  unsigned char *wbuf = smem + size_t(Vp) * 8 + size_t(wib) * 2 * size_t(Vp) * 8;
  const int64_t nw = int64_t(gridDim.x) * warps;
  const int V4 = V >> 2;
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  int buf = 0;
  int64_t row = int64_t(blockIdx.x) * warps + wib;
  int4 rec = make_int4(0, 0, 0, 0);
  if (row < B) rec = __ldg(t.clo_rec + __ldg(states + row));
  for (; row < B; row += nw) {
    // prefetch the next row's record and this row's first closure entries
    int4 nrec = make_int4(0, 0, 0, 0);
    if (row + nw < B) nrec = __ldg(t.clo_rec + __ldg(states + row + nw));
    int4 e0 = make_int4(0, 0, 0, 0);
    if (lane < rec.y) e0 = __ldg(t.clo + rec.x + lane);
    float *sb = reinterpret_cast<float *>(wbuf + size_t(buf) * Vp * 8);
    int32_t *nb = reinterpret_cast<int32_t *>(sb + Vp);
    // the bulk store issued two rows ago from this buffer must have
    // finished reading it
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    const float acc = __int_as_float(rec.z);
    float4 *sb4 = reinterpret_cast<float4 *>(sb);
    int4 *nb4 = reinterpret_cast<int4 *>(nb);
#pragma unroll 4
    for (int i = lane; i < V4; i += 32) {
      float4 r = r4[i];
      r.x = acc + r.x;
      r.y = acc + r.y;
      r.z = acc + r.z;
      r.w = acc + r.w;
      sb4[i] = r;
      nb4[i] = q4[i];
    }
    __syncwarp();
    if (lane < rec.y) {
      sb[e0.x] = __int_as_float(e0.z);
      nb[e0.x] = e0.y;
    }
    for (int i = lane + 32; i < rec.y; i += 32) {
      const int4 e = __ldg(t.clo + rec.x + i);
      sb[e.x] = __int_as_float(e.z);
      nb[e.x] = e.y;
    }
    fence_async_shared();
    __syncwarp();
    if (lane == 0) {
      bulk_store(scores + row * V, sb, uint32_t(V) * 4);
      bulk_store(next + row * V, nb, uint32_t(V) * 4);
      bulk_commit();
    }
    buf ^= 1;
    rec = nrec;
  }
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
}

// ---------------------------------------------------------------------------
// v5: single-pass full-line stores.  A row's closure overrides are first
// dropped into a per-warp shared scratch row + bitmap; the dense pass then
// merges them into the 16-byte vectors in registers, so every output byte is
// written exactly once with st.global.cs.v4 (no partial-sector rewrites).
// The next row's closure entries are prefetched into registers while the
// current row streams out.  Requires V % 4 == 0 and smem root staging.
__global__ void __launch_bounds__(kThreads, 3)
    advance_v5_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                      float *__restrict__ scores, int32_t *__restrict__ next, int rows_per_cta, int split) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vp = t.vocab_padded, Vw = (V + 31) >> 5;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int n = static_cast<int>(min(int64_t(rows_per_cta), B - r0));
  const size_t rec_bytes = (size_t(rows_per_cta) * 16 + 255) & ~size_t(255);
  int4 *s_rec = reinterpret_cast<int4 *>(smem);
  float *s_root = reinterpret_cast<float *>(smem + rec_bytes);
  int32_t *s_next = reinterpret_cast<int32_t *>(smem + rec_bytes + size_t(Vp) * 4);
  const size_t wbytes = size_t(Vp) * 8 + ((size_t(Vw) * 4 + 15) & ~size_t(15));
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wb = smem + rec_bytes + size_t(Vp) * 8 + size_t(wib) * wbytes;
  float *ovs = reinterpret_cast<float *>(wb);
  int32_t *ovn = reinterpret_cast<int32_t *>(wb + size_t(Vp) * 4);
  unsigned *bm = reinterpret_cast<unsigned *>(wb + size_t(Vp) * 8);
  // table-only prologue first; with programmatic dependent launch it overlaps
  // the previous kernel's tail, and the states are read after the wait
  stage_root(t, s_root, s_next);
  for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_rec[i] = __ldg(t.clo_rec + __ldg(states + r0 + i));
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const float4 *r4 = reinterpret_cast<const float4 *>(s_root);
  const int4 *q4 = reinterpret_cast<const int4 *>(s_next);
  const int V4 = V >> 2;
  // Work unit = (row, column part): rows split into `split` parts balance
  // the warps when a CTA's row count is not a multiple of its warp count.
  const int W = blockDim.x >> 5, nu = n * split;
  int u = wib;
  int j = u / split, q = u - j * split;
  int4 rec = u < nu ? s_rec[j] : make_int4(0, 0, 0, 0);
  int4 e = (lane < rec.y) ? __ldg(t.clo + rec.x + lane) : make_int4(0, 0, 0, 0);
  for (; u < nu; u += W) {
    const int c0 = (V4 * q) / split, c1 = (V4 * (q + 1)) / split;
    const int v0 = 4 * c0, v1 = 4 * c1;
    // overrides of this part -> scratch + bitmap
    if (lane < rec.y && e.x >= v0 && e.x < v1) {
      ovs[e.x] = __int_as_float(e.z);
      ovn[e.x] = e.y;
      atomicOr(bm + (e.x >> 5), 1u << (e.x & 31));
    }
    for (int i = lane + 32; i < rec.y; i += 32) {
      const int4 e2 = __ldg(t.clo + rec.x + i);
      if (e2.x < v0 || e2.x >= v1) continue;
      ovs[e2.x] = __int_as_float(e2.z);
      ovn[e2.x] = e2.y;
      atomicOr(bm + (e2.x >> 5), 1u << (e2.x & 31));
    }
    // prefetch the next unit's record and first closure entries
    const int un = u + W;
    const int jn = un / split, qn = un - jn * split;
    const int4 nrec = un < nu ? s_rec[jn] : make_int4(0, 0, 0, 0);
    const int4 ne = (lane < nrec.y) ? __ldg(t.clo + nrec.x + lane) : make_int4(0, 0, 0, 0);
    __syncwarp();
    const float acc = __int_as_float(rec.z);
    const int64_t row = r0 + j;
    float4 *s4 = reinterpret_cast<float4 *>(scores + row * V);
    int4 *n4 = reinterpret_cast<int4 *>(next + row * V);
#pragma unroll 4
    for (int c = c0 + lane; c < c1; c += 32) {
      float4 r = r4[c];
      int4 qv = q4[c];
      r.x = acc + r.x;
      r.y = acc + r.y;
      r.z = acc + r.z;
      r.w = acc + r.w;
      const unsigned bits = (bm[c >> 3] >> ((c & 7) * 4)) & 0xFu;
      if (bits) {
        const int v = 4 * c;
        if (bits & 1u) { r.x = ovs[v]; qv.x = ovn[v]; }
        if (bits & 2u) { r.y = ovs[v + 1]; qv.y = ovn[v + 1]; }
        if (bits & 4u) { r.z = ovs[v + 2]; qv.z = ovn[v + 2]; }
        if (bits & 8u) { r.w = ovs[v + 3]; qv.w = ovn[v + 3]; }
      }
      __stcs(s4 + c, r);
      __stcs(n4 + c, qv);
    }
    __syncwarp();
    for (int w = (v0 >> 5) + lane; w < ((v1 + 31) >> 5); w += 32) bm[w] = 0u;
    __syncwarp();
    rec = nrec;
    e = ne;
    j = jn;
    q = qn;
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
// v7: one warp per CTA and `rows_per_cta` rows each, so the block scheduler
// balances rows across SMs dynamically (no static rows-per-warp imbalance);
// the dense root row is read through L1 (__ldg: 8 KB per SM, every CTA on
// the SM hits it), overrides by bitmap rank as in v6.
__global__ void __launch_bounds__(32)
    advance_v7_kernel(TableView t, const int32_t *__restrict__ states, int64_t B,
                      float *__restrict__ scores, int32_t *__restrict__ next, int rows_per_cta) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int V = t.vocab_size, Vw = (V + 31) >> 5;
  const int lane = threadIdx.x;
  unsigned *bm = reinterpret_cast<unsigned *>(smem);
  int *pre = reinterpret_cast<int *>(bm + Vw);
  for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t r0 = int64_t(blockIdx.x) * rows_per_cta;
  const int n = static_cast<int>(min(int64_t(rows_per_cta), B - r0));
  const float4 *r4 = reinterpret_cast<const float4 *>(t.root_scores);
  const int4 *q4 = reinterpret_cast<const int4 *>(t.root_next);
  const int V4 = V >> 2;
  int4 rec = n > 0 ? __ldg(t.clo_rec + __ldg(states + r0)) : make_int4(0, 0, 0, 0);
  int4 e = (lane < rec.y) ? __ldg(t.clo + rec.x + lane) : make_int4(0, 0, 0, 0);
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    if (j == n - 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane < rec.y) atomicOr(bm + (e.x >> 5), 1u << (e.x & 31));
    for (int i = lane + 32; i < rec.y; i += 32) {
      const int tok = __ldg(&t.clo[rec.x + i].x);
      atomicOr(bm + (tok >> 5), 1u << (tok & 31));
    }
    const int4 nrec = j + 1 < n ? __ldg(t.clo_rec + __ldg(states + r0 + j + 1)) : make_int4(0, 0, 0, 0);
    const int4 ne = (lane < nrec.y) ? __ldg(t.clo + nrec.x + lane) : make_int4(0, 0, 0, 0);
    __syncwarp();
    {
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
    __syncwarp();
    const float acc = __int_as_float(rec.z);
    const int64_t row = r0 + j;
    float4 *s4 = reinterpret_cast<float4 *>(scores + row * V);
    int4 *n4 = reinterpret_cast<int4 *>(next + row * V);
    const int4 *arcs = t.clo + rec.x;
#pragma unroll 4
    for (int c = lane; c < V4; c += 32) {
      float4 r = __ldg(r4 + c);
      int4 qv = __ldg(q4 + c);
      r.x = acc + r.x;
      r.y = acc + r.y;
      r.z = acc + r.z;
      r.w = acc + r.w;
      const unsigned word = bm[c >> 3];
      const int sh = (c & 7) * 4;
      const unsigned bits = (word >> sh) & 0xFu;
      if (bits) {
        int k = pre[c >> 3] + __popc(word & ((1u << sh) - 1u));
        if (bits & 1u) { const int4 a = __ldg(arcs + k++); r.x = __int_as_float(a.z); qv.x = a.y; }
        if (bits & 2u) { const int4 a = __ldg(arcs + k++); r.y = __int_as_float(a.z); qv.y = a.y; }
        if (bits & 4u) { const int4 a = __ldg(arcs + k++); r.z = __int_as_float(a.z); qv.z = a.y; }
        if (bits & 8u) { const int4 a = __ldg(arcs + k); r.w = __int_as_float(a.z); qv.w = a.y; }
      }
      __stcs(s4 + c, r);
      __stcs(n4 + c, qv);
    }
    __syncwarp();
    for (int w = lane; w < Vw; w += 32) bm[w] = 0u;
    __syncwarp();
    rec = nrec;
    e = ne;
  }
}

static int advance_variant() {
  const char *e = getenv("PGPB_ADVANCE_VARIANT");
  return e ? atoi(e) : 6;
}

using AdvFn = void (*)(TableView, const int32_t *, int64_t, float *, int32_t *);

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
  const int variant = chain ? 1 : advance_variant();
  if (variant == 6 && vec && smem_root) {
    const int Vw = (t.vocab_size + 31) >> 5;
    const size_t wbytes = (size_t(Vw) * 8 + 15) & ~size_t(15);
    // Geometry: 4 CTAs per SM (64 registers per thread); rows go to warps
    // round-robin inside a CTA, so pick the warp count (4..8) that divides
    // the CTA's rows most evenly (8192 rows: 14 per CTA on 7 warps, measured
    // best of the 3..6 x 4..8 grid).
    const char *e = getenv("PGPB_V6_CTAS");
    const char *ew = getenv("PGPB_V6_WARPS");
    const int per_sm = e ? std::max(1, atoi(e)) : 4;
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
      if (ew) W = std::max(1, std::min(kWarpsPerBlock, atoi(ew)));
    }
    int64_t ctas = int64_t(nsm) * per_sm;
    int rows = int((B + ctas - 1) / ctas);
    if (rows < 1) rows = 1;
    ctas = (B + rows - 1) / rows;
    // Row map: strided (every step of the grid writes one contiguous block
    // of rows) once each warp has >= 4 rows (65536 rows: 79.1% vs 77.2% of
    // the measured HBM peak); blocked below (8192 rows: equal within noise).
    // PGPB_V6_MAP=0/1 forces either (timing experiments).
    const int64_t J = (B + ctas * W - 1) / (ctas * W);  // rows per warp, strided
    const char *emap = getenv("PGPB_V6_MAP");
    const int strided = emap ? atoi(emap) : (J >= 4 ? 1 : 0);
    if (strided) rows = int(J * W);  // capacity per CTA: J steps of W rows
    const size_t rec_bytes = (size_t(rows) * 16 + 255) & ~size_t(255);
    const size_t smem6 = rec_bytes + root_bytes + size_t(kWarpsPerBlock) * wbytes;
    if (smem6 <= 200 * 1024) {
      if (smem6 > 48 * 1024)
        PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(advance_v6_kernel),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem6)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(unsigned(ctas));
      cfg.blockDim = dim3(32 * W);
      cfg.dynamicSmemBytes = smem6;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      const char *epdl = getenv("PGPB_ADVANCE_PDL");
      cfg.attrs = attr;
      cfg.numAttrs = (epdl && atoi(epdl) == 0) ? 0 : 1;
      // The table's ranked bitmap rows (when built, V <= 1024) instead of a
      // per-row bitmap build, for batches where a warp has at most one row:
      // it takes the build off the dependent startup chain (B=128: 4.35% vs
      // 3.87% of the HBM peak, B=1024: 29.4% vs 27.4%); with more rows per
      // warp the build overlaps the previous row's stream and the per-chunk
      // word shuffles cost more than the shared-memory reads (B=8192: 73.6%
      // vs 74.5%, 65536: 78.2% vs 80.0%).  V % 128 == 0: every lane runs
      // every chunk iteration, so the shuffles are warp-uniform.
      // PGPB_V6_TBITS=0/1 forces either (A/B).
      const char *etb = getenv("PGPB_V6_TBITS");
      const bool tb_ok = t.clo_bits && Vw <= 32 && t.vocab_size % 128 == 0;
      const int tbits = tb_ok ? (etb ? atoi(etb) : (rows <= W ? 1 : 0)) : 0;
      PGPB_CUDA_TRY(cudaLaunchKernelEx(&cfg, advance_v6_kernel, t, d_states, B, d_scores, d_next, rows, strided,
                                       tbits));
      PGPB_CUDA_TRY(cudaGetLastError());
      return PGPB_OK;
    }
  }
  if (variant == 7 && vec) {
    const int Vw = (t.vocab_size + 31) >> 5;
    const char *e = getenv("PGPB_V7_ROWS");
    const int rows = e ? std::max(1, atoi(e)) : 2;
    const int64_t ctas = (B + rows - 1) / rows;
    const size_t smem7 = size_t(Vw) * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(ctas));
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem7;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    const char *epdl = getenv("PGPB_ADVANCE_PDL");
    cfg.attrs = attr;
    cfg.numAttrs = (epdl && atoi(epdl) == 0) ? 0 : 1;
    PGPB_CUDA_TRY(cudaLaunchKernelEx(&cfg, advance_v7_kernel, t, d_states, B, d_scores, d_next, rows));
    PGPB_CUDA_TRY(cudaGetLastError());
    return PGPB_OK;
  }
  if ((variant == 5 || variant == 6) && vec && smem_root) {
    const int Vw = (t.vocab_size + 31) >> 5;
    const size_t wbytes = size_t(t.vocab_padded) * 8 + ((size_t(Vw) * 4 + 15) & ~size_t(15));
    const char *e = getenv("PGPB_V5_CTAS");
    int per_sm = e ? atoi(e) : 3;
    int W = kWarpsPerBlock;
    for (;;) {
      int64_t ctas = int64_t(nsm) * per_sm;
      int rows = int((B + ctas - 1) / ctas);
      if (rows < 1) rows = 1;
      ctas = (B + rows - 1) / rows;
      const size_t rec_bytes = (size_t(rows) * 16 + 255) & ~size_t(255);
      const size_t smem5 = rec_bytes + root_bytes + size_t(W) * wbytes;
      if (smem5 * per_sm <= 224 * 1024 || (per_sm == 1 && smem5 <= 224 * 1024)) {
        PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(advance_v5_kernel),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem5)));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(ctas));
        cfg.blockDim = dim3(32 * W);
        cfg.dynamicSmemBytes = smem5;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        const char *epdl = getenv("PGPB_ADVANCE_PDL");
        cfg.attrs = attr;
        cfg.numAttrs = (epdl && atoi(epdl) == 0) ? 0 : 1;
        // column parts per row: balance rows over the W warps of a CTA
        int split = 1;  // column parts per row (measured: 1 is fastest at 8192 x 1024)
        if (const char *es = getenv("PGPB_V5_SPLIT")) split = std::max(1, atoi(es));
        PGPB_CUDA_TRY(cudaLaunchKernelEx(&cfg, advance_v5_kernel, t, d_states, B, d_scores, d_next, rows, split));
        PGPB_CUDA_TRY(cudaGetLastError());
        return PGPB_OK;
      }
      if (per_sm > 1) --per_sm;
      else if (W > 1) --W;
      else break;
    }
  }
  if (variant == 3 && vec) {
    // warps per CTA limited by the per-warp double buffer (2 rows of V*8 B)
    const size_t per_warp = 2 * root_bytes;
    int warps = int((200 * 1024 - root_bytes) / per_warp);
    if (const char *e = getenv("PGPB_V3_WARPS")) warps = std::min(warps, atoi(e));
    warps = warps < 1 ? 1 : (warps > kWarpsPerBlock ? kWarpsPerBlock : warps);
    const size_t smem3 = root_bytes + size_t(warps) * per_warp;
    if (smem3 <= 227 * 1024) {
      PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(advance_v3_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem3)));
      int64_t g = (B + warps - 1) / warps;
      const int per_sm3 = std::max(1, int((227 * 1024) / (smem3 + 1024)));
      if (g > int64_t(nsm) * per_sm3) g = int64_t(nsm) * per_sm3;
      advance_v3_kernel<<<unsigned(g), kThreads, smem3, st>>>(t, d_states, B, d_scores, d_next, warps);
      PGPB_CUDA_TRY(cudaGetLastError());
      return PGPB_OK;
    }
  }
  if (variant >= 2) {
    // v2: ~4 resident CTAs per SM, contiguous row chunks
    int64_t ctas = int64_t(nsm) * 4;
    int rows = int((B + ctas - 1) / ctas);
    if (rows < 1) rows = 1;
    ctas = (B + rows - 1) / rows;
    const size_t rec_bytes = (size_t(rows) * 16 + 255) & ~size_t(255);
    const size_t smem2 = rec_bytes + (smem_root ? root_bytes : 0);
    if (smem2 <= 200 * 1024) {
      auto fn2 = vec ? (smem_root ? advance_v2_kernel<true, true> : advance_v2_kernel<true, false>)
                     : (smem_root ? advance_v2_kernel<false, true> : advance_v2_kernel<false, false>);
      if (smem2 > 48 * 1024) {
        PGPB_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn2),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      }
      fn2<<<unsigned(ctas), kThreads, smem2, st>>>(t, d_states, B, d_scores, d_next, rows);
      PGPB_CUDA_TRY(cudaGetLastError());
      return PGPB_OK;
    }
  }
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
  fn<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(t, d_states, B, d_scores, d_next);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
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
