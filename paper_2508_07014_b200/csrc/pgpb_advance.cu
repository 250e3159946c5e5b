// Advance kernel: scores[B,V], next[B,V] for a batch of tree states.
//
// Reference: _kernels.score_batch (_kernels.pyx:30-72), R5 in SURVEY.md.
// HBM-write-bound (8 B written per cell).  One warp per row,
// rows grid-strided over a persistent grid; the dense root row is staged in
// shared memory once per CTA; every row is written with 16-byte streaming
// stores (st.global.cs.v4) shifted by the state's accumulated backoff, then
// the state's flattened first-hit arcs are scattered on top.  __syncwarp()
// orders the scatter after the dense stores of the same warp.

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

static int g_sm_count[64] = {0};

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
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
