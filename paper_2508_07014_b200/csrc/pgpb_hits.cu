// Phrase-hit counting on the GPU (pgpb_phrase_hits).
//
// Reference: evaluation.keyphrase_hits / count_occurrences
// (evaluation.py:90-134): for every utterance and phrase, the number of
// (overlapping) occurrences of the phrase's word tuple in the reference and
// in the hypothesis word lists.  The Python reference loops utterances x
// phrases x positions; here the phrases are compiled once into the same
// Aho-Corasick table the boosting path uses (token = word id), and one
// thread walks one word sequence through the automaton: after each word
// the phrases ending there are exactly the outputs of the current state
// (every phrase whose end node is on the state's failure chain, flattened
// on the host into out_start/out_len/out_phrase).  Occurrences are emitted
// as 64-bit keys phrase * n_seqs + seq; per-utterance clipping (tp =
// sum_u min(ref_u, hyp_u)) is a sort/segment step on the keys.
//
// Two passes over the same walk: d_keys == NULL counts occurrences per
// sequence into d_counts; otherwise keys are written at d_key_offsets[seq].

#include <string>

#include "pgpb_common.cuh"

namespace pgpb {

// Successor of (off, st) on token w: the state's first-hit arc if w is on its
// closure (bitmap word; the entry's index is the word's rank plus the closure
// tokens below w in it), otherwise the root row.  Without bitmaps: binary
// search of the token-sorted arcs.
__device__ __forceinline__ void ac_next(const TableView &t, int &off, int &st, int w) {
  const int4 *b = t.blob + off;
  if (t.clo_bits) {
    const uint2 cw = __ldg(t.clo_bits + int64_t(st) * t.bits_words + (w >> 5));
    if ((cw.x >> (w & 31)) & 1u) {
      const int4 e = __ldg(b + 1 + cw.y + __popc(cw.x & ((1u << (w & 31)) - 1u)));
      off = e.w;
      st = e.y;
      return;
    }
  } else {
    int lo = 0, hi = __ldg(&b->x) - 1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int4 e = __ldg(b + 1 + mid);
      if (e.x == w) {
        off = e.w;
        st = e.y;
        return;
      }
      if (e.x < w)
        lo = mid + 1;
      else
        hi = mid - 1;
    }
  }
  off = __ldg(t.root_next_off + w);
  st = __ldg(t.root_next + w);
}

__global__ void __launch_bounds__(kThreads)
    phrase_hits_kernel(TableView t, const int32_t *__restrict__ words, const int64_t *__restrict__ offsets,
                       int64_t n_seqs, const int32_t *__restrict__ out_start, const int32_t *__restrict__ out_len,
                       const int32_t *__restrict__ out_phrase, int32_t *__restrict__ counts,
                       int64_t *__restrict__ keys, const int64_t *__restrict__ key_offsets) {
  const int root_off = __ldg(t.blob_off);
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n_seqs;
       q += int64_t(gridDim.x) * blockDim.x) {
    int off = root_off, st = 0;
    int32_t n = 0;
    int64_t kpos = keys ? __ldg(key_offsets + q) : 0;
    for (int64_t i = __ldg(offsets + q), e = __ldg(offsets + q + 1); i < e; ++i) {
      const int w = __ldg(words + i);
      ac_next(t, off, st, w);
      const int len = __ldg(out_len + st);
      if (len) {
        if (keys) {
          const int s0 = __ldg(out_start + st);
          for (int k = 0; k < len; ++k) keys[kpos++] = int64_t(__ldg(out_phrase + s0 + k)) * n_seqs + q;
        }
        n += len;
      }
    }
    if (!keys) counts[q] = n;
  }
}

}  // namespace pgpb

extern "C" int pgpb_phrase_hits(const pgpb_table *table, const int32_t *d_words, const int64_t *d_offsets,
                                int64_t n_seqs, const int32_t *d_out_start, const int32_t *d_out_len,
                                const int32_t *d_out_phrase, int32_t *d_counts, int64_t *d_keys,
                                const int64_t *d_key_offsets, void *stream) {
  using namespace pgpb;
  if (!table) return fail(PGPB_EINVAL, "table is NULL");
  if (n_seqs < 0) return fail(PGPB_EINVAL, "n_seqs must be >= 0");
  if (n_seqs == 0) return PGPB_OK;
  if (!d_offsets || !d_out_start || !d_out_len || (!d_keys && !d_counts) || (d_keys && !d_key_offsets))
    return fail(PGPB_EINVAL, "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n_seqs + kThreads - 1) / kThreads;
  const int64_t cap = int64_t(sm_count(current_device())) * 8;
  phrase_hits_kernel<<<unsigned(blocks < cap ? blocks : cap), kThreads, 0, st>>>(
      table->view, d_words, d_offsets, n_seqs, d_out_start, d_out_len, d_out_phrase, d_counts, d_keys, d_key_offsets);
  PGPB_CUDA_TRY(cudaGetLastError());
  return PGPB_OK;
}
