// Internal declarations shared by the pgpb translation units.
#pragma once

#include <cstdint>
#include <exception>
#include <new>
#include <string>

#include <cuda_runtime.h>

#include "pgpb.h"

namespace pgpb {

// Code-path overrides for tests (pgpb_set_tuning): 0 = automatic choice.
// Every override selects between equivalent, bit-exact code paths; none
// changes results.  Read on the host at launch time (no getenv).
struct Tuning {
  int ctc_consumers = 0;  // walker warps per CTA (1..7)
  int ctc_segment = 0;    // frames per walker segment
  int ctc_seq = 0;        // 1 = sequential walk, 2 = speculative rounds only
  int ll_warps = 0;       // label-loop step: warps (rows) per CTA
  int beam_blobs = 0;     // device beams: 0 advance blobs when built, 1 closure records + bitmap marking
  int adv_compact = 0;    // chained advance table layout: 0 by regime, 1 ranked bitmap, 2 compact arrays, 3 blobs
  int cb_threads = 0;     // device CTC beam: threads per CTA (0 = by beam width)
};
Tuning &tuning();

// Thread-local last-error message (pgpb_last_error).
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

// Device view of a compiled table.  All arrays live in one cudaMalloc arena;
// every sub-array starts on a 256-byte boundary, so int4/float4 loads are
// aligned.  Layout rationale: DESIGN.md §3.
struct TableView {
  int32_t num_states;
  int32_t vocab_size;
  int32_t vocab_padded;        // V rounded up to a multiple of 4
  int32_t num_arcs;
  float unk_score;
  float max_root_score;
  float typ_gain;              // max over the root's children of (best closure score - best dense score)
  const float *root_scores;    // [Vp] f32: unk background, root arcs on top (table.py:74-81)
  const int32_t *root_next;    // [Vp]
  const int4 *state_rec;       // [S] {arc_start, arc_end, backoff_to, bits(backoff_weight)}
  const int4 *arcs;            // [A] {token, to, bits(weight), 0}, sorted by (from, token)
  const int4 *clo_rec;         // [S] {clo_start, clo_count, bits(acc_total), is_final}
  const int4 *clo;             // [C] {token, next, bits(score), 0}: flattened first-hit arcs
  const float *final_score;    // [S]
  // Linked-automaton layout for the sequential decoders: per state s, at
  // blob[blob_off[s]] a header {count, bits(acc_total), s, 0} followed by
  // its `count` closure entries {token, next, bits(score), blob_off[next]},
  // so a decoder that knows the blob offset of its current state resolves
  // it with one contiguous load and carries the successor's offset along.
  const int4 *blob;            // [S + C]
  const int32_t *blob_off;     // [S]
  const int32_t *root_next_off;  // [Vp] blob_off[root_next[v]]
  // Per state: bitmap of its closure tokens (Vw = ceil(V/32) words per
  // state), each word paired with the number of closure tokens below it, so
  // a decoder tests "is v a first-hit arc of s" with one 8-byte load and,
  // when it is, finds v's entry at blob[blob_off[s] + 1 + rank] (rank = the
  // word's count + popc of the lower bits) without a search; NULL when
  // S * Vw pairs would exceed the cap.  The blob header's 4th field holds the
  // state's largest closure-arc score (bits of an f32, -inf when empty).
  const uint2 *clo_bits;       // [S][Vw] {bits, closure tokens in words < w}
  int32_t bits_words;          // Vw
  // Advance-only compact copies (V <= 1024, else NULL): the closure bitmap
  // as plain words (one 128-byte line per state; a warp derives the ranks
  // with a popc scan) and the closure entries as {next, bits(score)} pairs
  // (clo without the token, which the bitmap rank already locates).  They
  // halve the table bytes a uniformly random row pulls from HBM.
  const uint32_t *adv_bits;    // [S][Vw]
  const int2 *adv_clo;         // [C]
  // Per-state advance blob, fixed stride (adv_stride16 x 16 B; NULL when
  // V > 1024 or a closure does not fit): int32 [0] bits(acc_total),
  // [1] closure count, [2..3] 0, [4, 4 + Vw) closure words, then Vw u16 word
  // ranks, then the closure's {next | count(next) << 25, bits(score)} pairs
  // (8-B aligned, at int32 index adv_ent0).  One warp-wide 16-B-per-lane copy
  // of its used prefix brings a state's whole advance operand set.
  const int4 *adv_blob;        // [S][adv_stride16]
  const uint8_t *adv_root_cnt; // [Vp] closure count of root_next[v] (sizes a dense successor's blob copy)
  int32_t adv_stride16;
  int32_t adv_ent0;
};

}  // namespace pgpb

struct pgpb_table {
  pgpb::TableView view;
  void *arena = nullptr;
  int64_t arena_bytes = 0;
  int32_t device = 0;
  int32_t max_chain = 0;
  int64_t closure_entries = 0;
  int32_t max_closure = 0;
};

// Host exceptions (std::bad_alloc from sizing vectors on untrusted input,
// std::length_error, ...) must not cross the C ABI: every entry point that
// allocates host containers runs its body through pgpb::guarded.
namespace pgpb {
template <typename F>
int guarded(F &&body) {
  try {
    return body();
  } catch (const std::bad_alloc &) {
    return fail(PGPB_ENOMEM, "host allocation failed");
  } catch (const std::exception &ex) {
    return fail(PGPB_EINVAL, std::string("internal error: ") + ex.what());
  } catch (...) {
    return fail(PGPB_EINVAL, "internal error");
  }
}
}  // namespace pgpb

#define PGPB_CUDA_TRY(expr)                                                           \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return ::pgpb::fail(PGPB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)
