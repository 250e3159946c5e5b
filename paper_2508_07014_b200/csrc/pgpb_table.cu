// Device-resident compiled table: validation, flattened backoff closure and
// the packed HBM layout.
//
// The reference resolves a cell by walking the failure chain of the query
// state (_kernels.pyx:56-71).  Chains are short but every level is a
// dependent load, so besides the packed chain arrays we precompute, once per
// table, each state's *closure*: the first-hit arcs along its whole chain
// with their fp32 scores accumulated exactly as the reference does
// (acc = acc + backoff_weight[s], in chain order) plus the final acc.  One
// (record, entries) load pair then resolves any state.

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pgpb_internal.h"

namespace {

inline int32_t f2i(float f) {
  int32_t i;
  std::memcpy(&i, &f, 4);
  return i;
}

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// Largest vocabulary a device table accepts: the dense root row (8 B per
// token) is staged per CTA or read per row by every kernel; 2^26 tokens is
// far beyond any tokenizer and keeps every size computation inside int32.
constexpr int32_t kMaxVocab = 1 << 26;

}  // namespace

extern "C" {

static int pgpb_table_create_impl(int32_t S, int32_t V, int32_t A, const int32_t *arc_token,
                      const int32_t *arc_to, const float *arc_weight,
                      const int32_t *state_start, const int32_t *state_end,
                      const int32_t *backoff_to, const float *backoff_weight,
                      const uint8_t *is_final, const float *final_score, float unk_score,
                      int32_t device, pgpb_table **out) {
  using pgpb::fail;
  if (!out) return fail(PGPB_EINVAL, "out is NULL");
  *out = nullptr;
  if (S < 1 || V < 1) return fail(PGPB_EFORMAT, "need at least 1 state and 1 token");
  if (A < 0) return fail(PGPB_EFORMAT, "negative arc count");
  if (V > kMaxVocab)
    return fail(PGPB_EFORMAT, "vocab_size " + std::to_string(V) + " exceeds the device table limit " +
                                  std::to_string(kMaxVocab));
  // Structural checks the kernels rely on (subset of table.py:87-127).
  for (int32_t s = 0; s < S; ++s) {
    if (state_start[s] < 0 || state_start[s] > state_end[s] || state_end[s] > A)
      return fail(PGPB_EFORMAT, "state " + std::to_string(s) + ": bad arc range");
    if (backoff_to[s] < 0 || backoff_to[s] >= S)
      return fail(PGPB_EFORMAT, "backoff_to out of range");
  }
  for (int32_t j = 0; j < A; ++j) {
    if (arc_token[j] < 0 || arc_token[j] >= V) return fail(PGPB_EFORMAT, "arc_token out of range");
    if (arc_to[j] < 0 || arc_to[j] >= S) return fail(PGPB_EFORMAT, "arc_to out of range");
  }
  if (backoff_to[0] != 0) return fail(PGPB_EFORMAT, "root backoff must be (0, 0)");

  const int32_t Vp = (V + 3) & ~3;
  // Dense root row (table.py:74-81).
  std::vector<float> root_scores(static_cast<size_t>(Vp), unk_score);
  std::vector<int32_t> root_next(static_cast<size_t>(Vp), 0);
  for (int32_t j = state_start[0]; j < state_end[0]; ++j) {
    root_scores[arc_token[j]] = arc_weight[j];
    root_next[arc_token[j]] = arc_to[j];
  }
  float max_root = root_scores[0];
  for (int32_t v = 1; v < V; ++v) max_root = std::max(max_root, root_scores[v]);

  std::vector<int4> state_rec(static_cast<size_t>(S));
  for (int32_t s = 0; s < S; ++s)
    state_rec[s] = make_int4(state_start[s], state_end[s], backoff_to[s], f2i(backoff_weight[s]));
  std::vector<int4> arcs(static_cast<size_t>(std::max(A, 1)));
  for (int32_t j = 0; j < A; ++j) arcs[j] = make_int4(arc_token[j], arc_to[j], f2i(arc_weight[j]), 0);

  // Flattened closure, R5 of SURVEY appendix / _kernels.pyx:56-67:
  // walk the chain, first hit per token wins, fp32 acc in chain order.
  std::vector<int4> clo_rec(static_cast<size_t>(S));
  std::vector<int4> clo;
  clo.reserve(static_cast<size_t>(A) * 3 + 16);
  std::vector<int32_t> stamp(static_cast<size_t>(V), -1);
  std::vector<int4> tmp;
  int32_t max_chain = 0, max_clo = 0;
  for (int32_t s0 = 0; s0 < S; ++s0) {
    tmp.clear();
    float acc = 0.0f;
    int32_t s = s0, steps = 0;
    while (s != 0) {
      if (++steps > S) return fail(PGPB_EFORMAT, "backoff chain does not reach the root");
      for (int32_t j = state_start[s]; j < state_end[s]; ++j) {
        const int32_t v = arc_token[j];
        if (stamp[v] != s0) {
          stamp[v] = s0;
          const float sc = acc + arc_weight[j];
          tmp.push_back(make_int4(v, arc_to[j], f2i(sc), 0));
        }
      }
      acc = acc + backoff_weight[s];
      s = backoff_to[s];
    }
    std::sort(tmp.begin(), tmp.end(), [](const int4 &a, const int4 &b) { return a.x < b.x; });
    max_chain = std::max(max_chain, steps);
    max_clo = std::max(max_clo, static_cast<int32_t>(tmp.size()));
    if (clo.size() + tmp.size() > static_cast<size_t>(INT32_MAX))
      return fail(PGPB_ENOMEM, "closure exceeds 2^31 entries");
    clo_rec[s0] = make_int4(static_cast<int32_t>(clo.size()), static_cast<int32_t>(tmp.size()),
                            f2i(acc), is_final ? static_cast<int32_t>(is_final[s0] != 0) : 0);
    clo.insert(clo.end(), tmp.begin(), tmp.end());
  }
  const int64_t C = static_cast<int64_t>(clo.size());
  if (clo.empty()) clo.push_back(make_int4(0, 0, 0, 0));

  // Blob layout (pgpb_internal.h): header + entries per state, entries carry
  // the successor's blob offset.
  std::vector<int32_t> boff(static_cast<size_t>(S));
  {
    int64_t o = 0;
    for (int32_t s0 = 0; s0 < S; ++s0) {
      boff[s0] = static_cast<int32_t>(o);
      o += 1 + clo_rec[s0].y;
    }
    if (o > INT32_MAX) return fail(PGPB_ENOMEM, "blob exceeds 2^31 entries");
  }
  // +64 zero entries of padding: warp-wide loads read up to 64 entries past a header
  std::vector<int4> blob(static_cast<size_t>(S) + static_cast<size_t>(C) + 64, make_int4(0, 0, 0, 0));
  for (int32_t s0 = 0; s0 < S; ++s0) {
    const int4 r = clo_rec[s0];
    int4 *b = blob.data() + boff[s0];
    float smax = -INFINITY;
    for (int32_t i = 0; i < r.y; ++i) {
      const int4 e = clo[static_cast<size_t>(r.x) + i];
      b[1 + i] = make_int4(e.x, e.y, e.z, boff[e.y]);
      float sc;
      std::memcpy(&sc, &e.z, 4);
      smax = std::max(smax, sc);
    }
    b[0] = make_int4(r.y, r.z, s0, f2i(smax));
  }
  // Closure-token bitmaps with per-word ranks (capped at 1 GiB).
  const int32_t Vw = (V + 31) / 32;
  const bool with_bits = int64_t(S) * Vw * 8 <= (int64_t(1) << 30);
  std::vector<uint32_t> bits(with_bits ? static_cast<size_t>(S) * Vw * 2 : 2, 0u);
  if (with_bits)
    for (int32_t s0 = 0; s0 < S; ++s0) {
      const int4 r = clo_rec[s0];
      uint32_t *w = bits.data() + static_cast<size_t>(s0) * Vw * 2;
      for (int32_t i = 0; i < r.y; ++i) {
        const int32_t v = clo[static_cast<size_t>(r.x) + i].x;
        w[2 * (v >> 5)] |= 1u << (v & 31);
      }
      uint32_t below = 0;
      for (int32_t k = 0; k < Vw; ++k) {
        w[2 * k + 1] = below;
        below += static_cast<uint32_t>(__builtin_popcount(w[2 * k]));
      }
    }
  // advance-only compact copies (pgpb_internal.h)
  const bool with_adv = with_bits && Vw <= 32;
  std::vector<uint32_t> adv_bits(with_adv ? static_cast<size_t>(S) * Vw : 1, 0u);
  if (with_adv)
    for (size_t i = 0; i < static_cast<size_t>(S) * Vw; ++i) adv_bits[i] = bits[2 * i];
  std::vector<int2> adv_clo(clo.size());
  for (size_t i = 0; i < clo.size(); ++i) adv_clo[i] = make_int2(clo[i].y, clo[i].z);
  // fixed-stride advance blobs (pgpb_internal.h)
  const int32_t ent0 = ((4 + Vw + (Vw + 1) / 2) + 1) & ~1;  // int32 index of the pairs, 8-B aligned
  const int64_t blob_i32 = (int64_t(ent0) + 2 * int64_t(max_clo) + 31) / 32 * 32;  // 128-B multiple
  // entries carry the successor's closure count in next's top bits (so a
  // copy can be sized before the blob arrives): S < 2^25, counts < 2^6
  const bool with_blob = with_adv && blob_i32 <= 256 && int64_t(S) * blob_i32 * 4 <= (int64_t(1) << 30) &&
                         S < (1 << 25) && max_clo < 64;
  std::vector<int32_t> adv_blob(with_blob ? static_cast<size_t>(S) * blob_i32 : 4, 0);
  if (with_blob)
    for (int32_t s0 = 0; s0 < S; ++s0) {
      int32_t *w = adv_blob.data() + static_cast<size_t>(s0) * blob_i32;
      const int4 r = clo_rec[s0];
      w[0] = r.z;
      w[1] = r.y;
      uint16_t *rk = reinterpret_cast<uint16_t *>(w + 4 + Vw);
      for (int32_t k = 0; k < Vw; ++k) {
        w[4 + k] = static_cast<int32_t>(bits[2 * (static_cast<size_t>(s0) * Vw + k)]);
        rk[k] = static_cast<uint16_t>(bits[2 * (static_cast<size_t>(s0) * Vw + k) + 1]);
      }
      for (int32_t i = 0; i < r.y; ++i) {
        const int4 e = clo[static_cast<size_t>(r.x) + i];
        w[ent0 + 2 * i] = e.y | (clo_rec[e.y].y << 25);
        w[ent0 + 2 * i + 1] = e.z;
      }
    }
  std::vector<uint8_t> root_cnt(static_cast<size_t>(Vp), 0);
  if (with_blob)
    for (int32_t v = 0; v < V; ++v) root_cnt[v] = static_cast<uint8_t>(clo_rec[root_next[v]].y);
  std::vector<int32_t> rn_off(static_cast<size_t>(Vp), 0);
  for (int32_t v = 0; v < Vp; ++v) rn_off[v] = boff[root_next[v]];

  std::vector<float> fscore(static_cast<size_t>(S), 0.0f);
  if (final_score) std::copy(final_score, final_score + S, fscore.begin());

  // One arena, 256-byte aligned sub-arrays.
  int64_t off = 0;
  auto place = [&](int64_t bytes) {
    int64_t o = off;
    off = align256(off + bytes);
    return o;
  };
  const int64_t o_rs = place(int64_t(Vp) * 4), o_rn = place(int64_t(Vp) * 4);
  const int64_t o_sr = place(int64_t(S) * 16), o_arc = place(int64_t(arcs.size()) * 16);
  const int64_t o_cr = place(int64_t(S) * 16), o_clo = place(int64_t(clo.size()) * 16);
  const int64_t o_fs = place(int64_t(S) * 4);
  const int64_t o_blob = place(int64_t(blob.size()) * 16);
  const int64_t o_boff = place(int64_t(S) * 4);
  const int64_t o_rno = place(int64_t(Vp) * 4);
  const int64_t o_bits = place(int64_t(bits.size()) * 4);
  const int64_t o_abits = place(int64_t(adv_bits.size()) * 4);
  const int64_t o_aclo = place(int64_t(adv_clo.size()) * 8);
  const int64_t o_ablob = place(int64_t(adv_blob.size()) * 4);
  const int64_t o_rcnt = place(int64_t(Vp));
  const int64_t total = off;

  int prev_dev = 0;
  PGPB_CUDA_TRY(cudaGetDevice(&prev_dev));
  PGPB_CUDA_TRY(cudaSetDevice(device));
  char *arena = nullptr;
  cudaError_t e = cudaMalloc(&arena, static_cast<size_t>(total));
  if (e != cudaSuccess) {
    cudaSetDevice(prev_dev);
    return fail(PGPB_ENOMEM, std::string("cudaMalloc(table): ") + cudaGetErrorString(e));
  }
  std::vector<char> staging(static_cast<size_t>(total), 0);
  std::memcpy(staging.data() + o_rs, root_scores.data(), size_t(Vp) * 4);
  std::memcpy(staging.data() + o_rn, root_next.data(), size_t(Vp) * 4);
  std::memcpy(staging.data() + o_sr, state_rec.data(), size_t(S) * 16);
  std::memcpy(staging.data() + o_arc, arcs.data(), arcs.size() * 16);
  std::memcpy(staging.data() + o_cr, clo_rec.data(), size_t(S) * 16);
  std::memcpy(staging.data() + o_clo, clo.data(), clo.size() * 16);
  std::memcpy(staging.data() + o_fs, fscore.data(), size_t(S) * 4);
  std::memcpy(staging.data() + o_blob, blob.data(), blob.size() * 16);
  std::memcpy(staging.data() + o_boff, boff.data(), size_t(S) * 4);
  std::memcpy(staging.data() + o_rno, rn_off.data(), size_t(Vp) * 4);
  std::memcpy(staging.data() + o_bits, bits.data(), bits.size() * 4);
  std::memcpy(staging.data() + o_abits, adv_bits.data(), adv_bits.size() * 4);
  std::memcpy(staging.data() + o_aclo, adv_clo.data(), adv_clo.size() * 8);
  std::memcpy(staging.data() + o_ablob, adv_blob.data(), adv_blob.size() * 4);
  std::memcpy(staging.data() + o_rcnt, root_cnt.data(), size_t(Vp));
  e = cudaMemcpy(arena, staging.data(), static_cast<size_t>(total), cudaMemcpyHostToDevice);
  cudaSetDevice(prev_dev);
  if (e != cudaSuccess) {
    cudaFree(arena);
    return fail(PGPB_ECUDA, std::string("cudaMemcpy(table): ") + cudaGetErrorString(e));
  }

  auto *t = new pgpb_table();
  t->arena = arena;
  t->arena_bytes = total;
  t->device = device;
  t->max_chain = max_chain;
  t->closure_entries = C;
  t->max_closure = max_clo;
  pgpb::TableView &v = t->view;
  v.num_states = S;
  v.vocab_size = V;
  v.vocab_padded = Vp;
  v.num_arcs = A;
  v.unk_score = unk_score;
  v.max_root_score = max_root;
  {  // typical advantage of a first-hit arc over the dense row (depth-1 states)
    float g = 0.0f;
    for (int32_t j = state_start[0]; j < state_end[0]; ++j) {
      const int4 r = clo_rec[arc_to[j]];
      float acc, smax = -INFINITY;
      std::memcpy(&acc, &r.z, 4);
      for (int32_t i = 0; i < r.y; ++i) {
        float sc;
        std::memcpy(&sc, &clo[static_cast<size_t>(r.x) + i].z, 4);
        smax = std::max(smax, sc);
      }
      if (r.y > 0) g = std::max(g, smax - (acc + max_root));
    }
    v.typ_gain = g;
  }
  v.root_scores = reinterpret_cast<const float *>(arena + o_rs);
  v.root_next = reinterpret_cast<const int32_t *>(arena + o_rn);
  v.state_rec = reinterpret_cast<const int4 *>(arena + o_sr);
  v.arcs = reinterpret_cast<const int4 *>(arena + o_arc);
  v.clo_rec = reinterpret_cast<const int4 *>(arena + o_cr);
  v.clo = reinterpret_cast<const int4 *>(arena + o_clo);
  v.final_score = reinterpret_cast<const float *>(arena + o_fs);
  v.blob = reinterpret_cast<const int4 *>(arena + o_blob);
  v.blob_off = reinterpret_cast<const int32_t *>(arena + o_boff);
  v.root_next_off = reinterpret_cast<const int32_t *>(arena + o_rno);
  v.clo_bits = with_bits ? reinterpret_cast<const uint2 *>(arena + o_bits) : nullptr;
  v.bits_words = Vw;
  v.adv_bits = with_adv ? reinterpret_cast<const uint32_t *>(arena + o_abits) : nullptr;
  v.adv_clo = reinterpret_cast<const int2 *>(arena + o_aclo);
  v.adv_blob = with_blob ? reinterpret_cast<const int4 *>(arena + o_ablob) : nullptr;
  v.adv_stride16 = with_blob ? int32_t(blob_i32 / 4) : 0;
  v.adv_root_cnt = reinterpret_cast<const uint8_t *>(arena + o_rcnt);
  v.adv_ent0 = ent0;
  *out = t;
  return PGPB_OK;
}

int pgpb_table_create(int32_t S, int32_t V, int32_t A, const int32_t *arc_token,
                      const int32_t *arc_to, const float *arc_weight,
                      const int32_t *state_start, const int32_t *state_end,
                      const int32_t *backoff_to, const float *backoff_weight,
                      const uint8_t *is_final, const float *final_score, float unk_score,
                      int32_t device, pgpb_table **out) {
  return pgpb::guarded([&] { return pgpb_table_create_impl(S, V, A, arc_token, arc_to, arc_weight, state_start, state_end, backoff_to, backoff_weight, is_final, final_score, unk_score, device, out); });
}

// GPB1 (table.py:16-29 of the reference; little-endian): header
// "<4sIIIIf" = magic, version=1, S, V, A, unk_score, then arc_from,
// arc_token, arc_to (i32[A]), arc_weight (f32[A]), state_start, state_end,
// backoff_to (i32[S]), backoff_weight (f32[S]), is_final (u8[S]),
// final_score (f32[S]).  Parsed and validated on the host (the reference's
// ArcTable.validate invariants, table.py:87-127), then the device arena is
// built directly: no intermediate Python arrays.
static int pgpb_table_load_gpb1_impl(const void *data, int64_t size, int32_t device, pgpb_table **out) {
  using pgpb::fail;
  if (!out) return fail(PGPB_EINVAL, "out is NULL");
  *out = nullptr;
  if (!data && size) return fail(PGPB_EINVAL, "data is NULL");
  const unsigned char *b = static_cast<const unsigned char *>(data);
  const int64_t hdr = 24;
  if (size < hdr) return fail(PGPB_EFORMAT, "truncated header");
  if (std::memcmp(b, "GPB1", 4) != 0) return fail(PGPB_EFORMAT, "bad magic");
  uint32_t version, S, V, A;
  float unk;
  std::memcpy(&version, b + 4, 4);
  std::memcpy(&S, b + 8, 4);
  std::memcpy(&V, b + 12, 4);
  std::memcpy(&A, b + 16, 4);
  std::memcpy(&unk, b + 20, 4);
  if (version != 1) return fail(PGPB_EFORMAT, "unsupported version " + std::to_string(version));
  if (S > uint32_t(INT32_MAX) || V > uint32_t(INT32_MAX) || A > uint32_t(INT32_MAX))
    return fail(PGPB_EFORMAT, "counts exceed int32");
  if (V > uint32_t(kMaxVocab))
    return fail(PGPB_EFORMAT, "vocab_size " + std::to_string(V) + " exceeds the device table limit " +
                                  std::to_string(kMaxVocab));
  const int64_t expected = hdr + int64_t(A) * 16 + int64_t(S) * 21;
  if (size != expected)
    return fail(PGPB_EFORMAT, "expected " + std::to_string(expected) + " bytes, found " + std::to_string(size));
  // copy out (the arrays are unaligned inside the file)
  int64_t off = hdr;
  auto take_i32 = [&](int64_t n) {
    std::vector<int32_t> v(static_cast<size_t>(n));
    if (n) std::memcpy(v.data(), b + off, size_t(n) * 4);
    off += n * 4;
    return v;
  };
  auto take_f32 = [&](int64_t n) {
    std::vector<float> v(static_cast<size_t>(n));
    if (n) std::memcpy(v.data(), b + off, size_t(n) * 4);
    off += n * 4;
    return v;
  };
  const std::vector<int32_t> arc_from = take_i32(A), arc_token = take_i32(A), arc_to = take_i32(A);
  const std::vector<float> arc_weight = take_f32(A);
  const std::vector<int32_t> state_start = take_i32(S), state_end = take_i32(S), backoff_to = take_i32(S);
  const std::vector<float> backoff_weight = take_f32(S);
  std::vector<uint8_t> is_final(static_cast<size_t>(S));  // normalised to 0/1 below
  if (S) std::memcpy(is_final.data(), b + off, S);
  off += S;
  const std::vector<float> final_score = take_f32(S);
  // ArcTable.validate (table.py:87-127), in the reference's check order:
  // ranges, sort order, backoff targets, per-state arc ranges, coverage,
  // root backoff, finals' zero backoff, non-final backoffs <= 0, finiteness.
  // is_final is any nonzero byte (astype(bool), table.py:300).
  if (S < 1 || V < 1)
    return fail(PGPB_EFORMAT, "need at least 1 state and 1 token, got S=" + std::to_string(S) + " V=" +
                                  std::to_string(V));
  for (uint8_t &f : is_final) f = f ? 1 : 0;
  auto all_in = [&](const std::vector<int32_t> &a, uint32_t hi) {
    for (int32_t x : a)
      if (x < 0 || uint32_t(x) >= hi) return false;
    return true;
  };
  if (A) {
    if (!all_in(arc_from, S)) return fail(PGPB_EFORMAT, "arc_from out of range");
    if (!all_in(arc_to, S)) return fail(PGPB_EFORMAT, "arc_to out of range");
    if (!all_in(arc_token, V)) return fail(PGPB_EFORMAT, "arc_token out of range");
    for (uint32_t j = 1; j < A; ++j)
      if (int64_t(arc_from[j]) * V + arc_token[j] <= int64_t(arc_from[j - 1]) * V + arc_token[j - 1])
        return fail(PGPB_EFORMAT, "arcs not strictly sorted by (from_state, token)");
  }
  if (!all_in(backoff_to, S)) return fail(PGPB_EFORMAT, "backoff_to out of range");
  int64_t covered = 0;
  for (uint32_t st = 0; st < S; ++st) {
    const int32_t lo = state_start[st], hi = state_end[st];
    if (!(0 <= lo && lo <= hi && uint32_t(hi) <= A))
      return fail(PGPB_EFORMAT, "state " + std::to_string(st) + ": bad arc range [" + std::to_string(lo) + ", " +
                                    std::to_string(hi) + ")");
    for (int32_t j = lo; j < hi; ++j)
      if (uint32_t(arc_from[j]) != st)
        return fail(PGPB_EFORMAT, "state " + std::to_string(st) + ": arc range covers foreign arcs");
    covered += int64_t(hi) - lo;
  }
  if (covered != int64_t(A)) return fail(PGPB_EFORMAT, "arc ranges do not cover the arc array");
  if (backoff_to[0] != 0 || backoff_weight[0] != 0.0f) return fail(PGPB_EFORMAT, "root backoff must be (0, 0)");
  for (uint32_t st = 0; st < S; ++st)
    if (is_final[st] && backoff_weight[st] != 0.0f)
      return fail(PGPB_EFORMAT, "final states must have zero backoff weight");
  for (uint32_t st = 1; st < S; ++st)
    if (!is_final[st] && !(backoff_weight[st] <= 0.0f))
      return fail(PGPB_EFORMAT, "non-final backoff weights must be <= 0");
  for (uint32_t j = 0; j < A; ++j)
    if (!std::isfinite(arc_weight[j])) return fail(PGPB_EFORMAT, "non-finite weight");
  for (uint32_t st = 0; st < S; ++st)
    if (!std::isfinite(backoff_weight[st])) return fail(PGPB_EFORMAT, "non-finite weight");
  return pgpb_table_create(int32_t(S), int32_t(V), int32_t(A), arc_token.data(), arc_to.data(), arc_weight.data(),
                           state_start.data(), state_end.data(), backoff_to.data(), backoff_weight.data(),
                           is_final.data(), final_score.data(), unk, device, out);
}

int pgpb_table_load_gpb1(const void *data, int64_t size, int32_t device, pgpb_table **out) {
  return pgpb::guarded([&] { return pgpb_table_load_gpb1_impl(data, size, device, out); });
}

static int pgpb_table_load_gpb1_file_impl(const char *path, int32_t device, pgpb_table **out) {
  using pgpb::fail;
  if (!path) return fail(PGPB_EINVAL, "path is NULL");
  FILE *f = std::fopen(path, "rb");
  if (!f) return fail(PGPB_EINVAL, std::string("cannot open ") + path);
  std::vector<unsigned char> buf;
  unsigned char chunk[1 << 16];
  size_t n;
  while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + n);
  std::fclose(f);
  const int rc = pgpb_table_load_gpb1(buf.data(), int64_t(buf.size()), device, out);
  if (rc != PGPB_OK) pgpb::set_error(std::string(path) + ": " + pgpb_last_error());
  return rc;
}

int pgpb_table_load_gpb1_file(const char *path, int32_t device, pgpb_table **out) {
  return pgpb::guarded([&] { return pgpb_table_load_gpb1_file_impl(path, device, out); });
}

int pgpb_table_info_get(const pgpb_table *t, pgpb_table_info *out) {
  if (!t || !out) return pgpb::fail(PGPB_EINVAL, "NULL argument");
  out->num_states = t->view.num_states;
  out->vocab_size = t->view.vocab_size;
  out->num_arcs = t->view.num_arcs;
  out->max_chain = t->max_chain;
  out->closure_entries = t->closure_entries;
  out->max_closure = t->max_closure;
  out->device = t->device;
  out->device_bytes = t->arena_bytes;
  out->unk_score = t->view.unk_score;
  out->max_root_score = t->view.max_root_score;
  return PGPB_OK;
}

void pgpb_table_destroy(pgpb_table *t) {
  if (!t) return;
  if (t->arena) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(t->device);
    cudaFree(t->arena);
    cudaSetDevice(prev);
  }
  delete t;
}

}  // extern "C"
