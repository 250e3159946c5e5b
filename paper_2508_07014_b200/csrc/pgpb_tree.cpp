// Host-side tree compilation: phrase list -> token trie -> Aho-Corasick fail
// links -> flat arc table.  Native replacement for the reference's Python
// build (tree.py:145-214, table.py:138-187); outputs are array-identical to
// the reference's (node numbering, arc order and every fp64->fp32 rounding
// point), which tests/test_tree_build.py pins against golden fixtures.
//
// Compiled with -ffp-contract=off: the reference computes c0*beta + ln(d)
// and acc sums as separately rounded IEEE doubles (Python floats).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "pgpb_internal.h"

namespace pgpb {

Tuning &tuning() {
  static Tuning t;
  return t;
}

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

// arc_score (tree.py:53-61): depth-scaled c0 | c0*beta + ln(d), or uniform c0.
static inline double arc_score(int32_t depth, double c0, double beta, int32_t mode) {
  if (mode == PGPB_WEIGHT_UNIFORM) return c0;
  if (depth == 1) return c0;
  volatile double cb = c0 * beta;  // separately rounded product, as Python
  return cb + std::log(static_cast<double>(depth));
}

}  // namespace pgpb

extern "C" {

const char *pgpb_last_error(void) { return pgpb::g_last_error.c_str(); }

int pgpb_abi_version(void) { return PGPB_ABI_VERSION; }

int pgpb_set_tuning(const char *key, int32_t value) {
  if (!key) return pgpb::fail(PGPB_EINVAL, "key is NULL");
  pgpb::Tuning &t = pgpb::tuning();
  const std::string k(key);
  if (value < 0) return pgpb::fail(PGPB_EINVAL, "tuning values are >= 0 (0 = automatic)");
  if (k == "ctc.consumers") t.ctc_consumers = value;
  else if (k == "ctc.segment") t.ctc_segment = value;
  else if (k == "ctc.seq") t.ctc_seq = value;
  else if (k == "ll.warps") t.ll_warps = value;
  else if (k == "adv.compact") t.adv_compact = value;
  else if (k == "beam.blobs") t.beam_blobs = value;
  else if (k == "cb.threads") t.cb_threads = value;
  else return pgpb::fail(PGPB_EINVAL, "unknown tuning key " + k);
  return PGPB_OK;
}

static int pgpb_trie_build_impl(const int32_t *tokens, const int64_t *offsets, int64_t n_phrases,
                    int32_t vocab_size, double c0, double beta, int32_t weight_mode,
                    double uniform_final_bonus, int64_t capacity, int32_t *parent,
                    int32_t *depth, int32_t *in_token, uint8_t *is_final, double *arc_sc,
                    double *acc, int64_t *num_nodes, int64_t *bad_phrase, int64_t *bad_token) {
  using pgpb::fail;
  if (vocab_size < 1) return fail(PGPB_EINVAL, "vocab_size must be >= 1");
  if (n_phrases < 0) return fail(PGPB_EINVAL, "n_phrases must be >= 0");
  if (weight_mode != PGPB_WEIGHT_DEPTH_SCALED && weight_mode != PGPB_WEIGHT_UNIFORM)
    return fail(PGPB_EINVAL, "unknown weight mode");
  if (capacity < 1) return fail(PGPB_EINVAL, "capacity must be >= 1");
  if (bad_phrase) *bad_phrase = -1;
  if (bad_token) *bad_token = -1;

  // Root = node 0 (tree.py:153-154).
  int64_t n = 1;
  parent[0] = -1;
  depth[0] = 0;
  in_token[0] = -1;
  is_final[0] = 0;
  // Child lookup: dense at the root (fan-out ~V), hashed below it.
  std::vector<int32_t> root_child(static_cast<size_t>(vocab_size), -1);
  std::unordered_map<uint64_t, int32_t> child;
  child.reserve(static_cast<size_t>(std::min<int64_t>(capacity, 1 << 22)));

  for (int64_t p = 0; p < n_phrases; ++p) {
    const int64_t lo = offsets[p], hi = offsets[p + 1];
    if (hi <= lo) {  // tree.py:156-157
      if (bad_phrase) *bad_phrase = p;
      return fail(PGPB_EINVAL, "empty phrase");
    }
    int32_t cur = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const int32_t tok = tokens[i];
      if (tok < 0 || tok >= vocab_size) {  // tree.py:160-163
        if (bad_phrase) *bad_phrase = p;
        if (bad_token) *bad_token = tok;
        return fail(PGPB_EINVAL, "token id out of range");
      }
      int32_t nxt;
      if (cur == 0) {
        nxt = root_child[tok];
      } else {
        auto it = child.find((static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tok));
        nxt = it == child.end() ? -1 : it->second;
      }
      if (nxt < 0) {  // new node: id = creation order (tree.py:165-168)
        if (n >= capacity) return fail(PGPB_EINVAL, "node capacity exceeded");
        nxt = static_cast<int32_t>(n++);
        parent[nxt] = cur;
        depth[nxt] = depth[cur] + 1;
        in_token[nxt] = tok;
        is_final[nxt] = 0;
        if (cur == 0)
          root_child[tok] = nxt;
        else
          child.emplace((static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tok), nxt);
      }
      cur = nxt;
    }
    is_final[cur] = 1;  // tree.py:172
  }

  // Scores after insertion (tree.py:174-184): arc score by depth (+ uniform
  // final bonus), acc = parent acc + arc, in creation order.
  arc_sc[0] = 0.0;
  acc[0] = 0.0;
  for (int64_t i = 1; i < n; ++i) {
    double s = pgpb::arc_score(depth[i], c0, beta, weight_mode);
    if (weight_mode == PGPB_WEIGHT_UNIFORM && is_final[i]) s = s + uniform_final_bonus;
    arc_sc[i] = s;
    acc[i] = acc[parent[i]] + s;
  }
  *num_nodes = n;
  return PGPB_OK;
}

int pgpb_trie_build(const int32_t *tokens, const int64_t *offsets, int64_t n_phrases,
                    int32_t vocab_size, double c0, double beta, int32_t weight_mode,
                    double uniform_final_bonus, int64_t capacity, int32_t *parent,
                    int32_t *depth, int32_t *in_token, uint8_t *is_final, double *arc_sc,
                    double *acc, int64_t *num_nodes, int64_t *bad_phrase, int64_t *bad_token) {
  return pgpb::guarded([&] { return pgpb_trie_build_impl(tokens, offsets, n_phrases, vocab_size, c0, beta, weight_mode, uniform_final_bonus, capacity, parent, depth, in_token, is_final, arc_sc, acc, num_nodes, bad_phrase, bad_token); });
}

// Children of every node as CSR sorted by (parent, token).
static void children_csr(int64_t n, const int32_t *parent, const int32_t *in_token,
                         std::vector<int32_t> &start, std::vector<int32_t> &kids) {
  start.assign(static_cast<size_t>(n + 1), 0);
  for (int64_t i = 1; i < n; ++i) start[parent[i] + 1]++;
  for (int64_t i = 0; i < n; ++i) start[i + 1] += start[i];
  kids.resize(static_cast<size_t>(n > 0 ? n - 1 : 0));
  std::vector<int32_t> fill(start.begin(), start.end() - 1);
  for (int64_t i = 1; i < n; ++i) kids[fill[parent[i]]++] = static_cast<int32_t>(i);
  for (int64_t p = 0; p < n; ++p) {
    std::sort(kids.begin() + start[p], kids.begin() + start[p + 1],
              [&](int32_t a, int32_t b) { return in_token[a] < in_token[b]; });
  }
}

static int pgpb_trie_fail_links_impl(int64_t n, const int32_t *parent, const int32_t *in_token,
                         int32_t vocab_size, int32_t *fail_out) {
  using pgpb::fail;
  if (n < 1) return fail(PGPB_EINVAL, "tree needs a root");
  std::vector<int32_t> start, kids;
  children_csr(n, parent, in_token, start, kids);
  std::vector<int32_t> root_child(static_cast<size_t>(vocab_size), -1);
  for (int32_t j = start[0]; j < start[1]; ++j) root_child[in_token[kids[j]]] = kids[j];
  auto lookup = [&](int32_t f, int32_t tok) -> int32_t {
    if (f == 0) return root_child[tok];
    auto b = kids.begin() + start[f], e = kids.begin() + start[f + 1];
    auto it = std::lower_bound(b, e, tok, [&](int32_t k, int32_t t) { return in_token[k] < t; });
    return (it != e && in_token[*it] == tok) ? *it : -1;
  };
  // BFS, children in ascending token order (tree.py:196-213).
  std::vector<int32_t> queue;
  queue.reserve(static_cast<size_t>(n));
  fail_out[0] = 0;
  for (int32_t j = start[0]; j < start[1]; ++j) {
    fail_out[kids[j]] = 0;
    queue.push_back(kids[j]);
  }
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    const int32_t nid = queue[qi];
    for (int32_t j = start[nid]; j < start[nid + 1]; ++j) {
      const int32_t c = kids[j];
      const int32_t tok = in_token[c];
      int32_t f = fail_out[nid];
      while (f != 0 && lookup(f, tok) < 0) f = fail_out[f];
      const int32_t hit = lookup(f, tok);
      fail_out[c] = (hit >= 0 && hit != c) ? hit : 0;
      queue.push_back(c);
    }
  }
  return PGPB_OK;
}

int pgpb_trie_fail_links(int64_t n, const int32_t *parent, const int32_t *in_token,
                         int32_t vocab_size, int32_t *fail_out) {
  return pgpb::guarded([&] { return pgpb_trie_fail_links_impl(n, parent, in_token, vocab_size, fail_out); });
}

static int pgpb_trie_compile_impl(int64_t n, const int32_t *parent, const int32_t *in_token,
                      const uint8_t *is_final, const double *arc_sc, const double *acc,
                      const int32_t *fail_in, int32_t *arc_from, int32_t *arc_token,
                      int32_t *arc_to, float *arc_weight, int32_t *state_start,
                      int32_t *state_end, int32_t *backoff_to, float *backoff_weight,
                      float *final_score) {
  using pgpb::fail;
  if (n < 1) return fail(PGPB_EINVAL, "tree needs a root");
  std::vector<int32_t> start, kids;
  children_csr(n, parent, in_token, start, kids);
  // Arcs sorted by (from, token) (table.py:147-158); weight = f32(score).
  for (int64_t p = 0; p < n; ++p) {
    state_start[p] = start[p];
    state_end[p] = start[p + 1];
    for (int32_t j = start[p]; j < start[p + 1]; ++j) {
      const int32_t c = kids[j];
      arc_from[j] = static_cast<int32_t>(p);
      arc_token[j] = in_token[c];
      arc_to[j] = c;
      arc_weight[j] = static_cast<float>(arc_sc[c]);
    }
  }
  // Backoff weights: f32(acc[fail] - acc) in fp64; 0 for finals and root;
  // final_score = f32(acc) for finals (table.py:163-169).
  for (int64_t s = 0; s < n; ++s) {
    const int32_t f = fail_in[s];
    if (f < 0 || f >= n) return fail(PGPB_EINVAL, "fail link out of range");
    backoff_to[s] = f;
    float bw = static_cast<float>(acc[f] - acc[s]);
    if (is_final[s] || s == 0) bw = 0.0f;
    backoff_weight[s] = bw;
    final_score[s] = is_final[s] ? static_cast<float>(acc[s]) : 0.0f;
  }
  return PGPB_OK;
}

int pgpb_trie_compile(int64_t n, const int32_t *parent, const int32_t *in_token,
                      const uint8_t *is_final, const double *arc_sc, const double *acc,
                      const int32_t *fail_in, int32_t *arc_from, int32_t *arc_token,
                      int32_t *arc_to, float *arc_weight, int32_t *state_start,
                      int32_t *state_end, int32_t *backoff_to, float *backoff_weight,
                      float *final_score) {
  return pgpb::guarded([&] { return pgpb_trie_compile_impl(n, parent, in_token, is_final, arc_sc, acc, fail_in, arc_from, arc_token, arc_to, arc_weight, state_start, state_end, backoff_to, backoff_weight, final_score); });
}

}  // extern "C"
