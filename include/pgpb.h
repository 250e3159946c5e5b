/*
 * pgpb.h — C-ABI of the B200-native GPU phrase-boosting tree (GPU-PB).
 *
 * This is the drop-in boundary for the reference's native kernel module
 * (`phraseboost._kernels`, /root/reference/pkg/src/phraseboost/_kernels.pyx)
 * and for the host-side tree compiler the reference implements in Python
 * (tree.py / table.py).  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - Every entry point returns PGPB_OK (0) or a negative PGPB_E* code; the
 *     message of the last failure on the calling thread is available from
 *     pgpb_last_error().  (The reference raises Python exceptions instead;
 *     the Python host layer maps these codes back to the reference's
 *     exception types and messages.)
 *   - `d_` pointers are device pointers, `h_` pointers host pointers.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     All device work is stream-ordered; nothing synchronises unless the
 *     function name ends in `_host` (those copy results back and wait).
 *   - The caller owns every buffer it passes in; a pgpb_table owns its own
 *     device copy of the compiled arc table and is immutable after creation,
 *     so one table may be used concurrently from many streams / threads
 *     (reference: SPEC.md:259, tests/test_table.py:330-343).
 */
#ifndef PGPB_H
#define PGPB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGPB_ABI_VERSION 1

#define PGPB_OK 0
#define PGPB_EINVAL (-1)     /* bad argument (maps to ValueError)            */
#define PGPB_ERANGE (-2)     /* index out of range (maps to IndexError)       */
#define PGPB_ECUDA (-3)      /* CUDA runtime failure                          */
#define PGPB_ENOMEM (-4)     /* allocation failure                            */
#define PGPB_EFORMAT (-5)    /* table invariant violated (TableFormatError)   */

#define PGPB_WEIGHT_DEPTH_SCALED 0 /* tree.py:30 */
#define PGPB_WEIGHT_UNIFORM 1      /* tree.py:31 */

const char *pgpb_last_error(void);
int pgpb_abi_version(void);

/* Code-path overrides for tests and measurements; value 0 restores the
 * automatic choice.  Keys: "ctc.consumers" (walker warps per CTA),
 * "ctc.segment" (frames per walker segment), "ctc.seq" (1 = sequential walk,
 * 2 = speculative rounds only), "ll.warps" (label-loop rows per CTA).  Every
 * setting selects between bit-identical code paths; process-wide, not
 * thread-safe against concurrent launches.  PGPB_EINVAL on an unknown key. */
int pgpb_set_tuning(const char *key, int32_t value);

/* ------------------------------------------------------------------------
 * Tree compilation (host code, C++).  Replaces the Python loops of
 *   build_prefix_tree   tree.py:145-186
 *   compute_fail_links  tree.py:189-214
 *   compile_arc_table   table.py:138-187
 * Node ids follow the reference exactly (creation order while inserting
 * phrases in ContextList order, root = 0), so next-state ids are
 * bit-identical to the reference's.
 * ---------------------------------------------------------------------- */

/* build_prefix_tree (tree.py:145-186).  Phrases are given as CSR:
 * tokens[offsets[i] .. offsets[i+1]) is phrase i.  `capacity` is the size of
 * every node output array (1 + offsets[n_phrases] always suffices).
 * On an empty phrase or an out-of-range token returns PGPB_EINVAL and sets
 * *bad_phrase (and *bad_token, -1 for "empty").                            */
int pgpb_trie_build(const int32_t *h_tokens, const int64_t *h_offsets, int64_t n_phrases,
                    int32_t vocab_size, double c0, double beta, int32_t weight_mode,
                    double uniform_final_bonus, int64_t capacity, int32_t *h_parent,
                    int32_t *h_depth, int32_t *h_in_token, uint8_t *h_is_final,
                    double *h_arc_score, double *h_acc_score, int64_t *num_nodes,
                    int64_t *bad_phrase, int64_t *bad_token);

/* compute_fail_links (tree.py:189-214): Aho-Corasick longest proper suffix.
 * Writes fail[num_nodes] (fail[0] = 0).                                    */
int pgpb_trie_fail_links(int64_t num_nodes, const int32_t *h_parent, const int32_t *h_in_token,
                         int32_t vocab_size, int32_t *h_fail);

/* compile_arc_table (table.py:138-187).  Arc arrays have num_nodes-1
 * entries, sorted by (from, token); state arrays have num_nodes entries.
 * fp64 -> fp32 rounding points follow table.py:158, :163-169.               */
int pgpb_trie_compile(int64_t num_nodes, const int32_t *h_parent, const int32_t *h_in_token,
                      const uint8_t *h_is_final, const double *h_arc_score,
                      const double *h_acc_score, const int32_t *h_fail, int32_t *h_arc_from,
                      int32_t *h_arc_token, int32_t *h_arc_to, float *h_arc_weight,
                      int32_t *h_state_start, int32_t *h_state_end, int32_t *h_backoff_to,
                      float *h_backoff_weight, float *h_final_score);

/* ------------------------------------------------------------------------
 * Device-resident compiled table.
 * Takes the reference ArcTable arrays (table.py:53-69, the 9 arrays the
 * reference passes to score_batch plus is_final / final_score) and builds
 * the device layout described in DESIGN.md §3: dense root row, packed
 * 16-byte state records and arcs, and the per-state flattened backoff
 * closure.  Validates chain termination (PGPB_EFORMAT on a backoff cycle).
 * ---------------------------------------------------------------------- */
typedef struct pgpb_table pgpb_table;

typedef struct pgpb_table_info {
  int32_t num_states;
  int32_t vocab_size;
  int32_t num_arcs;
  int32_t max_chain;        /* longest backoff chain (states, excluding root) */
  int64_t closure_entries;  /* total flattened first-hit arcs over all states */
  int32_t max_closure;      /* largest per-state closure                       */
  int32_t device;
  int64_t device_bytes;     /* HBM held by the table                           */
  float unk_score;
  float max_root_score;
} pgpb_table_info;

int pgpb_table_create(int32_t num_states, int32_t vocab_size, int32_t num_arcs,
                      const int32_t *h_arc_token, const int32_t *h_arc_to,
                      const float *h_arc_weight, const int32_t *h_state_start,
                      const int32_t *h_state_end, const int32_t *h_backoff_to,
                      const float *h_backoff_weight, const uint8_t *h_is_final,
                      const float *h_final_score, float unk_score, int32_t device,
                      pgpb_table **out);
/* GPB1 bytes (the reference's serialized table, table.py:16-29 / save_table
 * :250-264) straight to a device table: parse + the reference's validate
 * invariants (table.py:87-127) on the host, then pgpb_table_create.
 * Replaces load_table (table.py:267-310) + the Python ArcTable for callers
 * that only need the device table.  PGPB_EFORMAT on a malformed file.     */
int pgpb_table_load_gpb1(const void *data, int64_t size, int32_t device, pgpb_table **out);
int pgpb_table_load_gpb1_file(const char *path, int32_t device, pgpb_table **out);

int pgpb_table_info_get(const pgpb_table *table, pgpb_table_info *out);
void pgpb_table_destroy(pgpb_table *table);

/* ------------------------------------------------------------------------
 * Advance = get_scores_batch (table.py:190-214) / _kernels.score_batch
 * (_kernels.pyx:30-72): for each of B states, the boosting score and next
 * state of every token.  scores[B,V] f32 and next[B,V] i32, C order.
 * Bit-exact with the reference (fp32 accumulation in backoff-chain order,
 * first hit wins).  States are NOT range-checked on device (the reference
 * kernel does not either, _kernels.pyx:1); the host layer raises IndexError
 * as table.py:198-199 does.  B = 0 is a no-op.
 * ---------------------------------------------------------------------- */
int pgpb_advance(const pgpb_table *table, const int32_t *d_states, int64_t batch,
                 float *d_scores, int32_t *d_next, void *stream);

/* Same, host buffers in and out: H2D of the states, the kernel, D2H of both
 * outputs, then a stream synchronize — the exact contract of
 * _kernels.score_batch (fresh C-order [B,V] outputs the caller allocated).
 * Range-checks states (PGPB_ERANGE).                                       */
int pgpb_advance_host(const pgpb_table *table, const int32_t *h_states, int64_t batch,
                      float *h_scores, int32_t *h_next, void *stream);

/* R chained advances in one launch (BASELINE config 5):
 * s_0 = d_states[b]; step k advances s_k exactly as pgpb_advance does and
 * writes d_scores/d_next[(k*B + b)*V + v] (R x [B,V] outputs); then
 * s_{k+1} = next_k[b, d_tokens[k*B + b]].  Optional outputs: d_trace[k*B + b]
 * = s_k (R x B), d_final_states[b] = s_R.  `parts` = column parts per row
 * (0 = choose; a power of two dividing the row into multiples of 128
 * tokens).  Tokens and states are not range-checked on device.
 * Each step is the reference's get_scores_batch (table.py:190-214,
 * _kernels.pyx:30-72) of that step's states; the successor rule is the
 * reference's next-state lookup (decoding.py:379-383, _kernels.pyx:204-209). */
int pgpb_advance_steps(const pgpb_table *table, const int32_t *d_states, const int32_t *d_tokens,
                       int32_t steps, int64_t batch, float *d_scores, int32_t *d_next, int32_t *d_trace,
                       int32_t *d_final_states, int32_t parts, void *stream);

/* Reference chain-walk advance (no flattened closure): walks failure arcs
 * per row exactly as _kernels.pyx:56-71.  Same outputs as pgpb_advance;
 * kept for tables whose closure would not fit and as a cross-check.        */
int pgpb_advance_chain(const pgpb_table *table, const int32_t *d_states, int64_t batch,
                       float *d_scores, int32_t *d_next, void *stream);

/* ------------------------------------------------------------------------
 * Phrase-hit counting = evaluation.keyphrase_hits / count_occurrences
 * (evaluation.py:90-134) over a large corpus.  `table` is an Aho-Corasick
 * table compiled over word ids (phrase words 1..W, any other word 0);
 * out_start/out_len/out_phrase[state] list the phrases whose end node lies
 * on the state's failure chain.  n_seqs word sequences, words[offsets[q] ..
 * offsets[q+1]) for sequence q.  Pass 1 (d_keys == NULL): d_counts[q] =
 * occurrences in sequence q.  Pass 2: keys phrase * n_seqs + q written from
 * d_key_offsets[q] (an exclusive scan of the counts).                      */
int pgpb_phrase_hits(const pgpb_table *table, const int32_t *d_words, const int64_t *d_offsets,
                     int64_t n_seqs, const int32_t *d_out_start, const int32_t *d_out_len,
                     const int32_t *d_out_phrase, int32_t *d_counts, int64_t *d_keys,
                     const int64_t *d_key_offsets, void *stream);

/* ------------------------------------------------------------------------
 * Fused batched greedy CTC = _kernels.ctc_greedy (_kernels.pyx:75-225) /
 * ctc_greedy_boosted (decoding.py:156-229), over B utterances at once.
 * logprobs [B,T,V] f32 C order; lengths[B] (<= T) frames per utterance.
 * table may be NULL (boost inactive, decoding.py:103-104); otherwise
 * use_boost selects the boosted path.  The [B,V] score matrix is never
 * materialised.  Outputs (device):
 *   tokens[B,T] i32, deltas[B,T] f64, states[B,T] i32  (first num_out[b]
 *   entries of row b valid), num_out[B] i32, am[B] f64, boost[B] f64.
 * Results per utterance are bit-identical to the reference's per-utterance
 * call (fp64 fusion without FMA, tie-breaks: combined, raw logprob, id).    */
int pgpb_ctc_greedy(const pgpb_table *table, const float *d_logprobs, int64_t batch,
                    int64_t max_frames, int32_t vocab_size, const int32_t *d_lengths,
                    int32_t blank, double lam, int32_t use_boost, int32_t *d_tokens,
                    double *d_deltas, int32_t *d_states, int32_t *d_num_out, double *d_am,
                    double *d_boost, void *stream);

/* Host-buffer form of one utterance, the exact contract of
 * _kernels.ctc_greedy: h_logprobs [T,V]; outputs sized T; *num_out set.     */
int pgpb_ctc_greedy_host(const pgpb_table *table, const float *h_logprobs, int64_t frames,
                         int32_t vocab_size, int32_t blank, double lam, int32_t use_boost,
                         int32_t *h_tokens, double *h_deltas, int32_t *h_states,
                         int64_t *num_out, double *h_am, double *h_boost, void *stream);

/* ------------------------------------------------------------------------
 * Fused boosted greedy step for transducers (RNN-T / TDT label looping):
 * the body of transducer_greedy_boosted's inner loop (decoding.py:373-392)
 * for B rows at once.  For each row r with active[r] != 0:
 *   a = first argmax of logprobs[r,:];  is_blank[r] = (a == blank)
 *   if !is_blank: chosen = boosted rerank excluding blank only (R7/R6
 *   tie-breaks), delta = tree score, next = tree next state (when boost is
 *   off: chosen = a, delta = 0, next = 0).
 * Writes chosen[r] (= a when blank), lp_chosen[r] (f32 logprob of chosen),
 * delta[r] f64, next_state[r].  Inactive rows are left untouched.
 * ld = row stride of logprobs in elements.                                  */
int pgpb_greedy_step(const pgpb_table *table, const float *d_logprobs, int64_t ld,
                     int64_t rows, int32_t vocab_size, const int32_t *d_states,
                     const uint8_t *d_active, int32_t blank, double lam, int32_t use_boost,
                     int32_t *d_chosen, float *d_lp_chosen, double *d_delta,
                     int32_t *d_next_state, uint8_t *d_is_blank, void *stream);

/* Label-looping state of B transducer utterances (all device pointers).
 * Layout: t, k, lengths, n, last are int64[B]; tree int32[B]; am, boost
 * float64[B]; tokens/states int32[B, lmax], deltas float64[B, lmax].     */
typedef struct pgpb_label_loop_state {
  int64_t *t;        /* current frame                                     */
  int64_t *k;        /* symbols emitted at the current frame              */
  const int64_t *lengths;
  int64_t *n;        /* tokens emitted so far                             */
  int64_t *last;     /* last emitted token (prediction-net context)       */
  int32_t *tree;     /* GPU-PB tree state                                 */
  double *am;
  double *boost;
  int32_t *tokens;
  double *deltas;
  int32_t *states;
  int64_t lmax;
  int32_t cap;       /* max_symbols_per_frame                             */
  /* TDT (token-and-duration transducer): frames to advance per row, the
   * argmax of the duration head, or NULL for RNN-T.  A blank advances
   * max(d, 1) frames; an emission with d > 0 advances d frames and resets
   * the symbol counter; d == 0 stays on the frame (cap still applies).
   * No reference counterpart: parity-unpinned extension; with
   * d = 0 for every emission and d = 1 for blanks it is exactly R7.       */
  const int32_t *durations;
  /* Optional (NULL: looked up): blob offset of tree[r] (TableView blob
   * layout), carried across iterations so that a row's tree state costs one
   * dependent load instead of two; a negative entry means "look it up". */
  int32_t *tree_off;
} pgpb_label_loop_state;

/* One label-looping iteration fused with its bookkeeping: for every row r
 * with t[r] < lengths[r], decide the row exactly as pgpb_greedy_step does,
 * then apply R7 (decoding.py:371-392): blank -> am += lp[blank], next frame;
 * emission -> am/boost/outputs/tree updated, k += 1, and after `cap`
 * emissions the frame advances without a blank score.  Writes emit[r]
 * (1 iff row r emitted) and feed[r] (token the prediction network consumes
 * next: the emitted token, else last[r]); atomically ORs 1 into *any_active
 * when some row still has frames left (caller zeroes it).               */
int pgpb_label_loop_step(const pgpb_table *table, const float *d_logprobs, int64_t ld,
                         int64_t rows, int32_t vocab_size, int32_t blank, double lam,
                         int32_t use_boost, const pgpb_label_loop_state *state,
                         uint8_t *d_emit, int64_t *d_feed, int32_t *d_any_active, void *stream);

/* pgpb_label_loop_step with the joint's log-softmax fused in: row r's bf16
 * logits (row stride ld_logits) are log-softmaxed in fp32 into lp_out[r]
 * (stride vocab_size; torch's formula order (x - max) - log(sum exp(x -
 * max))), which the decision then reads; lp_out doubles as the record of
 * the log-probs each row was decided on.  Config-2 decoder glue
 * (rnnt.py), same decision and bookkeeping as pgpb_label_loop_step.      */
int pgpb_label_loop_step_logits(const pgpb_table *table, const void *d_logits_bf16, int64_t ld_logits,
                                float *d_lp_out, int64_t rows, int32_t vocab_size, int32_t blank,
                                double lam, int32_t use_boost, const pgpb_label_loop_state *state,
                                uint8_t *d_emit, int64_t *d_feed, int32_t *d_any_active, void *stream);

/* Config-2 prediction / joint network glue (rnnt.py; no reference
 * counterpart: the reference's transducer decoders take a host StepModel,
 * acoustic.py:203-255).  bf16 tensors, row-major.
 *  joint_hidden: z[b, :J] = relu(enc_proj[b, min(t[b], max(len[b]-1, 0)), :J]
 *                + pred_proj[b, :J]); enc_proj stride per utterance ld_b,
 *                pred_proj row stride ld_pred (elements).
 *  lstm_update:  gates = E[feed[b]] + hg[b] (E[V, 4H] = emb W_ih^T + b_ih,
 *                hg[B, 4H] = h W_hh^T + b_hh; gate order i, f, g, o), LSTM
 *                cell in fp32, h[b], c[b] overwritten iff emit[b] (NULL: all);
 *                hg row stride ld_hg (elements).                           */
int pgpb_rnnt_joint_hidden(const void *d_enc_proj, int64_t ld_b, int32_t J, const int64_t *d_t,
                           const int64_t *d_lengths, const void *d_pred_proj, int64_t ld_pred, void *d_z,
                           int64_t B, void *stream);
/* Stateless-transducer beam joint (beams.py, configs 3): z[b*K + k, :J] =
 * relu(enc_proj[b, min(t[b], max(len[b]-1, 0))] + pred_j[last[b, k] < 0 ?
 * blank : last[b, k]]), int32 t / lengths / last.                         */
int pgpb_rnnt_beam_hidden(const void *d_enc_proj, int64_t ld_b, int32_t J, const int32_t *d_t,
                          const int32_t *d_lengths, const void *d_pred_j, const int32_t *d_last, int64_t B,
                          int32_t K, int32_t blank, void *d_z, void *stream);
int pgpb_rnnt_lstm_update(const void *d_E, const int64_t *d_feed, const void *d_hg, int64_t ld_hg,
                          const uint8_t *d_emit, void *d_h, void *d_c, int64_t B, int32_t H, void *stream);

/* Per state: final_score[s] when is_final[s], else 0 (f32[S]) — the final
 * part of the AED eos bump (decoding.py:546-552), for tables that live only
 * on the device (load_table_device).                                        */
int pgpb_final_bonus(const pgpb_table *table, float *d_out, void *stream);

/* Per state: the fp32 sum of the backoff weights along its chain, in chain
 * order (_kernels.pyx:59-66) — the unfinished-phrase credit a hypothesis
 * ending in that state would give back (rollback extension).  out[S] f32.  */
int pgpb_backoff_total(const pgpb_table *table, float *d_out, void *stream);

/* Per-state maximum of the resolved score row, max_v scores[s, v]
 * (used by the AED eos bump, decoding.py:546-552).  out[S] f32.             */
int pgpb_row_max(const pgpb_table *table, float *d_out, void *stream);

/* ------------------------------------------------------------------------
 * Fused beam expansion (the V-wide inner loops of the reference's beam
 * decoders: ctc_beam_boosted decoding.py:294-321, transducer_beam_boosted
 * :473-489, aed_beam_boosted :544-583).  Hypotheses come in groups of
 * `group` consecutive rows (one utterance each, padded rows have
 * valid[h] == 0).  Every candidate (h, v) with v != exclude[h] is scored
 *      am'    = base(h, v) + (double)lp[h, v]
 *               base = alt_am[h] if v == alt_token[h] else am[h]
 *      boost' = boost[h] + (double)score[state[h], v]      (0 if !use_boost)
 *      key    = am' + lam * boost'      (fp64, unfused; decoding.py:323-327)
 * and the best `k` (any k; top-k runs in exact passes of 32 winners) per group are returned
 * ordered by key desc,
 * am' desc, then (h, v) ascending.  With skip_neg_inf, candidates whose am'
 * is -inf are dropped (decoding.py:303-304).  The [H,V] score matrix is
 * never materialised.  Outputs are [G, k]; unfilled slots get hyp = -1.
 * alt_token / alt_am / valid may be NULL.  ld = 0 broadcasts one row to all
 * hypotheses (CTC prefix beam: every prefix reads the same frame).  The
 * reference breaks (key, am) ties by token tuple; the Python drop-in beams
 * ask for k + 1, extend the cut by the whole tie group and re-rank on the
 * host with the tuples (decoding._TopK), so their results are exact on ties. */
int pgpb_beam_topk(const pgpb_table *table, const float *d_logprobs, int64_t ld,
                   int64_t hyps, int32_t vocab_size, int32_t group, int32_t k,
                   const int32_t *d_states, const double *d_am, const double *d_boost,
                   const int32_t *d_exclude, const int32_t *d_alt_token,
                   const double *d_alt_am, const uint8_t *d_valid, double lam,
                   int32_t use_boost, int32_t skip_neg_inf, int32_t *d_out_hyp,
                   int32_t *d_out_token, double *d_out_am, double *d_out_boost,
                   int32_t *d_out_next, float *d_out_delta, void *stream);

/* ------------------------------------------------------------------------
 * Device-resident batched beam search.  The hypothesis bookkeeping the
 * reference does in Python dicts (decoding.py:428-495 transducer beam,
 * :502-587 AED beam) runs inside the fused expansion + top-k kernels: one
 * CTA per utterance scores every (hypothesis, token) candidate, merges and
 * prunes, and writes the new beam in place.  Token sequences live in an
 * append-only per-utterance trie of trace nodes; hypotheses carry the node
 * of their last token plus (length, 64-bit hash) so sequence equality
 * (_keep_better's dict keys) is a hash filter followed by an exact walk.
 * Ranking is the reference's R11 (key = am + lam*boost in fp64, then am);
 * exact (key, am) ties between different hypotheses fall back to the slot
 * order instead of comparing token tuples.
 * ---------------------------------------------------------------------- */

/* K hypotheses per utterance, struct of arrays, each [B, K] row-major.   */
typedef struct pgpb_beam_hyps {
  double *am;
  double *boost;
  int32_t *tree;     /* GPU-PB tree state                                  */
  int32_t *last;     /* last token (-1: none yet, the start symbol)        */
  int32_t *node;     /* trace node of the last step (-1: empty sequence)   */
  int32_t *len;      /* number of tokens                                   */
  uint64_t *hash;    /* hash of the token sequence (0 for the empty one)   */
  uint8_t *flags;    /* bit 0 valid, bit 1 ended (AED eos)                 */
  int32_t *parent;   /* AED: slot of the previous beam this one came from  */
} pgpb_beam_hyps;

/* Append-only trie of trace steps; utterance b's node i at b*nmax + i.
 * TraceStep(token, delta, state) of decoding.py:63-69.                    */
typedef struct pgpb_beam_trace {
  int32_t *parent;
  int32_t *token;
  int32_t *state;
  double *delta;
  int32_t *count;    /* [B] nodes in use                                   */
  int32_t *overflow; /* set to 1 when an utterance runs out of nodes       */
  int64_t nmax;
} pgpb_beam_trace;

/* Transducer beam (R9, decoding.py:454-495): every frame runs exactly
 * cap + 1 waves.  Wave k: each valid hypothesis' blank extension is merged
 * into the frame's finished pool by token sequence (_keep_better, strict
 * improvement); for k < cap the top `beam` non-blank expansions become the
 * next wave's hypotheses; at k == cap the pool's top `beam` become the next
 * frame's beam and t[b] advances.  Rows: d_logprobs[(b*beam + r)*ld + v] is
 * step(last[b,r], t[b]).  rollback != 0 (opt-in, no reference counterpart):
 * at an utterance's last frame every finished hypothesis gets the backoff
 * total of its state added to its boost (unfinished phrase credit removed)
 * before the final top-k.  Utterances with t[b] >= lengths[b] are idle.   */
typedef struct pgpb_tbeam_state {
  pgpb_beam_hyps hyps;      /* [B, beam]                                   */
  pgpb_beam_hyps pool;      /* [B, pool_cap] finished (blank-extended)     */
  int32_t *pool_count;      /* [B]                                         */
  pgpb_beam_trace trace;
  int32_t *t;               /* [B] current frame                           */
  const int32_t *lengths;   /* [B]                                         */
  int32_t beam;
  int32_t cap;              /* max_symbols_per_frame                       */
  int32_t pool_cap;         /* >= beam * (cap + 1)                         */
  int32_t rollback;
} pgpb_tbeam_state;

int pgpb_tbeam_wave(const pgpb_table *table, const float *d_logprobs, int64_t ld, int64_t batch,
                    int32_t vocab_size, int32_t blank, double lam, int32_t use_boost, int32_t wave,
                    const pgpb_tbeam_state *state, void *stream);

/* The same wave with the stateless joint's tail fused in: d_logits_bf16
 * [batch*beam, V] (row stride ld_logits) are log-softmaxed in the kernel
 * (written to d_lp_out, stride ld: the rows the wave decided on), and the
 * next wave's joint hidden rows z[b*beam + k] = relu(enc_proj[b, t_b] +
 * pred_j[last_k]) (bf16, J wide; enc_proj [batch, T, J] with utterance
 * stride enc_ld_b; pred_j [V, J]) are written to d_z_out at the end — one
 * kernel instead of three per wave (beams.TransducerBeamDecoder).          */
int pgpb_tbeam_wave_fused(const pgpb_table *table, const void *d_logits_bf16, int64_t ld_logits, float *d_lp_out,
                          int64_t ld, int64_t batch, int32_t vocab_size, int32_t blank, double lam,
                          int32_t use_boost, int32_t wave, const pgpb_tbeam_state *state, const void *d_enc_proj,
                          int64_t enc_ld_b, int32_t J, const void *d_pred_j, void *d_z_out, void *stream);

/* AED beam step (R10, decoding.py:532-584): candidates are the beam's
 * ended / length-capped hypotheses (carried unchanged) plus every token
 * expansion of the others; eos ends a hypothesis with
 *   bump = max(0, row_max[state]) + (final_score[state] if is_final)
 * added to its boost when use_boost && eos_bump.  The top `beam` replace
 * the beam in place; hyps.parent[b, r] receives the source slot (for the
 * decoder's KV-cache reorder).  *any_active is OR-ed with 1 when some new
 * hypothesis can still expand.  Rows: step(prefix of slot r, len).        */
typedef struct pgpb_aed_state {
  pgpb_beam_hyps hyps;      /* [B, beam]                                   */
  pgpb_beam_trace trace;
  const float *row_max;     /* [S] from pgpb_row_max                       */
  int32_t *any_active;
  int32_t beam;
  int32_t max_len;
  int32_t eos;
  int32_t eos_bump;
  int32_t rollback;         /* extension (no reference counterpart): the eos
                               step also adds the state's backoff total      */
} pgpb_aed_state;

int pgpb_aed_step(const pgpb_table *table, const float *d_logprobs, int64_t ld, int64_t batch,
                  int32_t vocab_size, double lam, int32_t use_boost, const pgpb_aed_state *state,
                  void *stream);

/* ------------------------------------------------------------------------
 * Batched boosted greedy AED: aed_beam_boosted (decoding.py:502-587, R10)
 * at beam 1, one decoder step for all B utterances.  Per utterance the step
 * keeps the best of the eos candidate (am + lp[eos], boost + bump with the
 * eos bump of decoding.py:546-552 when row_max != NULL) and every token
 * v != eos (am + lp[v], boost + score[tree, v]) under the reference's rank
 * (key = am + lam*boost, then am, then the token tuple: eos first on exact
 * ties, then lower v).  Utterances with ended[b] or len[b] >= max_len are
 * left untouched.  Writes tokens[b*max_len + len], the trace step
 * (deltas / states at b*(max_len+1) + len: score or bump, next state), and
 * feed[b] = the token the decoder consumes next; sets *any_active = 1 when
 * an utterance can still extend (the caller zeroes it before the step).    */
typedef struct pgpb_aed_greedy_state {
  int32_t *tree;            /* [B] tree state                                */
  double *am;               /* [B]                                           */
  double *boost;            /* [B]                                           */
  int32_t *len;             /* [B] tokens so far (eos not counted)           */
  uint8_t *ended;           /* [B] 1 after eos                               */
  int64_t *feed;            /* [B] next decoder input token                  */
  int32_t *tokens;          /* [B, max_len]                                  */
  double *deltas;           /* [B, max_len + 1] trace boosts (eos: the bump) */
  int32_t *states;          /* [B, max_len + 1] trace states                 */
  const float *row_max;     /* [S] pgpb_row_max, NULL = no eos bump          */
  const float *final_bonus; /* [S] pgpb_final_bonus (with row_max)           */
  int32_t *any_active;
  int32_t max_len;
  int32_t eos;
  int32_t rollback;         /* extension: eos also adds the backoff total    */
} pgpb_aed_greedy_state;

int pgpb_aed_greedy_step(const pgpb_table *table, const float *d_logprobs, int64_t ld, int64_t batch,
                         int32_t vocab_size, double lam, int32_t use_boost, const pgpb_aed_greedy_state *state,
                         void *stream);

/* ------------------------------------------------------------------------
 * Batched boosted CTC prefix beam search on the device: ctc_beam_boosted
 * (decoding.py:232-343, R8) for B utterances of [T, V] log-probs
 * (d_lp[(b*T + t)*V + v], f32; d_lengths[b] frames or NULL = T), beam <= 32.
 * One launch decodes every frame.  Per utterance the final beam, in rank
 * order (am + lam*boost, then am): count[b] prefixes, and per prefix r at
 * b*beam + r: pb / pnb (blank / non-blank ending mass; am = logaddexp of
 * both), boost, tree state, token count and the last trace node.  The trace
 * (TraceStep(token, delta, state) of decoding.py:63-69) is an append-only
 * trie per utterance at b*trace_nmax + i (parent -1 = empty prefix);
 * trace_nmax >= T*beam + 1.  am is exact up to the device exp/log1p (within
 * 1 ulp of the host libm); tokens, boost and states are exact.              */
typedef struct pgpb_ctc_beam_out {
  double *pb, *pnb, *boost;   /* [B, beam] */
  int32_t *tree, *len, *node; /* [B, beam] */
  int32_t *count;             /* [B]       */
  int32_t *trace_parent, *trace_token, *trace_state; /* [B, trace_nmax] */
  double *trace_delta;
  int64_t trace_nmax;
  int32_t *overflow;          /* set to 1 if a trace ran out of nodes */
} pgpb_ctc_beam_out;

int pgpb_ctc_beam(const pgpb_table *table, const float *d_logprobs, int64_t batch, int64_t frames,
                  int32_t vocab_size, const int32_t *d_lengths, int32_t blank, int32_t beam, double lam,
                  int32_t use_boost, const pgpb_ctc_beam_out *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PGPB_H */
