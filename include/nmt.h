/*
 * nmt.h — C ABI of the B200-native NiuTrans-WNGT2020 translation hot path.
 *
 * The path (PAPER.md = arXiv 2109.08008, cited by line):
 *   encoder: deep pre-norm Transformer with relative position representations
 *            (Shaw et al., clip 8) and the dynamic linear
 *            combination of layers x_{l+1} = sum_k W_k^{(l+1)} LN(y_k)
 *            (Eq. 1-2);
 *   decoder: incremental greedy decoding with cached self-attention K/V and
 *            encoder-decoder K/V projected once per sentence,
 *            tied 32K-vocab projection fused with argmax — no log_softmax for
 *            greedy — and batch pruning of finished sentences
 *             over length-sorted dynamic batches
 *             in FP16 with FP32 reductions
 *            (PAPER.md:122-123).
 * Readings where the paper is silent are listed in DESIGN.md ("Readings").
 *
 * Conventions
 *   - Every call returns nmt_status (NMT_OK == 0); details in nmt_last_error().
 *     No C++ exception crosses the ABI.
 *   - h_* = host pointer, d_* = device pointer on the model's device.
 *     The caller owns every buffer passed in; the library never frees them.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered and asynchronous unless documented otherwise.
 *   - All device memory the path needs is allocated once by nmt_load_weights
 *     (the paper's memory pool): encode / decode / prune /
 *     translate never call cudaMalloc.
 *   - Token ids: PAD 0, UNK 1, BOS 2, EOS 3; sources end with EOS.
 */
#ifndef NMT_H_
#define NMT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NMT_OK = 0,
  NMT_E_ARG = 1,         /* null / negative / out-of-range argument                 */
  NMT_E_SHAPE = 2,       /* dimension mismatch or limit exceeded (message has both)  */
  NMT_E_INPUT = 3,       /* token id outside [0,V) or source longer than max_src_len */
  NMT_E_STATE = 4,       /* call out of sequence (e.g. step != batch step)           */
  NMT_E_FORMAT = 5,      /* bad NTSD magic / version                                 */
  NMT_E_INTEGRITY = 6,   /* missing / duplicate / mis-shaped tensor, truncated blob   */
  NMT_E_RESOURCE = 7,    /* device allocation failed at load                          */
  NMT_E_CUDA = 8,        /* CUDA error (message from cudaGetErrorString)              */
  NMT_E_UNSUPPORTED = 9  /* feature not built (e.g. precision / shape not supported)  */
} nmt_status;

typedef enum { NMT_FP32 = 0, NMT_FP16 = 1 } nmt_precision;

/* Model hyper-parameters, stored in the NTSD config block. */
typedef struct {
  int32_t enc_layers, dec_layers, d_model, n_heads, d_ffn, vocab_size;
  int32_t max_rel_pos;            /* 8: "maximum relative length was 8"        */
  int32_t use_dlcl, use_rpr, dlcl_ln;
  int32_t max_src_len, max_tgt_len; /* 120 / 200                               */
  int32_t max_pos;                /* 1024                                      */
  int32_t pad_id, unk_id, bos_id, eos_id;
  float ln_eps;                   /* 1e-5 (reading R10)                                      */
} nmt_config;

/* Sizes the arenas are allocated for (nmt_load_weights) — the paper's memory pool
 * (PAPER.md:143, :154): every device buffer of the path is carved from these arenas at load. */
typedef struct {
  int32_t max_tokens;   /* padded source tokens per batch: n_sent * s_max <= max_tokens          */
  int32_t max_sents;    /* sentences per batch (PAPER.md:138 uses 512)                           */
  int32_t max_tgt_len;  /* <= config max_tgt_len; decode steps per batch                          */
  int32_t beam;         /* 1 = greedy                                                              */
  int32_t n_workspaces; /* arenas allocated at load (0 or 1 = one, at most 16): the upper bound
                           of nmt_translate_opts.n_workers (concurrent batch workers)              */
} nmt_limits;

typedef struct nmt_model nmt_model;   /* opaque: device weights + arena */
typedef struct nmt_batch nmt_batch;   /* opaque: one encoded batch living in the model's arena */

/* Load an NTSD blob (host memory, `nbytes`; "stored in FP16").
 * Two versions are read (all little endian):
 *   v1 — the SPEC checkpoint layout: "NTSD" | u32 1 | 8 x u32 config (enc_layers,
 *        dec_layers, d_model, n_heads, d_ffn, vocab_size, max_rel_pos, flags: bit0 use_dlcl,
 *        bit1 shared_emb — must be set: the embedding is tied) | u32 n_tensors |
 *        per tensor {u16 name_len, name, u8 rank, u32 dims[rank], u8 dtype (0 F32, 1 F16),
 *        payload inline}.  Fields v1 lacks take the DESIGN.md readings: use_rpr =
 *        (max_rel_pos > 0), dlcl_ln 1, max_src_len 120, max_tgt_len 200, max_pos 1024,
 *        ids PAD 0 / UNK 1 / BOS 2 / EOS 3, ln_eps 1e-5.
 *   v2 — this build's extended layout: "NTSD" | u32 2 | u32 72 | nmt_config | u32 n |
 *        per tensor {u16 name_len, name, u8 dtype, u8 rank, u32 dims, u64 offset, u64 nbytes}
 *        | aligned payloads.
 * Tensor names are the canonical names of DESIGN.md / SURVEY Appendix B.  Weights are
 * converted to `prec` on the device; every arena (limits->n_workspaces) is allocated here.
 * Errors: NMT_E_FORMAT (magic, version, flags), NMT_E_INTEGRITY (missing / duplicate /
 * mis-shaped tensor, truncated blob, offsets outside the blob; no partial model is
 * returned), NMT_E_RESOURCE (device allocation). */
nmt_status nmt_load_weights(const void* h_ntsd, size_t nbytes, int device, nmt_precision prec,
                            const nmt_limits* lim, nmt_model** out);
nmt_status nmt_get_config(const nmt_model* m, nmt_config* out);
void nmt_free_model(nmt_model* m);

/* Parse and validate an NTSD blob on the host only (no device work): the same checks as
 * nmt_load_weights up to the device upload.  *h_n_tensors (may be NULL) receives the
 * tensor count, *h_version (may be NULL) the format version. */
nmt_status nmt_ntsd_inspect(const void* h_ntsd, size_t nbytes, nmt_config* out,
                            int64_t* h_n_tensors, int32_t* h_version);

/* Encode one batch (encoder output and per-decoder-layer cross K/V
 * are computed once here and cached).
 *   d_src     [n_sent][s_max] int32 row-major, PAD-filled, each row EOS-terminated
 *   h_src_len [n_sent] lengths incl. EOS, 1 <= len <= s_max
 *   h_tgt_cap [n_sent] per-sentence cap on generated tokens (NULL = max_tgt_len)
 * Requires n_sent <= max_sents, n_sent*s_max <= max_tokens, s_max <= max_src_len.
 * Only one batch per model may be live; encoding a new one invalidates the previous. */
nmt_status nmt_encode(nmt_model* m, const int32_t* d_src, const int32_t* h_src_len,
                      const int32_t* h_tgt_cap, int32_t n_sent, int32_t s_max, int32_t beam,
                      void* stream, nmt_batch** out);
/*   beam: 1 = greedy; 2..min(4, limits.beam) = beam search: each
 *   sentence gets `beam` consecutive live rows; nmt_decode_step then performs a whole beam
 *   step (log-softmax, top-2K, EOS finalisation, early stop "when any candidate predicts the
 *   EOS symbol, and there are no candidates with higher scores") and the batch results are
 *   the best finished hypothesis per sentence.  Teacher forcing (d_prev) is greedy-only. */

/* Copy the batch's encoder output enc [n_sent][s_max][d] as FP32 into d_dst (parity/debug). */
nmt_status nmt_batch_encoder_output(const nmt_batch* b, float* d_dst, void* stream);

/* Per-step outputs; every pointer optional (NULL = not written). Sizes are n_live rows
 * of the live batch *before* this step's pruning (beam: n_live = live sentences * K). */
typedef struct {
  int32_t* d_next;    /* [n_live]    next token per live row (greedy: argmax, ties ->
                                     lowest id; beam: the token of the hypothesis now in
                                     this row)                                         */
  int32_t* d_parent;  /* [n_live]    beam: pre-step live row this hypothesis extends
                                     (-1: row holds no continuation / sentence finished);
                                     greedy: the row itself                             */
  float* d_score;     /* [n_live]    beam: cumulative log-probability of the row's
                                     hypothesis (-inf when empty); greedy: not written  */
  uint8_t* d_done;    /* [n_live]    row finished (EOS or cap; beam: sentence search
                                     stopped) at or before this step                    */
  float* d_logits;    /* [n_live][V] FP32 logits (parity / debug; slows the step)      */
} nmt_step_out;

/* One greedy decode step t for all live rows: embed w_t, cached RPR self-attention
 * (appends k_t, v_t), cross-attention on the cached encoder K/V, FFN, final LN,
 * tied vocab projection fused with argmax.  `step` must equal the batch's step count.
 *   d_prev: [n_live] tokens w_t to feed (teacher forcing); NULL = the tokens this
 *           batch chose at step t-1 (BOS at t = 0) — the normal, sync-free path. */
nmt_status nmt_decode_step(nmt_model* m, nmt_batch* b, const int32_t* d_prev, int32_t step,
                           const nmt_step_out* out, void* stream);

/* Batch pruning (reading R18), after a decode step.
 *   d_keep == NULL: if #done >= max(1, ceil(ratio*n_live)) (ratio < 0: never, except when
 *                 every row is done), compact the live rows stably, dropping done rows.
 *   d_keep [n_live] (device, optional; greedy batches only): the caller's mask — rows with
 *                 d_keep[r] == 0 are removed (their outputs so far are final), rows with
 *                 d_keep[r] != 0 stay live in their order (a finished row that is kept keeps
 *                 its sticky done flag; its tokens are ignored); `ratio` is ignored.
 *   d_new_to_old [n_live] (optional): ascending pre-prune indices of surviving rows;
 *                 entries past the new count are -1.  Unchanged identity if no prune.
 *   h_n_live (optional): new live count — synchronises the stream when non-NULL.
 * Errors: NMT_E_STATE (no decode step since the last prune), NMT_E_UNSUPPORTED (d_keep on a
 * beam batch).  Never allocates. */
nmt_status nmt_prune_batch(nmt_model* m, nmt_batch* b, float ratio, const uint8_t* d_keep,
                           int32_t* d_new_to_old, int32_t* h_n_live, void* stream);

/* Number of live rows (synchronises the stream). */
nmt_status nmt_batch_live(nmt_batch* b, int32_t* h_n_live, void* stream);

/* Results in batch order (synchronous): h_ids [n_sent][max_tgt_len] generated tokens
 * (EOS included when produced), h_len [n_sent] generated counts. */
nmt_status nmt_batch_results(nmt_batch* b, int32_t* h_ids, int32_t* h_len, void* stream);

/* Release a batch: its arena becomes free for the next nmt_encode (no device call, no
 * free — the arena belongs to the model).  NULL is a no-op; a released or superseded batch
 * handle is rejected by every other call with NMT_E_ARG. */
void nmt_batch_free(nmt_batch* b);

typedef struct {
  int32_t max_tokens;    /* dynamic-batch token budget, <= limits */
  int32_t max_sents;     /* sentence cap per batch, <= limits     */
  int32_t prune_every;   /* decision point every c steps (>= 1)                  */
  float prune_ratio;     /* rho (0.25); < 0 = never prune                        */
  int32_t sync_every;    /* host polls the live count every k steps (>= 1)       */
  const int32_t* h_tgt_cap; /* optional [n] per-sentence caps (synthetic workloads) */
  int32_t n_workers;     /* concurrent batch workers (own arena + stream each, shared
                            weights); 0/1 = one.  Outputs do not depend on it.     */
  int32_t beam;          /* 0/1 = greedy; 2..4 = beam search     */
  int32_t nbest;         /* 0/1 = best only; 2..beam = keep the N best finished
                            hypotheses (the KD "4-best list"; reading R27) */
} nmt_translate_opts;

typedef struct {
  int64_t sentences, src_tokens, gen_tokens, out_tokens, decode_steps, prunes, batches, launches;
  int64_t truncated;            /* sources cut to max_src_len - 1 tokens + EOS (translate only) */
  int64_t arena_system_allocs;  /* cudaMalloc / cudaMallocHost calls of the model since load
                                   (weights + every arena); flat across translate calls      */
  double ms_total;              /* host wall time of the call                                 */
  double ms_encode, ms_decode;  /* device time (CUDA events on each worker's stream) summed
                                   over batches: encoder + cross K/V, and the decode loop     */
} nmt_stats;

/* Whole translation with HOST buffers (synchronous): length sort, dynamic batches,
 * encode, greedy decode with pruning, output in the original order
 * with the terminating EOS stripped.
 *   h_ids [h_off[n]] int32 flat EOS-terminated sources, h_off [n+1] int64.
 *   h_out [out_cap] receives the flat outputs, h_out_off [n+1] their offsets.
 * Sources longer than min(max_src_len, max_tokens) are truncated to that many tokens with
 * EOS last ("maximum length ... 120"; counted in stats->truncated) — a batch
 * pipeline never aborts on one long line; empty sources (len 0) are NMT_E_INPUT.
 * opts->n_workers must not exceed limits.n_workspaces (NMT_E_ARG): no arena is allocated
 * here. */
nmt_status nmt_translate(nmt_model* m, const int32_t* h_ids, const int64_t* h_off, int64_t n,
                         const nmt_translate_opts* opts, int32_t* h_out, int64_t out_cap,
                         int64_t* h_out_off, nmt_stats* stats, void* stream);

/* N-best translation (beam search, opts->beam >= opts->nbest >= 2), HOST buffers
 * (synchronous).  "We collected the 4-best list for each sentence": per
 * sentence the N best finished hypotheses, best first (score desc, ties -> earlier
 * finalised; the search stops once N are finished and the N-th best is >= every active
 * hypothesis, or at the cap — reading R27).
 *   h_out [out_cap] flat outputs of hypothesis (i, r) at index i*nbest + r (EOS stripped),
 *   h_out_off [n*nbest + 1] their offsets (an empty entry when fewer than N finished),
 *   h_score [n*nbest] (may be NULL) their scores (sum of log-probabilities; -inf if empty).
 * Errors: NMT_E_ARG for nbest outside [2, beam] or beam > limits.beam. */
nmt_status nmt_translate_nbest(nmt_model* m, const int32_t* h_ids, const int64_t* h_off, int64_t n,
                               const nmt_translate_opts* opts, int32_t* h_out, int64_t out_cap,
                               int64_t* h_out_off, float* h_score, nmt_stats* stats, void* stream);

/* Teacher ensemble ("a simple ensemble strategy"; §8(f) row f1).
 * members: 1..8 loaded models with one vocabulary, special ids, precision, device and
 * equal limits (limits.beam >= 2); they may differ in depth, DLCL and RPR (the paper's
 * 35-6 / 35-6+DLCL / 40-6 / 40-6+DLCL teachers).  The ensemble clones every member
 * (own arena, weights shared with the member) — the members must outlive it.  Per beam
 * step each member decodes its own caches and the next-token distributions are averaged:
 * log p = logsumexp_m(log_softmax(logits_m)) - log M (reading R26), then beam search
 * (reading R15) and optional N-best lists (R27) run once on the average. */
typedef struct nmt_ensemble nmt_ensemble;
nmt_status nmt_ensemble_create(nmt_model* const* members, int32_t n_members, nmt_ensemble** out);
void nmt_ensemble_free(nmt_ensemble* e);
/* Host-buffer ensemble translation (synchronous; one stream, batches in plan order).
 * opts->beam in [2, min(4, limits.beam)], opts->nbest in [0, beam].  Output layout as
 * nmt_translate_nbest with N = max(1, nbest): entry i*N + r is hypothesis r of sentence i
 * (EOS stripped), h_out_off [n*N + 1], h_score [n*N] (may be NULL) the ensemble scores. */
nmt_status nmt_translate_ensemble(nmt_ensemble* e, const int32_t* h_ids, const int64_t* h_off,
                                  int64_t n, const nmt_translate_opts* opts, int32_t* h_out,
                                  int64_t out_cap, int64_t* h_out_off, float* h_score,
                                  nmt_stats* stats, void* stream);

/* ---- Text pipeline (§8(f) row f3), host side.  "jointly byte pair encoded with 32K
 * merge operations using a shared vocabulary ... After decoding, we removed the BPE
 * separators", with the C++ subword codec of PAPER.md:141 (fastBPE
 * conventions, reading R28): pretokenised lines split on ASCII whitespace; a word starts
 * as its UTF-8 characters; the adjacent pair of lowest merge rank is merged at every
 * non-overlapping occurrence, left to right, until none applies; non-final subwords end
 * in "@@".  Vocabulary: reserved PAD, UNK, BOS, EOS = 0..3, vocabulary-file token i has
 * id 4 + i.  The codec is immutable after load (safe for concurrent use). */
typedef struct nmt_text nmt_text;
/* vocab: UTF-8, one token per line; merges: one "a b" pair per line, rank = line order,
 * "#version" lines skipped.  NMT_E_FORMAT names the offending line (malformed merge,
 * duplicate pair or token). */
nmt_status nmt_text_load(const char* vocab, int64_t vocab_len, const char* merges,
                         int64_t merges_len, nmt_text** out);
void nmt_text_free(nmt_text* t);
int32_t nmt_text_vocab_size(const nmt_text* t);   /* 4 reserved + file tokens */
/* '\n'-separated lines -> ids: BPE, token -> id (unknown -> UNK), EOS appended per line.
 * h_ids [cap] flat ids, h_off [max_lines + 1] line offsets, *n_lines the line count;
 * n_threads >= 1 host threads split the lines.  NMT_E_SHAPE if cap / max_lines are short. */
nmt_status nmt_text_encode(const nmt_text* t, const char* text, int64_t len, int32_t n_threads,
                           int32_t* h_ids, int64_t cap, int64_t* h_off, int64_t max_lines,
                           int64_t* n_lines);
/* ids -> text: per sequence stop at EOS, skip PAD / UNK / BOS, join tokens by spaces and
 * delete every "@@ "; each line '\n'-terminated into out [cap], *out_len bytes.
 * NMT_E_INPUT for an id outside [0, vocab size). */
nmt_status nmt_text_decode(const nmt_text* t, const int32_t* h_ids, const int64_t* h_off,
                           int64_t n, char* out, int64_t cap, int64_t* out_len);

/* Same with DEVICE-resident sources and outputs (inputs already in HBM):
 *   d_ids [h_off[n]] int32 flat sources on the device; h_off [n+1] host offsets (plan);
 *   d_out [n][out_stride] int32 generated tokens (EOS included if produced),
 *   d_out_len [n] generated counts; out_stride >= max_tgt_len. Asynchronous
 *   except for live-count polls (sync_every). */
nmt_status nmt_translate_device(nmt_model* m, const int32_t* d_ids, const int64_t* h_off, int64_t n,
                                const nmt_translate_opts* opts, int32_t* d_out, int32_t out_stride,
                                int32_t* d_out_len, nmt_stats* stats, void* stream);

const char* nmt_last_error(void);   /* thread-local; valid until the next nmt_* call */

/* Per-kernel-class profile, measured with CUDA events recorded on the launching stream
 * around every launch while enabled (adds two event records per launch).
 * mode: 1 = enable, 2 = reset counters and enable, 0 = reset and disable,
 *       -1 = read only, 3 = reset the step records and time decode steps only (no
 *       per-kernel events: each step's plain graph between two event nodes, see
 *       nmt_profile_steps).  When `out` is non-NULL, up to `cap` entries for the classes
 * that ran are written (read happens before any reset) and *n_out is set.
 * flops / bytes are the ALGORITHMIC work of the launches.
 * Synchronises the device. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms, flops, bytes;
} nmt_prof_entry;
nmt_status nmt_profile(nmt_model* m, int32_t mode, nmt_prof_entry* out, int32_t cap,
                       int32_t* n_out);

/* Decode steps run while profiling (translate paths; greedy and beam): for each step, the
 * step counter t and live rows entering it (read back before the step) and the device time
 * of the step as replayed in its CUDA graph, finish/prune tail included — SURVEY §8(d)
 * "ms/decode step".  Mode 3 brackets the plain step graph with two event nodes (the
 * production kernel-to-kernel transitions); modes 1 / 2 time the per-kernel-profiled
 * graph (an event pair around every kernel: longer).
 * Copies up to `cap` records in step order, sets *n_out to the number recorded since the
 * last profile reset (nmt_profile mode 0 / 2). */
typedef struct {
  int32_t t, n_live;
  float ms;
} nmt_step_rec;
nmt_status nmt_profile_steps(nmt_model* m, nmt_step_rec* out, int32_t cap, int32_t* n_out);

/* Debug timeline of the model's last fused decode-step launch (models loaded with the
 * environment variable NMT_FUSED_TRACE set; tools/fused_trace.py): per work item 4 x u64
 * {phase << 40 | row block << 20 | CTA, received, inputs ready, done} (globaltimer ns) at
 * index 4 * item, then one start time per CTA at 4 * 65536 + CTA.  Synchronises the device.
 * NMT_E_STATE when the model was loaded without the variable. */
nmt_status nmt_debug_fused_trace(nmt_model* m, uint64_t* h_out, int64_t cap);

/* Debug timeline of the last tcgen05 encoder-attention launch (NMT_ENC_ATTN=2 with the
 * environment variable NMT_ATTN_TRACE set at the first launch): CTA 0, per local tile k < 64,
 * 8 globaltimer stamps {Q/K TMA, V TMA, QK^T issued, S seen, P ready, P V issued, O seen,
 * TMEM freed} at h_out[8k + e].  Synchronises the device. */
nmt_status nmt_debug_attn_trace(uint64_t* h_out, int64_t cap);

/* Debug timeline of the persistent tcgen05 GEMM (environment variable NMT_GEMM_TRACE set at
 * the launch; single-CTA units): for CTA c < 148 and its local unit k < 32, 8 globaltimer
 * stamps at h_out[(c*32 + k)*8 + e]: {producer first / last load of the unit, MMA accumulator
 * free / last commit, epilogue warp 4 waits / sees the accumulator, releases it, issues the
 * unit's last store}.  Stamps persist until overwritten.  Synchronises the device. */
nmt_status nmt_debug_gemm_trace(uint64_t* h_out, int64_t cap);

/* ---- kernel-level entry points used by the unit parity tests ------------------- */
/* C[M][N] = A[M][K] * B[N][K]^T (+bias[N]) (+R[M][N]) (relu) in the model precision
 * (FP16: tcgen05/TMEM/TMA tensor-core GEMM; FP32: SIMT), all pointers device, row-major
 * with leading dimensions lda/ldb/ldr/ldc in elements.  `prec` selects the element
 * type of A, B, bias, R and C.  Asynchronous. */
nmt_status nmt_dev_gemm(nmt_precision prec, int32_t M, int32_t N, int32_t K, const void* d_A,
                        int32_t lda, const void* d_B, int32_t ldb, const void* d_bias,
                        const void* d_R, int32_t ldr, void* d_C, int32_t ldc, int32_t relu,
                        void* stream);
/* Same GEMM in the decode-step configuration (FP16 only): 64-wide tiles and the
 * deterministic split-K factor the decoder uses for this (N, K) (partials reduced in split
 * order by the last-arriving CTA).  Uses a library-owned workspace; M <= 16384. */
nmt_status nmt_dev_gemm_decode(int32_t M, int32_t N, int32_t K, const void* d_A, int32_t lda,
                               const void* d_B, int32_t ldb, const void* d_bias, const void* d_R,
                               int32_t ldr, void* d_C, int32_t ldc, int32_t relu, void* stream);
/* Fused vocab projection + argmax: d_next[m] = argmax_n (A[m] . B[n]) with ties to the
 * lowest n, FP32 accumulation; optional FP32 logits dump.  M <= 16384. */
nmt_status nmt_dev_gemm_argmax(nmt_precision prec, int32_t M, int32_t N, int32_t K,
                               const void* d_A, int32_t lda, const void* d_B, int32_t ldb,
                               int32_t* d_next, float* d_logits, void* stream);

/* Encoder RPR self-attention alone (Shaw et al. with clipped relative keys AND values,
 * PAPER.md:23, :34; reading R7): for sentence b, head h, query i < len[b]:
 *   e_ij = q_i . (k_j + A^K[r(i,j)]) / sqrt(dh),  r(i,j) = clip(j - i, -k, k) + k, j < len[b]
 *   o_i  = sum_j softmax_j(e_i) (v_j + A^V[r(i,j)]);   rows i >= len[b] are written 0.
 * d_qkv [B*S][3d] (Q | K | V, head h at columns h*dh of each third), d_len int32 [B]
 * (device), d_relk / d_relv [2k+1][dh] (may be NULL when use_rpr = 0), d_out [B*S][d];
 * all device memory in the precision `prec`, row-major, owned by the caller.  S <= 128.
 * FP16: tensor-core kernel (TMA-fed pipeline for dh = 64).  Asynchronous on `stream`. */
nmt_status nmt_dev_attn_encoder(nmt_precision prec, int32_t B, int32_t S, int32_t d, int32_t H,
                                int32_t kclip, int32_t use_rpr, const void* d_qkv,
                                const int32_t* d_len, const void* d_relk, const void* d_relv,
                                void* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NMT_H_ */
