// kernels.h — launchers for every sm_100a kernel of the hot path.
// Each launcher cites the PAPER.md passage / DESIGN.md reading of the step it computes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nmt {

struct DevState;

// ---------------------------------------------------------------- GEMM family
// C[M][N] = A[M][K] . B[N][K]^T (+bias[N]) (+R[M][N]) (ReLU), FP32 accumulation
// (reductions in FP32).  A, B, bias, R, C are element type T.
// If dM != nullptr the effective M is min(M, *dM) (live rows read from the device,
// so decode steps need no host round-trip).  argmax != nullptr switches to the
// vocab epilogue: logits are not stored in C; per row, the packed (value, ~id)
// maximum is atomically max-reduced into argmax[m] (no log_softmax
// for greedy); logits (FP32, ld = N) is an optional dump.
struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr; int lda = 0;
  const void* B = nullptr; int ldb = 0;
  const void* bias = nullptr;
  const void* R = nullptr; int ldr = 0;
  void* C = nullptr; int ldc = 0;
  int relu = 0;
  const int* dM = nullptr;
  unsigned long long* argmax = nullptr;
  float* logits = nullptr;
  // beam epilogue (FP16 tcgen05 path): per (row, 256-column segment) log-sum-exp partial and
  // top-8 candidates instead of logits, [M][ceil(N/256)][2 + 16] floats (beam_merge)
  float* beam_part = nullptr;
  // tcgen05 path only: output tile width (128, or 64 for decode-size GEMMs) and a
  // deterministic split-K factor with its FP32 workspace / self-resetting counters.
  int tile_n = 256;
  int splits = 1;
  float* ws = nullptr;
  int* counters = nullptr;
  // LayerNorm folded into the GEMM (FP16 tcgen05 path):
  // producer: per-row (mean, M2) of every 32 FP16-rounded output columns -> st_out[M][N/32];
  // consumer: A = the raw residual stream x, B = W o gamma, bias = b + W beta, and the
  // epilogue applies y = rstd (acc - mu c[n]) + bias with (mu, rstd) merged from ln_st.
  float2* st_out = nullptr;
  const float2* ln_st = nullptr;
  const float* ln_c = nullptr;
  float ln_eps = 0.f;
};

// Split-K factor for a decode-size GEMM of shape (N, K) with 64-wide tiles: a function of
// the weight shape only (never of the live-row count), so results are batch invariant.
int decode_splits(int N, int K);
// Decode-step GEMM configuration (tile width, split-K factor) from the weight shape only.
void decode_config(GemmArgs& a);
// LN folding at load time (FP16): Wf = W o g, c[n] = sum_k Wf[n][k], bf = bias + W beta.
void fold_ln(const void* W, const void* g, const void* beta, const void* bias, int N, int K,
             void* Wf, float* c, void* bf, cudaStream_t s);

template <class T> void gemm_simt(const GemmArgs& a, cudaStream_t s);
void gemm_tc(const GemmArgs& a, cudaStream_t s);   // FP16 tcgen05 / TMEM / TMA
template <class T> void gemm(const GemmArgs& a, cudaStream_t s);  // product dispatch by T

// ---------------------------------------------------------------- elementwise / LN
// y0[r] = sqrt(d) * E[id(r)] + PE[pos(r)]   (tied embedding + sinusoid)
// encoder: rows r = b*S + p, pos = p;  decoder: pos = *d_t, ids = tokens[r], rows < *dR.
template <class T>
void embed(const int* ids, const T* E, const float* pe, T* out, int rows, int d, int S,
           const int* d_t, const int* dR, float scale, cudaStream_t s);

// out = LN(in; g, b) row-wise, FP32 statistics
template <class T>
void layernorm(const T* in, int ldi, const T* g, const T* b, T* out, int ldo, int rows, int d,
               float eps, const int* dR, cudaStream_t s);

// DLCL combine (Eq. 1-2), one launch per layer boundary l:
//   z_l = LN^dl_l(y_l) -> hist[l];  x = sum_{k<=l} w[k] z_k;  (x -> xout, LN(x; g2,b2) -> uout)
// dlcl_ln = 0: z_l = y_l (reading A22 test switch).
// Lookahead in blocks of boundaries (d = 256 / 512 only: dlcl_lookahead_ok; x is the same
// in every mode): mode 1 (a block's first boundary) also writes the FP32 partials
// P_i = sum_{k<=l} W^(l+1+i)[k] z_k, i = 1..arg (arg <= 3), at P + (i-1)*rows*d (wall = the
// packed weight rows, row r at r(r-1)/2); mode 2 (a later boundary of the block) computes
// x = P + sum_{k=l-arg}^{l-1} w[k] z_k + w[l] z_l from its partial and the arg history rows
// written since the block started.
bool dlcl_lookahead_ok(int d);
template <class T>
void dlcl_combine(const T* y, T* hist, size_t hist_stride, int l, const float* w, const T* gdl,
                  const T* bdl, int dlcl_ln, const T* g2, const T* b2, T* xout, T* uout, int rows,
                  int d, float eps, cudaStream_t s, int mode = 0, const float* wall = nullptr,
                  float* P = nullptr, int arg = 0);

// ---------------------------------------------------------------- attention
// Encoder RPR self-attention (Shaw et al.) per (sentence, head):
// qkv [B*S][3d]; out [B*S][d]; key mask j < len[b]; rows p >= len[b] are written 0.
template <class T>
void attn_encoder(const T* qkv, const int* len, const T* relk, const T* relv, T* out, int B,
                  int S, int d, int H, int kclip, int use_rpr, cudaStream_t s);

// tcgen05 / TMEM encoder attention (attention_umma.cu): dh = 64, S <= 128, k <= 8, RPR on.
void attn_encoder_umma(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                       __half* out, int B, int S, int d, int H, int kclip, cudaStream_t s);
void attn_umma_trace(unsigned long long* h_out, int cap);   // debug (nmt_debug_attn_trace)
namespace tc {
void gemm_trace(unsigned long long* h_out, int cap);   // debug (nmt_debug_gemm_trace)
}
// FP16 path of attn_encoder: Q K^T, q.A^K and P V + B A^V on tensor cores (attention_tc.cu).
void attn_encoder_tc(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                     __half* out, int B, int S, int d, int H, int kclip, int use_rpr,
                     cudaStream_t s);

// Decoder cached self-attention at step t = *d_t: for live row r
// (< *dR), slot = row_slot[r]; appends k_t, v_t (from qkv[r]) into the cache at
// [slot][t] and attends over positions 0..t with r(i,j) = clip(j - t, -k, k) + k.
// cache layout: K at kc + (slot*Tmax + j)*d, V at vc + ... (same).
// anc (beam, optional): [slot][Tmax] ancestry — position j < t of this hypothesis lives in
// slot anc[slot][j] (beam reorder without K/V copies).
template <class T>
void attn_decoder_self(const T* qkv, T* kc, T* vc, int Tmax, const int* row_slot, const T* relk,
                       const T* relv, T* out, int rows, int d, int H, int kclip, int use_rpr,
                       const int* d_t, const int* dR, const int* anc, cudaStream_t s);

// Cross-attention over the once-per-sentence encoder K/V:
// keys at ckv + (sent*S + j)*ldkv + koff, values at + voff, sent = row_slot[r] / beam;
// mask j < src_len[sent]; S = *dS read on the device (graph-replayable), Smax sizes smem.
template <class T>
void attn_cross(const T* q, const T* ckv, int ldkv, int koff, int voff, const int* dS, int Smax,
                const int* src_len, const int* row_slot, T* out, int rows, int d, int H,
                const int* dR, int beam, cudaStream_t s);

// ---------------------------------------------------------------- beam search (beam.cu)
// FP32 logits [rows][V] -> per row the top-KB log-probs (value desc, id asc), LSE in FP32.
void beam_row_topk(const float* logits, int V, int KB, const int* dR, int rows_upper,
                   float* cand_v, int* cand_i, cudaStream_t s);
// Per sentence (K consecutive live rows): top-2K candidates, EOS finalisation, early stop
// (PAPER.md:103), new rows (tokens, scores, ancestry / token histories), winner written to
// out_tok / gen_len of the sentence slot.  NB > 1 also keeps the NB best finished
// hypotheses (reading R27): nb_score / nb_len [B][NB], nb_tok [B][NB][Tmax], nb_cnt [B].
void beam_select(int K, const float* cand_v, const int* cand_i, float* score, int* prev_tok,
                 uint8_t* done, const int* row_slot, const int* cap, int* anc, int* htok,
                 int Tmax, float* best_score, int* out_tok, int* gen_len, DevState* st,
                 int V, int eos, int rows_upper, cudaStream_t s, int NB = 1,
                 float* nb_score = nullptr, int* nb_len = nullptr, int* nb_tok = nullptr,
                 int* nb_cnt = nullptr, int* parent_out = nullptr);
// Merge of the vocab GEMM's beam epilogue partials (GemmArgs::beam_part, nseg segments of
// 256 columns per row): per row LSE = M + log sum_i s_i exp(m_i - M) and the top-KB
// candidates (value desc, id asc) as log-probabilities -> cand_v / cand_i (= beam_row_topk).
void beam_merge(const float* part, int nseg, int KB, const int* dR, int rows_upper, float* cand_v,
                int* cand_i, cudaStream_t s);
// Teacher ensemble (reading R26): ens[r][v] = logsumexp_m(log_softmax(logits_m[r])[v]) - log M.
void ens_combine(const float* const* logits, int nm, int V, const int* dR, int rows_upper,
                 float* ens, cudaStream_t s);
void beam_init(int* row_slot, int* prev_tok, uint8_t* done, float* score, int* htok, int Tmax,
               float* best_score, int* gen_len, DevState* st, int B, int K, int S, int bos,
               cudaStream_t s, int* nb_cnt = nullptr);

// Decoder input + first pre-norm, fused (one warp per live row):
//   g = sqrt(d) E[w_r] + PE(t),  u = LN(g; gam, bet)     (t = *d_t)
template <class T>
void embed_dec_ln(const int* ids, const T* E, const float* pe, const T* gam, const T* bet, T* g,
                  T* u, int rows, int d, float scale, float eps, const int* d_t, const int* dR,
                  cudaStream_t s);

// ---------------------------------------------------------------- greedy bookkeeping
// Batch state on the device (one int32 block):
struct DevState {
  int t;          // current decode step
  int n_live;     // live rows
  int n_done;     // done rows among live ones (sticky flags)
  int prunes;     // number of compactions so far
  int S;          // padded source length of the batch (cross-attention stride)
};

// After the vocab argmax of step t: next token per live row, sticky done flag
// (EOS or cap, reading R12), outputs per sentence slot.
void greedy_finish(unsigned long long* keys, const int* force_next, int* prev_tok, uint8_t* done,
                   const int* row_slot, const int* cap, int* out_tok, int out_stride, int* gen_len,
                   DevState* st, int rows_upper, int eos, int* d_next_copy, uint8_t* d_done_copy,
                   cudaStream_t s);

// Batch pruning decision + stable compaction (reading R18), one CTA.
// Advances st->t.  new_to_old (optional) receives the map (or identity) for the
// pre-prune rows; entries >= new count are -1.
void prune_compact(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, int every,
                   float ratio, int* new_to_old, int rows_upper, cudaStream_t s,
                   float* score = nullptr /* beam: per-row scores compacted alongside */);

// Caller-mask compaction (nmt_prune_batch d_keep): rows with keep[r] == 0 are removed,
// survivors keep their order and sticky done flags; n_done is recounted.  Advances st->t.
void prune_keep(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, const uint8_t* keep,
                int* new_to_old, int rows_upper, cudaStream_t s);
// Step outputs for rows < n_live: d_next = prev_tok, d_score = score, d_done = done (beam);
// d_parent_identity[r] = r (greedy: every row extends itself).  Null pointers are skipped.
void step_outputs(const DevState* st, const int* prev_tok, const float* score, const uint8_t* done,
                  int* d_next, float* d_score, uint8_t* d_done, int rows_upper, cudaStream_t s,
                  int* d_parent_identity = nullptr);

// greedy_finish + prune_compact fused into one single-CTA launch (translate loop).
void finish_prune(unsigned long long* keys, int* prev_tok, uint8_t* done, int* row_slot,
                  const int* cap, int* out_tok, int out_stride, int* gen_len, DevState* st,
                  int eos, int every, float ratio, int rows_upper, cudaStream_t s);

// Fresh batch state: row_slot[r] = r, prev_tok[r] = BOS, done = 0, gen_len = 0,
// st = {t 0, n_live B, n_done 0, prunes 0}.
void batch_init(int* row_slot, int* prev_tok, uint8_t* done, int* gen_len, DevState* st, int B,
                int S, int bos, cudaStream_t s);

// Scatter a finished batch's per-slot outputs to their original sentence ids.
void scatter_outputs(const int* out_tok, int out_stride, const int* gen_len, const int* sent_ids,
                     int B, int* d_out, int d_out_stride, int* d_out_len, cudaStream_t s);

// Pack flat EOS-terminated device sources into padded [B][S]: row b copies blen[b]
// ids from ids + boff[b]; PAD elsewhere.  Ids outside [0, V) set *bad |= 1.
// blen[b] < 0 marks a truncated source: |blen[b]| - 1 ids, then `eos`.
void pack_sources(const int* ids, const long long* boff, const int* blen, int B, int S, int* out,
                  int vocab, int* bad, int eos, cudaStream_t s);

// Convert a [rows][d] T buffer to FP32 (debug / parity output).
template <class T> void to_float(const T* in, float* out, size_t n, cudaStream_t s);
// Convert packed argmax keys to token ids.
void argmax_ids(unsigned long long* keys, int* ids, int rows, cudaStream_t s);

}  // namespace nmt
