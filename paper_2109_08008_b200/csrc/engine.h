// engine.h — internal state of libnmt: model (weights + arena, the paper's memory pool,
// PAPER.md:143), batch, profiler, decode-step graph cache.  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/nmt.h"
#include "common.cuh"
#include "decode_fused.h"
#include "kernels.h"

namespace nmt {

struct NmtError : std::runtime_error {
  nmt_status code;
  NmtError(nmt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define NMT_REQUIRE(cond, code, msg)                             \
  do {                                                           \
    if (!(cond)) throw ::nmt::NmtError(code, std::string(msg)); \
  } while (0)

struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  size_t take(size_t bytes) {
    size_t off = used;
    used += (bytes + 255) & ~size_t(255);
    return off;
  }
};

// Device pointers of one encoder layer l (0-based; the paper's layer l+1).
struct EncW {
  const void *attn_g, *attn_b, *qkv_w, *qkv_b, *out_w, *out_b, *relk, *relv, *ffn_g, *ffn_b, *w1,
      *b1, *w2, *b2;
  const void *dl_g, *dl_b;  // LN^dl_{l+1} (applied to y_{l+1}), DLCL only
};
// LN-folded decoder weights (FP16 path, see fold_ln): B operand, c[n], folded bias.
struct FoldW {
  const void* w = nullptr;
  const float* c = nullptr;
  const void* b = nullptr;
};
struct DecFold {
  FoldW qkv, cq, w1;   // behind LN_self (layers >= 1), LN_cross, LN_ffn
};
struct DecW {
  const void *self_g, *self_b, *qkv_w, *qkv_b, *so_w, *so_b, *relk, *relv, *cross_g, *cross_b,
      *cq_w, *cq_b, *co_w, *co_b, *ffn_g, *ffn_b, *w1, *b1, *w2, *b2;
};

enum ProfClass {
  P_ENC_GEMM = 0, P_ENC_ATTN, P_DLCL, P_ENC_LN, P_EMBED, P_DEC_GEMM, P_VOCAB, P_DEC_SELF,
  P_DEC_CROSS, P_DEC_LN, P_BOOK, P_DEC_FUSED, P_NCLS
};
extern const char* kProfNames[P_NCLS];

}  // namespace nmt

struct nmt_batch {
  nmt_model* m = nullptr;
  int B = 0, S = 0;
  int step = 0;          // host mirror of decode steps issued
  int rows_upper = 0;    // host upper bound of live rows (grid sizing)
  int max_cap = 0;
  int K = 1;             // beam width (1 = greedy)
  int NB = 1;            // finished hypotheses kept per sentence (n-best, <= K)
  bool valid = false;
  bool pending_step_done = false;  // nmt_decode_step issued, nmt_prune_batch not yet
};

struct nmt_model {
  nmt_config cfg{};
  nmt_precision prec = NMT_FP16;
  nmt_limits lim{};
  int device = 0;
  size_t tb = 2;  // bytes per stored element
  // weights
  void* wbuf = nullptr;
  std::unordered_map<std::string, void*> W;
  std::vector<nmt::EncW> enc;
  std::vector<nmt::DecW> dec;
  const void *emb = nullptr, *dl0_g = nullptr, *dl0_b = nullptr, *enc_fg = nullptr,
             *enc_fb = nullptr, *dec_fg = nullptr, *dec_fb = nullptr;
  void* ckv_w = nullptr;   // [Ld*2d][d] cross K/V projection of every decoder layer
  void* ckv_b = nullptr;   // [Ld*2d]
  float* dlcl_w = nullptr; // packed rows m = 1..L+1 (row m at offset m(m-1)/2)
  float* pe = nullptr;     // [max_pos][d] FP32 sinusoid table
  // LN folding (FP16): per decoder layer (LN_self of layers >= 1, LN_cross, LN_ffn)
  void* foldbuf = nullptr;
  std::vector<nmt::DecFold> fold;
  // arena
  nmt::Arena ar;
  int *src = nullptr, *src_len = nullptr, *tgt_cap = nullptr;
  void *x = nullptr, *u = nullptr, *qkv = nullptr, *o = nullptr, *h = nullptr, *enc_out = nullptr,
       *hist = nullptr, *ckv = nullptr;
  void *g = nullptr, *du = nullptr, *dqkv = nullptr, *dout = nullptr, *dq = nullptr, *dh = nullptr;
  void *kc = nullptr, *vc = nullptr;
  unsigned long long* keys = nullptr;
  int *row_slot = nullptr, *prev_tok = nullptr, *out_tok = nullptr, *gen_len = nullptr;
  uint8_t* done = nullptr;
  nmt::DevState* st = nullptr;
  int* bad = nullptr;
  long long* boff = nullptr;
  int* blen = nullptr;
  int* sent_ids = nullptr;
  float* gemm_ws = nullptr;   // split-K partials of the decode GEMMs
  int* gemm_cnt = nullptr;    // split-K arrival counters (self-resetting)
  // beam search state (allocated when limits.beam > 1)
  float* bscore = nullptr;    // [R] cumulative log-prob per live row
  int* anc = nullptr;         // [R][Tmax] ancestry (slot holding position j)
  int* htok = nullptr;        // [R][Tmax] token history per slot (j = 0: BOS)
  float* best_score = nullptr;  // [max_sents] best finished hypothesis score
  float* nb_score = nullptr;  // [max_sents][beam] n-best finished scores (desc)
  int* nb_len = nullptr;      // [max_sents][beam] their generated lengths
  int* nb_tok = nullptr;      // [max_sents][beam][Tmax] their tokens
  int* nb_cnt = nullptr;      // [max_sents] list sizes
  float* blogits = nullptr;   // [R][V] FP32 logits of the step
  float* bpart = nullptr;     // [R][ceil(V/256)][18] beam-epilogue partials (FP16 beam)
  bool beam_epi = false;      // FP16 beam steps use the fused epilogue (opt-in: env NMT_BEAM_EPI)
  float2* lnst = nullptr;     // [R][d/32] row-chunk (mean, M2) of the decoder residual stream
  float* dlcl_p = nullptr;    // [blk-1][N][d] FP32 DLCL lookahead partials (kernels.h dlcl_combine)
  int* fused_ctr = nullptr;   // fused decode step: item / completion counters (decode_fused.cu)
  // fused decode step policy, read at load: live rows up to which one launch runs every
  // phase (env NMT_FUSE_ROWS; above it fused GEMM segments around the standalone attention
  // kernels); -1 = the unfused step (default, and env NMT_NO_FUSE)
  int fuse_rows = -1;
  unsigned long long* fused_trace = nullptr;   // NMT_FUSED_TRACE: timeline of the last fused launch
  std::unique_ptr<nmt::FusedParams> fused;   // its parameter block (built on first use)
  float* cand_v = nullptr;    // [R][2K] top log-probs per row
  int* cand_i = nullptr;      // [R][2K] their token ids
  // pinned host staging
  struct Pinned {
    int* src; int* len; int* cap; long long* boff; int* blen; int* sent; int* out_tok; int* gen_len;
    nmt::DevState* st; int* bad;
  } hp{};
  void* pinned = nullptr;
  nmt_batch batch;
  // per-kernel-class CUDA-event profile (bench roofline)
  struct ProfRec { int cls; cudaEvent_t a, b; double flops, bytes; };
  struct Prof {
    bool on = false;
    bool steps_only = false;   // mode 3: per-step device time only (no per-kernel events)
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<ProfRec> pending;
    double ms[16] = {}, flops[16] = {}, bytes[16] = {};
    long long n[16] = {};
    // per decode step while profiling: (t, live rows, device ms of the step's kernels)
    struct Step { int t, live; float ms; };
    std::vector<Step> steps;
  } prof;
  // decode-step CUDA graphs keyed by (rows bucket, prune_every, prune_ratio bits), with the
  // number of kernel nodes each replay launches (nmt_stats.launches)
  std::map<std::tuple<int, int, unsigned, int>, std::pair<cudaGraphExec_t, int>> graphs;
  std::set<std::tuple<int, int, unsigned, int>> eager_keys;  // configurations run eagerly once
  // profiled variants of the step graphs: the graph plus its per-launch event pairs
  std::map<std::tuple<int, int, unsigned, int>,
           std::pair<cudaGraphExec_t, std::vector<ProfRec>>> pgraphs;
  // step-timed variants (profile mode 3): the plain step graph between two event nodes
  std::map<std::tuple<int, int, unsigned, int>, std::pair<cudaGraphExec_t, ProfRec>> sgraphs;
  // Concurrent batch workers (the GPU analog of the paper's parallel decoding processes,
  // PAPER.md:129-131): clones sharing this model's weights, each with its own arena,
  // stream, batch state and graphs.  Allocated at load (nmt_limits.n_workspaces - 1 clones).
  bool owns_weights = true;
  std::vector<nmt_model*> workers;
  cudaStream_t own_stream = nullptr;
  // decode phase on a high-priority stream (translate loop): a batch's latency-bound decode
  // steps are scheduled ahead of the other workers' encoder kernels when SMs free up
  cudaStream_t dec_stream = nullptr;
  cudaEvent_t ev_enc = nullptr, ev_dec = nullptr;
  // memory-pool accounting (nmt_stats.arena_system_allocs): cudaMalloc / cudaMallocHost calls
  int64_t sys_allocs = 0;
  // per-batch device timing of the translate loop (nmt_stats.ms_encode / ms_decode):
  // before encode, after encode, after the decode loop
  cudaEvent_t ev_t[3] = {nullptr, nullptr, nullptr};
  ~nmt_model() {
    for (auto e : ev_t)
      if (e) cudaEventDestroy(e);
    if (dec_stream) cudaStreamDestroy(dec_stream);
    if (ev_enc) cudaEventDestroy(ev_enc);
    if (ev_dec) cudaEventDestroy(ev_dec);
    for (auto* w : workers) delete w;
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
    for (auto& kv : pgraphs) {
      cudaGraphExecDestroy(kv.second.first);
      for (auto& r : kv.second.second) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
      }
    }
    for (auto& kv : sgraphs) {
      cudaGraphExecDestroy(kv.second.first);
      cudaEventDestroy(kv.second.second.a);
      cudaEventDestroy(kv.second.second.b);
    }
    for (auto e : prof.pool) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (wbuf && owns_weights) cudaFree(wbuf);
    if (foldbuf && owns_weights) cudaFree(foldbuf);
    if (ar.base) cudaFree(ar.base);
    if (fused_trace) cudaFree(fused_trace);
    if (pinned) cudaFreeHost(pinned);
  }
};

// Teacher ensemble: one clone per member (own arena + caches, shared
// weights); the search state (row_slot, tokens, scores, ancestry, DevState ...) of clones
// 1.. aliases clone 0's, so one beam search drives every member's decoder.
struct nmt_ensemble {
  std::vector<nmt_model*> members;
  float* ens = nullptr;   // [R][V] FP32 ensemble log-probabilities of the step
  // whole-ensemble decode steps (every member's decoder, the averaging, the beam update and
  // pruning) as CUDA graphs keyed by (rows bucket, n-best, prune cadence, ratio bits), with
  // their kernel-node counts; configurations run eagerly once first
  std::map<std::tuple<int, int, int, unsigned>, std::pair<cudaGraphExec_t, int>> graphs;
  std::set<std::tuple<int, int, int, unsigned>> eager_keys;
  ~nmt_ensemble() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
    for (auto* c : members) delete c;
    if (ens) cudaFree(ens);
  }
};

namespace nmt {
// Every C-ABI entry point runs its body through guard(): exceptions become status codes,
// the message goes to the thread-local last error (nmt_last_error).
std::string& last_error();
template <class F> nmt_status guard(F f) {
  try {
    last_error().clear();
    f();
    return NMT_OK;
  } catch (const NmtError& e) {
    last_error() = e.what();
    return e.code;
  } catch (const CudaError& e) {
    last_error() = e.what();
    return NMT_E_CUDA;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return NMT_E_ARG;
  }
}
// forward.cu
void encode_any(nmt_model* m, int B, int S, cudaStream_t s);
// finish = false leaves the greedy bookkeeping to a following finish_prune launch.
void decode_step_any(nmt_model* m, nmt_batch* b, const int* d_prev, const nmt_step_out* out,
                     cudaStream_t s, bool finish = true);
void prof_flush(nmt_model* m);
// DLCL lookahead block size (kernels.h dlcl_combine): 1 = none (no DLCL, d not 256 / 512,
// or NMT_NO_DLCL_LA); NMT_DLCL_LA = 1..4 overrides the default for A/B runs.
constexpr int kDlclBlock = 4;   // measured: 2 -> 513 ms, 3 -> 597 ms, 4 -> 475 ms DLCL per 192000-sentence chunk
int dlcl_blocks(const nmt_config& c, int d);
// While a profiled decode step is being captured, its event pairs are recorded as external
// event nodes of the graph (replayed and read after every launch of that graph).
extern thread_local std::vector<nmt_model::ProfRec>* g_prof_capture;
template <class F>
void prof_run(nmt_model* m, int cls, double flops, double bytes, cudaStream_t s, F&& f) {
  auto& P = m->prof;
  if (!P.on || P.steps_only) {
    f();
    return;
  }
  if (g_prof_capture) {
    cudaEvent_t a, b;
    NMT_CUDA(cudaEventCreate(&a));
    NMT_CUDA(cudaEventCreate(&b));
    NMT_CUDA(cudaEventRecordWithFlags(a, s, cudaEventRecordExternal));
    f();
    NMT_CUDA(cudaEventRecordWithFlags(b, s, cudaEventRecordExternal));
    g_prof_capture->push_back({cls, a, b, flops, bytes});
    return;
  }
  while (P.pool.size() < P.used + 2) {
    cudaEvent_t e;
    NMT_CUDA(cudaEventCreate(&e));
    P.pool.push_back(e);
  }
  cudaEvent_t a = P.pool[P.used++], b = P.pool[P.used++];
  NMT_CUDA(cudaEventRecord(a, s));
  f();
  NMT_CUDA(cudaEventRecord(b, s));
  P.pending.push_back({cls, a, b, flops, bytes});
}
// Runs one launch; when profiling, brackets it with stream events and records its
// ALGORITHMIC FLOPs / bytes.
#define PROF(cls, fl, by, stmt) \
  ::nmt::prof_run(m, cls, (double)(fl), (double)(by), s, [&] { stmt; })
}  // namespace nmt
