// engine.cu — NTSD loader, arena (the paper's memory pool), batch planning
// (PAPER.md:121, :138, :154), translate drivers with device-side pruning and CUDA-graph
// decode steps, and the extern "C" ABI of include/nmt.h.  Host code only plans and
// orchestrates; every step of the path runs in kernels on the device.
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <mutex>
#include <thread>

#include "engine.h"

namespace nmt {
std::atomic<unsigned long long> g_launches{0};
thread_local bool g_pdl = false;
thread_local std::vector<nmt_model::ProfRec>* g_prof_capture = nullptr;
thread_local std::string g_err;
int dlcl_blocks(const nmt_config& c, int d) {
  static const int blk = [] {
    if (getenv("NMT_NO_DLCL_LA")) return 1;
    const char* e = getenv("NMT_DLCL_LA");
    const int v = e ? atoi(e) : kDlclBlock;
    return v < 1 ? 1 : v > 4 ? 4 : v;
  }();
  return c.use_dlcl && dlcl_lookahead_ok(d) ? blk : 1;
}

}  // namespace nmt

using namespace nmt;

namespace {

// ------------------------------------------------------------------ NTSD parsing
struct TensorRec {
  std::string name;
  int dtype;  // 0 f32, 1 f16
  std::vector<uint32_t> dims;
  const uint8_t* data;
  size_t nbytes;
};

std::vector<std::pair<std::string, std::vector<uint32_t>>> canonical(const nmt_config& c) {
  std::vector<std::pair<std::string, std::vector<uint32_t>>> s;
  const uint32_t d = c.d_model, F = c.d_ffn, V = c.vocab_size, R = 2 * c.max_rel_pos + 1,
                 dh = c.d_model / c.n_heads;
  auto add = [&](const std::string& n, std::vector<uint32_t> sh) { s.emplace_back(n, sh); };
  add("emb", {V, d});
  for (int l = 0; l < c.enc_layers; ++l) {
    std::string p = "enc." + std::to_string(l) + ".";
    add(p + "attn_ln.g", {d}); add(p + "attn_ln.b", {d});
    add(p + "qkv.w", {3 * d, d}); add(p + "qkv.b", {3 * d});
    add(p + "out.w", {d, d}); add(p + "out.b", {d});
    if (c.use_rpr) { add(p + "rel_k", {R, dh}); add(p + "rel_v", {R, dh}); }
    add(p + "ffn_ln.g", {d}); add(p + "ffn_ln.b", {d});
    add(p + "ffn1.w", {F, d}); add(p + "ffn1.b", {F});
    add(p + "ffn2.w", {d, F}); add(p + "ffn2.b", {d});
  }
  if (c.use_dlcl) {
    for (int k = 0; k <= c.enc_layers; ++k) {
      add("enc.dlcl.ln." + std::to_string(k) + ".g", {d});
      add("enc.dlcl.ln." + std::to_string(k) + ".b", {d});
    }
    uint32_t L1 = c.enc_layers + 1;
    add("enc.dlcl.w", {L1 * (L1 + 1) / 2});
  }
  add("enc.final_ln.g", {d}); add("enc.final_ln.b", {d});
  for (int m = 0; m < c.dec_layers; ++m) {
    std::string p = "dec." + std::to_string(m) + ".";
    add(p + "self_ln.g", {d}); add(p + "self_ln.b", {d});
    add(p + "self_qkv.w", {3 * d, d}); add(p + "self_qkv.b", {3 * d});
    add(p + "self_out.w", {d, d}); add(p + "self_out.b", {d});
    if (c.use_rpr) { add(p + "rel_k", {R, dh}); add(p + "rel_v", {R, dh}); }
    add(p + "cross_ln.g", {d}); add(p + "cross_ln.b", {d});
    add(p + "cross_q.w", {d, d}); add(p + "cross_q.b", {d});
    add(p + "cross_kv.w", {2 * d, d}); add(p + "cross_kv.b", {2 * d});
    add(p + "cross_out.w", {d, d}); add(p + "cross_out.b", {d});
    add(p + "ffn_ln.g", {d}); add(p + "ffn_ln.b", {d});
    add(p + "ffn1.w", {F, d}); add(p + "ffn1.b", {F});
    add(p + "ffn2.w", {d, F}); add(p + "ffn2.b", {d});
  }
  add("dec.final_ln.g", {d}); add("dec.final_ln.b", {d});
  return s;
}

template <class U> U rd(const uint8_t*& p, const uint8_t* end) {
  NMT_REQUIRE(p + sizeof(U) <= end, NMT_E_INTEGRITY, "NTSD: truncated blob");
  U v;
  memcpy(&v, p, sizeof(U));
  p += sizeof(U);
  return v;
}

float half_bits_to_float(uint16_t h) {
  __half_raw r;
  r.x = h;
  return __half2float(__half(r));
}
uint16_t float_to_half_bits(float f) {
  __half hv = __float2half_rn(f);
  __half_raw r = hv;
  return r.x;
}

void validate_config(const nmt_config& c) {
  NMT_REQUIRE(c.enc_layers >= 1 && c.dec_layers >= 1 && c.n_heads >= 1 && c.vocab_size >= 8,
              NMT_E_FORMAT, "NTSD: bad layer/head/vocab counts");
  NMT_REQUIRE(c.d_model % 32 == 0 && c.d_model <= 512 && c.d_model % c.n_heads == 0,
              NMT_E_UNSUPPORTED, "d_model must be a multiple of 32, <= 512, divisible by heads");
  const int dh = c.d_model / c.n_heads;
  NMT_REQUIRE(dh == 16 || dh == 32 || dh == 64, NMT_E_UNSUPPORTED, "head dim must be 16, 32 or 64");
  NMT_REQUIRE(c.d_ffn % 32 == 0, NMT_E_UNSUPPORTED, "d_ffn must be a multiple of 32");
  NMT_REQUIRE(c.max_rel_pos >= 1 && 2 * c.max_rel_pos + 1 <= 32, NMT_E_UNSUPPORTED,
              "max_rel_pos must be in [1, 15]");
  NMT_REQUIRE(c.max_src_len >= 1 && c.max_src_len <= 120 && c.max_src_len <= c.max_pos &&
                  c.max_tgt_len >= 1 && c.max_tgt_len <= c.max_pos,
              NMT_E_FORMAT, "NTSD: bad max lengths (max_src_len <= 120)");
}

// ------------------------------------------------------------------ arena
void init_arena(nmt_model* m) {
  const nmt_config& c = m->cfg;
  const nmt_limits& L = m->lim;
  const size_t tb = m->tb, d = c.d_model, F = c.d_ffn, Ld = c.dec_layers;
  const size_t N = L.max_tokens, Bm = L.max_sents, Tm = L.max_tgt_len;
  const size_t R = Bm * std::max(1, L.beam);
  Arena& a = m->ar;
  // split-K workspace: max over the decode GEMM shapes of m_tiles * n_tiles * splits * 128*64
  size_t ws_floats = 0;
  {
    const int shapes[5][2] = {{3 * (int)d, (int)d}, {(int)d, (int)d}, {(int)F, (int)d},
                              {(int)d, (int)F}, {(int)d, (int)d}};
    const size_t mt = (R + 127) / 128;
    for (auto& sh : shapes) {
      const size_t nt = (sh[0] + 63) / 64, sp = decode_splits(sh[0], sh[1]);
      if (sp > 1) ws_floats = std::max(ws_floats, mt * nt * sp * 128 * 64);
    }
  }
  const size_t cnt_ints = ((R + 127) / 128) * ((std::max(3 * d, F) + 63) / 64);
  std::vector<std::pair<void**, size_t>> items = {
      {(void**)&m->src, N * 4}, {(void**)&m->src_len, Bm * 4}, {(void**)&m->tgt_cap, Bm * 4},
      {&m->x, N * d * tb}, {&m->u, N * d * tb}, {&m->qkv, N * 3 * d * tb}, {&m->o, N * d * tb},
      {&m->h, N * F * tb}, {&m->enc_out, N * d * tb},
      {&m->hist, c.use_dlcl ? (size_t)(c.enc_layers + 1) * N * d * tb : 256},
      {&m->ckv, N * Ld * 2 * d * tb},
      {&m->g, R * d * tb}, {&m->du, R * d * tb}, {&m->dqkv, R * 3 * d * tb},
      {&m->dout, R * d * tb}, {&m->dq, R * d * tb}, {&m->dh, R * F * tb},
      {&m->kc, Ld * R * Tm * d * tb}, {&m->vc, Ld * R * Tm * d * tb},
      {(void**)&m->keys, R * 8}, {(void**)&m->row_slot, R * 4}, {(void**)&m->prev_tok, R * 4},
      {(void**)&m->done, R}, {(void**)&m->out_tok, Bm * Tm * 4}, {(void**)&m->gen_len, Bm * 4},
      {(void**)&m->st, sizeof(DevState)}, {(void**)&m->bad, 4}, {(void**)&m->boff, Bm * 8},
      {(void**)&m->blen, Bm * 4}, {(void**)&m->sent_ids, Bm * 4},
      {(void**)&m->gemm_ws, std::max<size_t>(ws_floats * 4, 256)},
      {(void**)&m->gemm_cnt, std::max<size_t>(cnt_ints * 4, 256)},
      // beam search: only sized when the limits ask for beam > 1
      {(void**)&m->bscore, L.beam > 1 ? R * 4 : 256},
      {(void**)&m->anc, L.beam > 1 ? R * Tm * 4 : 256},
      {(void**)&m->htok, L.beam > 1 ? R * Tm * 4 : 256},
      {(void**)&m->best_score, L.beam > 1 ? Bm * 4 : 256},
      {(void**)&m->nb_score, L.beam > 1 ? Bm * L.beam * 4 : 256},
      {(void**)&m->nb_len, L.beam > 1 ? Bm * L.beam * 4 : 256},
      {(void**)&m->nb_tok, L.beam > 1 ? Bm * L.beam * Tm * 4 : 256},
      {(void**)&m->nb_cnt, L.beam > 1 ? Bm * 4 : 256},
      {(void**)&m->blogits, L.beam > 1 ? R * (size_t)c.vocab_size * 4 : 256},
      {(void**)&m->lnst, R * (d / 32) * 8},
      {(void**)&m->dlcl_p, dlcl_blocks(c, (int)d) > 1 ? (dlcl_blocks(c, (int)d) - 1) * N * d * 4 : 256},
      {(void**)&m->cand_v, L.beam > 1 ? R * 8 * 4 : 256},
      {(void**)&m->cand_i, L.beam > 1 ? R * 8 * 4 : 256},
      {(void**)&m->fused_ctr, fused_counter_ints() * 4},
      {(void**)&m->bpart, L.beam > 1 && m->prec == NMT_FP16
                              ? R * (size_t)((c.vocab_size + 127) / 128) * 18 * 4 : 256},
  };
  std::vector<size_t> offs;
  for (auto& it : items) offs.push_back(a.take(it.second));
  cudaError_t e = cudaMalloc(&a.base, a.used);
  NMT_REQUIRE(e == cudaSuccess, NMT_E_RESOURCE,
              std::string("arena cudaMalloc failed: ") + cudaGetErrorString(e));
  a.cap = a.used;
  m->sys_allocs += 1;
  for (size_t i = 0; i < items.size(); ++i) *items[i].first = a.base + offs[i];
  NMT_CUDA(cudaMemset(a.base, 0, a.used));
  for (auto& ev : m->ev_t) NMT_CUDA(cudaEventCreate(&ev));
  // fused beam epilogue (logits never written): opt-in, NMT_BEAM_EPI=1 — measured slower
  // than the logits + two-pass row top-K path on B200
  m->beam_epi = L.beam > 1 && m->prec == NMT_FP16 && getenv("NMT_BEAM_EPI") != nullptr;
  // pinned host staging (each region rounded to 64 B)
  size_t pb = N * 4 + Bm * 4 * 2 + Bm * 8 + Bm * 4 * 2 + Bm * Tm * 4 + Bm * 4 + 64 + 64 + 16 * 64;
  NMT_CUDA(cudaMallocHost(&m->pinned, pb));
  m->sys_allocs += 1;
  char* p = (char*)m->pinned;
  auto take = [&](size_t b) { char* r = p; p += (b + 63) & ~size_t(63); return r; };
  m->hp.boff = (long long*)take(Bm * 8);
  m->hp.src = (int*)take(N * 4);
  m->hp.len = (int*)take(Bm * 4);
  m->hp.cap = (int*)take(Bm * 4);
  m->hp.blen = (int*)take(Bm * 4);
  m->hp.sent = (int*)take(Bm * 4);
  m->hp.out_tok = (int*)take(Bm * Tm * 4);
  m->hp.gen_len = (int*)take(Bm * 4);
  m->hp.st = (DevState*)take(sizeof(DevState));
  m->hp.bad = (int*)take(4);
}

// LN folding for the FP16 decode step: the decoder LayerNorms that
// feed a projection GEMM (LN_self of layers >= 1, LN_cross, LN_ffn) are folded into that
// GEMM's weights, bias and epilogue; the final LN before the tied vocab projection stays a
// kernel (see decode_step_impl).
void fold_weights(nmt_model* m) {
  const nmt_config& c = m->cfg;
  const size_t d = c.d_model, F = c.d_ffn, Ld = c.dec_layers;
  const size_t rows = Ld * (3 * d + d + F);
  const size_t wbytes = rows * d * 2, cbytes = rows * 4, bbytes = rows * 2;
  cudaError_t e = cudaMalloc(&m->foldbuf, wbytes + cbytes + bbytes + 1024);
  NMT_REQUIRE(e == cudaSuccess, NMT_E_RESOURCE,
              std::string("fold cudaMalloc failed: ") + cudaGetErrorString(e));
  m->sys_allocs += 1;
  char* wp = (char*)m->foldbuf;
  float* cp = (float*)(wp + wbytes);
  char* bp = (char*)(cp + rows) + 256;
  size_t r0 = 0;
  auto fold = [&](const void* W, const void* g, const void* beta, const void* bias, size_t N) {
    FoldW f;
    f.w = wp + r0 * d * 2;
    f.c = cp + r0;
    f.b = bp + r0 * 2;
    fold_ln(W, g, beta, bias, (int)N, (int)d, (void*)f.w, (float*)f.c, (void*)f.b, 0);
    r0 += N;
    return f;
  };
  for (size_t l = 0; l < Ld; ++l) {
    const DecW& w = m->dec[l];
    DecFold df;
    df.qkv = fold(w.qkv_w, w.self_g, w.self_b, w.qkv_b, 3 * d);
    df.cq = fold(w.cq_w, w.cross_g, w.cross_b, w.cq_b, d);
    df.w1 = fold(w.w1, w.ffn_g, w.ffn_b, w.b1, F);
    m->fold.push_back(df);
  }
}

void bind_weights(nmt_model* m) {
  const nmt_config& c = m->cfg;
  auto W = [&](const std::string& n) -> const void* {
    auto it = m->W.find(n);
    NMT_REQUIRE(it != m->W.end(), NMT_E_INTEGRITY, "missing tensor " + n);
    return it->second;
  };
  m->emb = W("emb");
  m->enc_fg = W("enc.final_ln.g");
  m->enc_fb = W("enc.final_ln.b");
  m->dec_fg = W("dec.final_ln.g");
  m->dec_fb = W("dec.final_ln.b");
  if (c.use_dlcl) {
    m->dl0_g = W("enc.dlcl.ln.0.g");
    m->dl0_b = W("enc.dlcl.ln.0.b");
  }
  for (int l = 0; l < c.enc_layers; ++l) {
    const std::string p = "enc." + std::to_string(l) + ".";
    EncW e{};
    e.attn_g = W(p + "attn_ln.g"); e.attn_b = W(p + "attn_ln.b");
    e.qkv_w = W(p + "qkv.w"); e.qkv_b = W(p + "qkv.b");
    e.out_w = W(p + "out.w"); e.out_b = W(p + "out.b");
    e.relk = c.use_rpr ? W(p + "rel_k") : nullptr;
    e.relv = c.use_rpr ? W(p + "rel_v") : nullptr;
    e.ffn_g = W(p + "ffn_ln.g"); e.ffn_b = W(p + "ffn_ln.b");
    e.w1 = W(p + "ffn1.w"); e.b1 = W(p + "ffn1.b"); e.w2 = W(p + "ffn2.w"); e.b2 = W(p + "ffn2.b");
    if (c.use_dlcl) {
      e.dl_g = W("enc.dlcl.ln." + std::to_string(l + 1) + ".g");
      e.dl_b = W("enc.dlcl.ln." + std::to_string(l + 1) + ".b");
    }
    m->enc.push_back(e);
  }
  for (int l = 0; l < c.dec_layers; ++l) {
    const std::string p = "dec." + std::to_string(l) + ".";
    DecW e{};
    e.self_g = W(p + "self_ln.g"); e.self_b = W(p + "self_ln.b");
    e.qkv_w = W(p + "self_qkv.w"); e.qkv_b = W(p + "self_qkv.b");
    e.so_w = W(p + "self_out.w"); e.so_b = W(p + "self_out.b");
    e.relk = c.use_rpr ? W(p + "rel_k") : nullptr;
    e.relv = c.use_rpr ? W(p + "rel_v") : nullptr;
    e.cross_g = W(p + "cross_ln.g"); e.cross_b = W(p + "cross_ln.b");
    e.cq_w = W(p + "cross_q.w"); e.cq_b = W(p + "cross_q.b");
    e.co_w = W(p + "cross_out.w"); e.co_b = W(p + "cross_out.b");
    e.ffn_g = W(p + "ffn_ln.g"); e.ffn_b = W(p + "ffn_ln.b");
    e.w1 = W(p + "ffn1.w"); e.b1 = W(p + "ffn1.b"); e.w2 = W(p + "ffn2.w"); e.b2 = W(p + "ffn2.b");
    m->dec.push_back(e);
  }
}

// NTSD parsing (host only; shared by nmt_load_weights and nmt_ntsd_inspect).  Every size
// check is written so that no sum can wrap (a crafted blob must fail with NMT_E_INTEGRITY).
struct Parsed {
  nmt_config cfg{};
  int version = 0;
  std::unordered_map<std::string, TensorRec> recs;
};

void set_defaults(nmt_config& c) {   // fields the SPEC's v1 block does not carry
  c.dlcl_ln = 1;
  c.max_src_len = 120;
  c.max_tgt_len = 200;
  c.max_pos = 1024;
  c.pad_id = 0; c.unk_id = 1; c.bos_id = 2; c.eos_id = 3;
  c.ln_eps = 1e-5f;
}

Parsed parse_blob(const void* blob, size_t nbytes) {
  NMT_REQUIRE(blob, NMT_E_ARG, "null blob");
  Parsed P;
  const uint8_t* p = (const uint8_t*)blob;
  const uint8_t* end = p + nbytes;
  NMT_REQUIRE(nbytes >= 8 && memcmp(p, "NTSD", 4) == 0, NMT_E_FORMAT, "NTSD: bad magic");
  p += 4;
  const uint32_t ver = rd<uint32_t>(p, end);
  NMT_REQUIRE(ver == 1 || ver == 2, NMT_E_FORMAT, "NTSD: unsupported version " + std::to_string(ver));
  P.version = (int)ver;
  nmt_config& cfg = P.cfg;
  if (ver == 1) {   // SPEC layout: 8 x u32 config, inline payloads
    uint32_t v[8];
    for (auto& x : v) x = rd<uint32_t>(p, end);
    NMT_REQUIRE((v[7] & ~3u) == 0, NMT_E_FORMAT, "NTSD v1: unknown flag bits");
    NMT_REQUIRE(v[7] & 2u, NMT_E_UNSUPPORTED, "NTSD v1: untied embeddings (shared_emb = 0) not built");
    for (int i = 0; i < 7; ++i)
      NMT_REQUIRE(v[i] <= (1u << 24), NMT_E_FORMAT, "NTSD v1: config field out of range");
    cfg.enc_layers = (int)v[0]; cfg.dec_layers = (int)v[1]; cfg.d_model = (int)v[2];
    cfg.n_heads = (int)v[3]; cfg.d_ffn = (int)v[4]; cfg.vocab_size = (int)v[5];
    cfg.use_rpr = v[6] > 0;
    cfg.max_rel_pos = v[6] > 0 ? (int)v[6] : 8;
    cfg.use_dlcl = v[7] & 1u;
    set_defaults(cfg);
  } else {
    const uint32_t cb = rd<uint32_t>(p, end);
    NMT_REQUIRE(cb == sizeof(nmt_config), NMT_E_FORMAT, "NTSD: config block size mismatch");
    NMT_REQUIRE((size_t)(end - p) >= cb, NMT_E_INTEGRITY, "NTSD: truncated config");
    memcpy(&cfg, p, cb);
    p += cb;
  }
  validate_config(cfg);
  const uint32_t nt = rd<uint32_t>(p, end);
  for (uint32_t i = 0; i < nt; ++i) {
    TensorRec r;
    const uint16_t nl = rd<uint16_t>(p, end);
    NMT_REQUIRE((size_t)(end - p) >= nl, NMT_E_INTEGRITY, "NTSD: truncated name");
    r.name.assign((const char*)p, nl);
    p += nl;
    uint8_t nd;
    if (ver == 1) {
      nd = rd<uint8_t>(p, end);
      NMT_REQUIRE(nd <= 8, NMT_E_INTEGRITY, "NTSD: rank > 8 for " + r.name);
      for (int k = 0; k < nd; ++k) r.dims.push_back(rd<uint32_t>(p, end));
      r.dtype = rd<uint8_t>(p, end);
    } else {
      r.dtype = rd<uint8_t>(p, end);
      nd = rd<uint8_t>(p, end);
      NMT_REQUIRE(nd <= 8, NMT_E_INTEGRITY, "NTSD: rank > 8 for " + r.name);
      for (int k = 0; k < nd; ++k) r.dims.push_back(rd<uint32_t>(p, end));
    }
    NMT_REQUIRE(r.dtype == 0 || r.dtype == 1, NMT_E_FORMAT, "NTSD: bad dtype for " + r.name);
    // element count without overflow: every dim < 2^32, product capped at 2^40
    uint64_t cnt = 1;
    for (auto dd : r.dims) {
      NMT_REQUIRE(dd == 0 || cnt <= (uint64_t(1) << 40) / dd, NMT_E_INTEGRITY,
                  "NTSD: tensor too large: " + r.name);
      cnt *= dd;
    }
    const uint64_t es = r.dtype == 1 ? 2 : 4;
    if (ver == 1) {
      const uint64_t nb = cnt * es;
      NMT_REQUIRE(nb <= (uint64_t)(end - p), NMT_E_INTEGRITY, "NTSD: truncated tensor " + r.name);
      r.data = p;
      r.nbytes = nb;
      p += nb;
    } else {
      const uint64_t off = rd<uint64_t>(p, end), nb = rd<uint64_t>(p, end);
      // off + nb <= nbytes, written so that it cannot wrap
      NMT_REQUIRE(nb <= nbytes && off <= nbytes - nb, NMT_E_INTEGRITY,
                  "NTSD: tensor " + r.name + " outside the blob");
      NMT_REQUIRE(nb == cnt * es, NMT_E_INTEGRITY, "NTSD: byte size mismatch for " + r.name);
      r.data = (const uint8_t*)blob + off;
      r.nbytes = nb;
    }
    NMT_REQUIRE(P.recs.count(r.name) == 0, NMT_E_INTEGRITY, "NTSD: duplicate tensor " + r.name);
    P.recs.emplace(r.name, r);
  }
  auto can = canonical(cfg);
  NMT_REQUIRE(P.recs.size() == can.size(), NMT_E_INTEGRITY,
              "NTSD: expected " + std::to_string(can.size()) + " tensors, got " +
                  std::to_string(P.recs.size()));
  for (auto& kv : can) {
    auto it = P.recs.find(kv.first);
    NMT_REQUIRE(it != P.recs.end(), NMT_E_INTEGRITY, "NTSD: missing tensor " + kv.first);
    NMT_REQUIRE(it->second.dims == kv.second, NMT_E_INTEGRITY, "NTSD: shape mismatch for " + kv.first);
  }
  return P;
}

nmt_model* clone_worker(nmt_model* m);

nmt_model* load(const void* blob, size_t nbytes, int device, nmt_precision prec,
                const nmt_limits* lim) {
  NMT_REQUIRE(blob && lim, NMT_E_ARG, "null blob or limits");
  NMT_REQUIRE(prec == NMT_FP16 || prec == NMT_FP32, NMT_E_ARG, "bad precision");
  Parsed P = parse_blob(blob, nbytes);
  const nmt_config cfg = P.cfg;
  auto& recs = P.recs;
  NMT_REQUIRE(lim->max_tokens >= 1 && lim->max_sents >= 1 && lim->max_tgt_len >= 1 &&
                  lim->max_tgt_len <= cfg.max_tgt_len && lim->beam >= 1 &&
                  lim->n_workspaces >= 0 && lim->n_workspaces <= 16,
              NMT_E_ARG, "bad limits");
  NMT_REQUIRE(lim->beam <= 4, NMT_E_UNSUPPORTED, "beam > 4 is not built");
  NMT_REQUIRE((size_t)lim->max_sents * lim->beam <= 16384, NMT_E_ARG, "max_sents*beam > 16384");

  std::unique_ptr<nmt_model> m(new nmt_model());
  m->cfg = cfg;
  m->prec = prec;
  m->lim = *lim;
  m->lim.n_workspaces = std::max(1, lim->n_workspaces);
  m->device = device;
  m->tb = prec == NMT_FP16 ? 2 : 4;
  // fused decode step (decode_fused.cu): opt-in (NMT_FUSE_ROWS = live-row threshold of the
  // single launch) — measured slower than the graph-replayed unfused step at every live-row
  // count on B200 (profiles/r2g_*), so the product default is unfused
  m->fuse_rows = getenv("NMT_NO_FUSE") ? -1
                 : getenv("NMT_FUSE_ROWS") ? atoi(getenv("NMT_FUSE_ROWS")) : -1;
  if (getenv("NMT_FUSED_TRACE")) {   // debug timeline of the fused decode step (not the product path)
    NMT_CUDA(cudaMalloc(&m->fused_trace, (4 * 65536 + 1024) * 8));
    NMT_CUDA(cudaMemset(m->fused_trace, 0, (4 * 65536 + 1024) * 8));
    m->sys_allocs += 1;
  }
  NMT_CUDA(cudaSetDevice(device));
  auto can = canonical(cfg);
  size_t total = 0;
  std::vector<size_t> offs;
  for (auto& kv : can) {
    auto it = recs.find(kv.first);
    NMT_REQUIRE(it != recs.end(), NMT_E_INTEGRITY, "NTSD: missing tensor " + kv.first);
    size_t cnt = 1;
    for (auto dd : kv.second) cnt *= dd;
    offs.push_back(total);
    total += (cnt * m->tb + 255) & ~size_t(255);
  }
  const int d = cfg.d_model, Ld = cfg.dec_layers;
  const size_t ckv_w_off = total;
  total += ((size_t)Ld * 2 * d * d * m->tb + 255) & ~size_t(255);
  const size_t ckv_b_off = total;
  total += ((size_t)Ld * 2 * d * m->tb + 255) & ~size_t(255);
  const int L1 = cfg.enc_layers + 1;
  const size_t dlcl_off = total;
  total += ((size_t)L1 * (L1 + 1) / 2 * 4 + 255) & ~size_t(255);
  const size_t pe_off = total;
  total += (size_t)cfg.max_pos * d * 4;
  std::vector<uint8_t> host(total, 0);
  auto get_f = [](const TensorRec& r, size_t i) -> float {
    if (r.dtype == 1) {
      uint16_t hb;
      memcpy(&hb, r.data + 2 * i, 2);
      return half_bits_to_float(hb);
    }
    float f;
    memcpy(&f, r.data + 4 * i, 4);
    return f;
  };
  auto put = [&](size_t dst, float f) {
    if (m->tb == 2) {
      uint16_t hb = float_to_half_bits(f);
      memcpy(&host[dst], &hb, 2);
    } else {
      memcpy(&host[dst], &f, 4);
    }
  };
  for (size_t t = 0; t < can.size(); ++t) {
    const TensorRec& r = recs.at(can[t].first);
    const size_t cnt = r.nbytes / (r.dtype == 1 ? 2 : 4);
    if (r.dtype == 1 && m->tb == 2) memcpy(&host[offs[t]], r.data, r.nbytes);  // FP16 -> FP16
    else for (size_t i = 0; i < cnt; ++i) put(offs[t] + i * m->tb, get_f(r, i));
  }
  for (int l = 0; l < Ld; ++l) {
    const TensorRec& w = recs.at("dec." + std::to_string(l) + ".cross_kv.w");
    const TensorRec& bb = recs.at("dec." + std::to_string(l) + ".cross_kv.b");
    size_t wc = (size_t)2 * d * d;
    for (size_t i = 0; i < wc; ++i) put(ckv_w_off + ((size_t)l * wc + i) * m->tb, get_f(w, i));
    for (int i = 0; i < 2 * d; ++i) put(ckv_b_off + ((size_t)l * 2 * d + i) * m->tb, get_f(bb, i));
  }
  if (cfg.use_dlcl) {
    const TensorRec& w = recs.at("enc.dlcl.w");
    for (int i = 0; i < L1 * (L1 + 1) / 2; ++i) {
      float f = get_f(w, i);
      memcpy(&host[dlcl_off + 4 * i], &f, 4);
    }
  }
  {  // sinusoid table in double precision, stored FP32 (reading R8)
    const int half = d / 2;
    for (int pos = 0; pos < cfg.max_pos; ++pos)
      for (int i = 0; i < half; ++i) {
        double w = std::exp(-std::log(10000.0) * i / (half - 1));
        float sv = (float)std::sin(pos * w), cv = (float)std::cos(pos * w);
        memcpy(&host[pe_off + ((size_t)pos * d + i) * 4], &sv, 4);
        memcpy(&host[pe_off + ((size_t)pos * d + half + i) * 4], &cv, 4);
      }
  }
  cudaError_t e = cudaMalloc(&m->wbuf, total);
  NMT_REQUIRE(e == cudaSuccess, NMT_E_RESOURCE,
              std::string("weights cudaMalloc failed: ") + cudaGetErrorString(e));
  m->sys_allocs += 1;
  NMT_CUDA(cudaMemcpy(m->wbuf, host.data(), total, cudaMemcpyHostToDevice));
  char* base = (char*)m->wbuf;
  for (size_t t = 0; t < can.size(); ++t) m->W[can[t].first] = base + offs[t];
  m->ckv_w = base + ckv_w_off;
  m->ckv_b = base + ckv_b_off;
  m->dlcl_w = (float*)(base + dlcl_off);
  m->pe = (float*)(base + pe_off);
  bind_weights(m.get());
  if (prec == NMT_FP16) fold_weights(m.get());
  init_arena(m.get());
  // the remaining worker arenas of the memory pool: translate never allocates
  for (int w = 1; w < m->lim.n_workspaces; ++w) m->workers.push_back(clone_worker(m.get()));
  NMT_CUDA(cudaDeviceSynchronize());
  return m.release();
}

// ------------------------------------------------------------------ batches
void encode_common(nmt_model* m, int B, int S, const int* h_len, const int* h_cap,
                   cudaStream_t s, int K = 1) {
  nmt_batch& b = m->batch;
  NMT_REQUIRE(K >= 1 && K <= m->lim.beam && K <= 4, NMT_E_ARG,
              "beam " + std::to_string(K) + " outside [1, min(4, limits.beam)]");
  const int Tm = m->lim.max_tgt_len;
  int mc = 0;
  for (int i = 0; i < B; ++i) {
    m->hp.len[i] = h_len[i];
    int cp = h_cap ? std::min(h_cap[i], Tm) : Tm;
    cp = std::max(cp, 1);
    m->hp.cap[i] = cp;
    mc = std::max(mc, cp);
  }
  NMT_CUDA(cudaMemcpyAsync(m->src_len, m->hp.len, B * 4, cudaMemcpyHostToDevice, s));
  NMT_CUDA(cudaMemcpyAsync(m->tgt_cap, m->hp.cap, B * 4, cudaMemcpyHostToDevice, s));
  encode_any(m, B, S, s);
  if (K == 1)
    PROF(P_BOOK, 0, 0,
         batch_init(m->row_slot, m->prev_tok, m->done, m->gen_len, m->st, B, S, m->cfg.bos_id, s));
  else
    PROF(P_BOOK, 0, 0,
         beam_init(m->row_slot, m->prev_tok, m->done, m->bscore, m->htok, Tm, m->best_score,
                   m->gen_len, m->st, B, K, S, m->cfg.bos_id, s, m->nb_cnt));
  b.m = m; b.B = B; b.S = S; b.step = 0; b.rows_upper = B * K; b.max_cap = mc; b.valid = true;
  b.K = K;
  b.NB = 1;
  b.pending_step_done = false;
}

void check_batch_shape(nmt_model* m, int B, int S) {
  NMT_REQUIRE(B >= 1 && S >= 1, NMT_E_ARG, "n_sent and s_max must be >= 1");
  NMT_REQUIRE(B <= m->lim.max_sents, NMT_E_SHAPE,
              "n_sent " + std::to_string(B) + " > max_sents " + std::to_string(m->lim.max_sents));
  NMT_REQUIRE((long long)B * S <= m->lim.max_tokens, NMT_E_SHAPE,
              "n_sent*s_max " + std::to_string((long long)B * S) + " > max_tokens " +
                  std::to_string(m->lim.max_tokens));
  NMT_REQUIRE(S <= m->cfg.max_src_len, NMT_E_INPUT,
              "s_max " + std::to_string(S) + " > max_src_len " + std::to_string(m->cfg.max_src_len));
}

void poll_state(nmt_model* m, cudaStream_t s) {
  NMT_CUDA(cudaMemcpyAsync(m->hp.st, m->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  NMT_CUDA(cudaStreamSynchronize(s));
  if (!m->prof.pending.empty()) prof_flush(m);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("NMT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One greedy step + pruning decision for `rows` live rows.  After one eager step the
// pair is captured once per (rows bucket, cadence, ratio) into a CUDA graph and
// replayed: every kernel reads t, the live count and S from device memory, so a graph
// serves every step of every batch (no per-step host round trip).
void step_and_prune(nmt_model* m, nmt_batch& b, int rows, int every, float ratio,
                    cudaStream_t s) {
  const int Rmax = m->lim.max_sents * std::max(1, m->lim.beam);
  const int bucket = std::min(Rmax, (rows + 31) & ~31);
  auto eager = [&] {
    if (b.K == 1) {  // greedy: argmax epilogue, then finish + prune in one CTA
      decode_step_any(m, &b, nullptr, nullptr, s, /*finish=*/false);
      PROF(P_BOOK, 0, 0,
           finish_prune(m->keys, m->prev_tok, m->done, m->row_slot, m->tgt_cap, m->out_tok,
                        m->lim.max_tgt_len, m->gen_len, m->st, m->cfg.eos_id, every, ratio,
                        b.rows_upper, s));
    } else {         // beam: logits -> row top-2K -> per-sentence select, then prune
      decode_step_any(m, &b, nullptr, nullptr, s, /*finish=*/true);
      PROF(P_BOOK, 0, 0,
           prune_compact(m->st, m->row_slot, m->prev_tok, m->done, every, ratio, nullptr,
                         b.rows_upper, s, m->bscore));
    }
  };
  unsigned rb;
  memcpy(&rb, &ratio, 4);
  auto key = std::make_tuple(bucket, every, rb, b.K * 8 + b.NB);
  if (s == nullptr || !m->eager_keys.count(key)) {
    b.rows_upper = rows;
    eager();  // first use of a configuration runs eagerly (sets kernel attributes)
    m->eager_keys.insert(key);
    return;
  }
  int nodes = 0;   // kernel nodes of the captured graph
  auto capture = [&](std::vector<nmt_model::ProfRec>* recs, nmt_model::ProfRec* bracket = nullptr) {
    b.rows_upper = bucket;
    cudaGraph_t g;
    NMT_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    g_pdl = pdl_enabled();  // programmatic edges between the step's kernels
    g_prof_capture = recs;
    try {
      if (bracket) NMT_CUDA(cudaEventRecordWithFlags(bracket->a, s, cudaEventRecordExternal));
      eager();
      if (bracket) NMT_CUDA(cudaEventRecordWithFlags(bracket->b, s, cudaEventRecordExternal));
    } catch (...) {
      g_pdl = false;
      g_prof_capture = nullptr;
      cudaStreamEndCapture(s, &g);
      throw;
    }
    g_pdl = false;
    g_prof_capture = nullptr;
    NMT_CUDA(cudaStreamEndCapture(s, &g));
    size_t nn = 0;
    NMT_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> ns(nn);
    if (nn) NMT_CUDA(cudaGraphGetNodes(g, ns.data(), &nn));
    nodes = 0;
    for (auto n : ns) {
      cudaGraphNodeType ty;
      NMT_CUDA(cudaGraphNodeGetType(n, &ty));
      nodes += ty == cudaGraphNodeTypeKernel;
    }
    cudaGraphExec_t ex;
    NMT_CUDA(cudaGraphInstantiate(&ex, g, 0));
    NMT_CUDA(cudaGraphDestroy(g));
    return ex;
  };
  if (m->prof.on && m->prof.steps_only) {
    // step-timed replay: the plain step graph between two event nodes (kernel-to-kernel
    // transitions as in production), synchronised so t and the live rows are exact
    auto it = m->sgraphs.find(key);
    if (it == m->sgraphs.end()) {
      nmt_model::ProfRec br{};
      NMT_CUDA(cudaEventCreate(&br.a));
      NMT_CUDA(cudaEventCreate(&br.b));
      cudaGraphExec_t ex = capture(nullptr, &br);
      br.cls = nodes;
      it = m->sgraphs.emplace(key, std::make_pair(ex, br)).first;
    }
    poll_state(m, s);
    const int live = m->hp.st->n_live, tt = m->hp.st->t;
    NMT_CUDA(cudaGraphLaunch(it->second.first, s));
    NMT_CUDA(cudaStreamSynchronize(s));
    float sm = 0.f;
    NMT_CUDA(cudaEventElapsedTime(&sm, it->second.second.a, it->second.second.b));
    if (m->prof.steps.size() < (1u << 22)) m->prof.steps.push_back({tt, live, sm});
    g_launches += it->second.second.cls;
    return;
  }
  if (m->prof.on) {
    // profiled replay: the same graph with an external event pair around every kernel,
    // read back after each step (timings of the kernels as they run in the graph)
    auto it = m->pgraphs.find(key);
    if (it == m->pgraphs.end()) {
      std::vector<nmt_model::ProfRec> recs;
      cudaGraphExec_t ex = capture(&recs);
      it = m->pgraphs.emplace(key, std::make_pair(ex, std::move(recs))).first;
    }
    poll_state(m, s);   // live rows and t entering this step (profiled steps synchronise)
    const int live = m->hp.st->n_live, tt = m->hp.st->t;
    NMT_CUDA(cudaGraphLaunch(it->second.first, s));
    NMT_CUDA(cudaStreamSynchronize(s));
    auto& P = m->prof;
    if (!it->second.second.empty() && P.steps.size() < (1u << 22)) {
      float sm = 0.f;
      NMT_CUDA(cudaEventElapsedTime(&sm, it->second.second.front().a, it->second.second.back().b));
      P.steps.push_back({tt, live, sm});
    }
    for (auto& r : it->second.second) {
      float ms = 0.f;
      NMT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      P.ms[r.cls] += ms;
      P.flops[r.cls] += r.flops;
      P.bytes[r.cls] += r.bytes;
      P.n[r.cls] += 1;
    }
    g_launches += it->second.second.size();
    return;
  }
  auto it = m->graphs.find(key);
  if (it == m->graphs.end()) {
    cudaGraphExec_t ex = capture(nullptr);
    it = m->graphs.emplace(key, std::make_pair(ex, nodes)).first;
  }
  NMT_CUDA(cudaGraphLaunch(it->second.first, s));
  g_launches += it->second.second;   // the replay launches the graph's kernels
}

// ------------------------------------------------------------------ translate core
struct Plan {
  std::vector<int> order;
  std::vector<int> bstart;  // batch boundaries into order
};

// Dynamic batching over length-sorted input, reading R17:
// stable sort by (-len, index); b = min(max_sents, floor(max_tokens / len_first), rest).
// len = the (possibly truncated) source lengths.
Plan plan_batches(const int* len, int64_t n, int max_tokens, int max_sents) {
  Plan p;
  p.order.resize(n);
  std::iota(p.order.begin(), p.order.end(), 0);
  std::stable_sort(p.order.begin(), p.order.end(), [&](int a, int b) { return len[a] > len[b]; });
  int64_t i = 0;
  while (i < n) {
    p.bstart.push_back((int)i);
    int first = len[p.order[i]];
    int64_t b = std::min<int64_t>({(int64_t)max_sents, std::max<int64_t>(1, max_tokens / first),
                                   n - i});
    i += b;
  }
  p.bstart.push_back((int)n);
  return p;
}

nmt_model* clone_worker(nmt_model* m) {
  std::unique_ptr<nmt_model> c(new nmt_model());
  c->cfg = m->cfg; c->prec = m->prec; c->lim = m->lim; c->device = m->device; c->tb = m->tb;
  c->wbuf = m->wbuf; c->owns_weights = false;
  c->W = m->W; c->enc = m->enc; c->dec = m->dec;
  c->emb = m->emb; c->dl0_g = m->dl0_g; c->dl0_b = m->dl0_b; c->enc_fg = m->enc_fg;
  c->enc_fb = m->enc_fb; c->dec_fg = m->dec_fg; c->dec_fb = m->dec_fb;
  c->ckv_w = m->ckv_w; c->ckv_b = m->ckv_b; c->dlcl_w = m->dlcl_w; c->pe = m->pe;
  c->foldbuf = m->foldbuf; c->fold = m->fold;
  c->fuse_rows = m->fuse_rows;
  init_arena(c.get());
  NMT_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
  return c.release();
}

// Separate decode stream of a worker (tuning: NMT_PRIO=1 high / 2 low priority for the
// decode phase; unset or 0 keeps everything on `ws`, measured best).
cudaStream_t decode_stream(nmt_model* m, cudaStream_t ws) {
  static const int mode = getenv("NMT_PRIO") ? atoi(getenv("NMT_PRIO")) : 0;
  if (mode != 1 && mode != 2) return ws;
  if (!m->dec_stream) {
    int least = 0, greatest = 0;
    NMT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    NMT_CUDA(cudaStreamCreateWithPriority(&m->dec_stream, cudaStreamNonBlocking,
                                          mode == 1 ? greatest : least));
    NMT_CUDA(cudaEventCreateWithFlags(&m->ev_enc, cudaEventDisableTiming));
    NMT_CUDA(cudaEventCreateWithFlags(&m->ev_dec, cudaEventDisableTiming));
  }
  return m->dec_stream;
}

// Source lengths seen by the path: sources longer than min(max_src_len, max_tokens) are cut
// to that length with EOS last (counted).  Empty sources are rejected.
std::vector<int> effective_lengths(const nmt_model* m, const int64_t* h_off, int64_t n,
                                   int max_tokens, int64_t* truncated) {
  const int cut = std::min(m->cfg.max_src_len, max_tokens);
  std::vector<int> len(n);
  int64_t tr = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t l = h_off[i + 1] - h_off[i];
    NMT_REQUIRE(l >= 1, NMT_E_INPUT, "empty source sentence " + std::to_string(i));
    if (l > cut) ++tr;
    len[i] = (int)std::min<int64_t>(l, cut);
  }
  if (truncated) *truncated = tr;
  return len;
}

// Whole-set driver.  Batches (length-sorted plan) are taken from a shared counter by
// `n_workers` workers, each a (model-or-clone, stream) pair on its own host thread; worker 0
// is the model itself on the caller's stream; the worker arenas were allocated at load.
// load_src(wm, stream, order, B, S, lens) stages the batch sources into wm->src (lens are the
// effective lengths: a source with lens < its length is truncated, EOS last); emit(wm,
// stream, order, B) consumes the results and returns the batch's generated-token count.
template <class LoadF, class EmitF>
void translate_core(nmt_model* m, const int64_t* h_off, int64_t n, const nmt_translate_opts* o,
                    LoadF load_src, EmitF emit, nmt_stats* st, cudaStream_t s) {
  const int max_tokens = o && o->max_tokens > 0 ? o->max_tokens : m->lim.max_tokens;
  const int max_sents = o && o->max_sents > 0 ? o->max_sents : m->lim.max_sents;
  const int every = o && o->prune_every > 0 ? o->prune_every : 1;
  const float ratio = o ? o->prune_ratio : 0.25f;
  const int sync_every = o && o->sync_every > 0 ? o->sync_every : 4;
  const int W = o && o->n_workers > 1 ? std::min(o->n_workers, 16) : 1;
  const int K = o && o->beam > 1 ? o->beam : 1;  // beam width; 1 = greedy
  const int NB = o && o->nbest > 1 ? o->nbest : 1;  // n-best lists
  NMT_REQUIRE(NB <= K, NMT_E_ARG, "nbest must be <= beam");
  NMT_REQUIRE(max_tokens <= m->lim.max_tokens && max_sents <= m->lim.max_sents, NMT_E_ARG,
              "translate opts exceed the model limits");
  NMT_REQUIRE(W <= 1 + (int)m->workers.size(), NMT_E_ARG,
              "n_workers " + std::to_string(W) + " > limits.n_workspaces " +
                  std::to_string(1 + m->workers.size()));
  int64_t truncated = 0;
  const std::vector<int> elen = effective_lengths(m, h_off, n, max_tokens, &truncated);
  Plan p = plan_batches(elen.data(), n, max_tokens, max_sents);
  const int nb = (int)p.bstart.size() - 1;
  auto t0 = std::chrono::steady_clock::now();
  unsigned long long l0 = g_launches;
  std::atomic<int> next{0};
  std::atomic<int64_t> steps{0}, prunes{0}, gen{0};
  std::atomic<bool> failed{false};
  std::mutex tmu;
  double ms_enc = 0.0, ms_dec = 0.0;

  auto run = [&](nmt_model* wm, cudaStream_t ws) {
    std::vector<int> lens, caps;
    for (;;) {
      const int bi = next++;
      if (bi >= nb || failed) break;
      const int lo = p.bstart[bi], B = p.bstart[bi + 1] - lo;
      const int S = elen[p.order[lo]];
      lens.resize(B);
      caps.resize(B);
      for (int j = 0; j < B; ++j) {
        int sid = p.order[lo + j];
        lens[j] = elen[sid];
        caps[j] = o && o->h_tgt_cap ? o->h_tgt_cap[sid] : wm->lim.max_tgt_len;
      }
      NMT_CUDA(cudaEventRecord(wm->ev_t[0], ws));
      load_src(wm, ws, &p.order[lo], B, S, lens.data());
      encode_common(wm, B, S, lens.data(), caps.data(), ws, K);
      NMT_CUDA(cudaEventRecord(wm->ev_t[1], ws));
      cudaStream_t ds = decode_stream(wm, ws);
      if (ds != ws) {   // decode after this batch's encoder, on the high-priority stream
        NMT_CUDA(cudaEventRecord(wm->ev_enc, ws));
        NMT_CUDA(cudaStreamWaitEvent(ds, wm->ev_enc, 0));
      }
      nmt_batch& b = wm->batch;
      b.NB = NB;
      int rows = B * K;
      int t = 0;
      // the live count is polled every `sync_every` steps (lagged upper bound for grids)
      for (; t < b.max_cap && rows > 0; ++t) {
        step_and_prune(wm, b, rows, every, ratio, ds);
        if ((t + 1) % sync_every == 0) {
          poll_state(wm, ds);
          rows = wm->hp.st->n_live;
        }
      }
      NMT_CUDA(cudaEventRecord(wm->ev_t[2], ds));
      poll_state(wm, ds);
      {
        float e1 = 0.f, e2 = 0.f;
        NMT_CUDA(cudaEventElapsedTime(&e1, wm->ev_t[0], wm->ev_t[1]));
        NMT_CUDA(cudaEventElapsedTime(&e2, wm->ev_t[1], wm->ev_t[2]));
        std::lock_guard<std::mutex> g(tmu);
        ms_enc += e1;
        ms_dec += e2;
      }
      steps += t;
      prunes += wm->hp.st->prunes;
      b.step = t;
      gen += emit(wm, ds, &p.order[lo], B);
      if (ds != ws) {   // the next batch's staging / encoder reuse the arena
        NMT_CUDA(cudaEventRecord(wm->ev_dec, ds));
        NMT_CUDA(cudaStreamWaitEvent(ws, wm->ev_dec, 0));
      }
      b.valid = false;
    }
  };

  if (W == 1) {
    run(m, s);
  } else {
    cudaEvent_t ev;
    NMT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    NMT_CUDA(cudaEventRecord(ev, s));  // workers start after prior work on the caller stream
    for (int w = 0; w < W - 1; ++w) NMT_CUDA(cudaStreamWaitEvent(m->workers[w]->own_stream, ev, 0));
    std::mutex emu;
    std::string emsg;
    nmt_status ecode = NMT_OK;
    auto guarded = [&](nmt_model* wm, cudaStream_t ws) {
      try {
        NMT_CUDA(cudaSetDevice(m->device));
        run(wm, ws);
      } catch (const NmtError& e) {
        std::lock_guard<std::mutex> g(emu);
        if (ecode == NMT_OK) { ecode = e.code; emsg = e.what(); }
        failed = true;
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> g(emu);
        if (ecode == NMT_OK) { ecode = NMT_E_CUDA; emsg = e.what(); }
        failed = true;
      }
    };
    std::vector<std::thread> th;
    for (int w = 0; w < W - 1; ++w)
      th.emplace_back(guarded, m->workers[w], m->workers[w]->own_stream);
    guarded(m, s);
    for (auto& t : th) t.join();
    for (int w = 0; w < W - 1; ++w) {
      NMT_CUDA(cudaEventRecord(ev, m->workers[w]->own_stream));
      NMT_CUDA(cudaStreamWaitEvent(s, ev, 0));  // caller stream orders after every worker
    }
    NMT_CUDA(cudaEventDestroy(ev));
    if (ecode != NMT_OK) throw NmtError(ecode, emsg);
  }
  NMT_CUDA(cudaStreamSynchronize(s));
  if (st) {
    st->sentences = n;
    st->src_tokens = h_off[n] - h_off[0];
    st->gen_tokens = gen;
    st->decode_steps = steps;
    st->prunes = prunes;
    st->batches = nb;
    st->launches = (int64_t)(g_launches - l0);
    st->truncated = truncated;
    st->arena_system_allocs = m->sys_allocs;
    for (auto* w : m->workers) st->arena_system_allocs += w->sys_allocs;
    st->ms_encode = ms_enc;
    st->ms_decode = ms_dec;
    st->ms_total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
}

}  // namespace

std::string& nmt::last_error() { return g_err; }

// ====================================================================== C ABI
extern "C" {

const char* nmt_last_error(void) { return g_err.c_str(); }

nmt_status nmt_load_weights(const void* h_ntsd, size_t nbytes, int device, nmt_precision prec,
                            const nmt_limits* lim, nmt_model** out) {
  return guard([&] {
    NMT_REQUIRE(out, NMT_E_ARG, "null out");
    *out = nullptr;
    *out = load(h_ntsd, nbytes, device, prec, lim);
  });
}

nmt_status nmt_get_config(const nmt_model* m, nmt_config* out) {
  return guard([&] {
    NMT_REQUIRE(m && out, NMT_E_ARG, "null argument");
    *out = m->cfg;
  });
}

void nmt_free_model(nmt_model* m) { delete m; }

nmt_status nmt_encode(nmt_model* m, const int32_t* d_src, const int32_t* h_src_len,
                      const int32_t* h_tgt_cap, int32_t n_sent, int32_t s_max, int32_t beam,
                      void* stream,
                      nmt_batch** out) {
  return guard([&] {
    NMT_REQUIRE(m && d_src && h_src_len && out, NMT_E_ARG, "null argument");
    check_batch_shape(m, n_sent, s_max);
    for (int i = 0; i < n_sent; ++i)
      NMT_REQUIRE(h_src_len[i] >= 1 && h_src_len[i] <= s_max, NMT_E_INPUT,
                  "src_len[" + std::to_string(i) + "] out of [1, s_max]");
    cudaStream_t s = (cudaStream_t)stream;
    NMT_CUDA(cudaMemcpyAsync(m->src, d_src, (size_t)n_sent * s_max * 4, cudaMemcpyDeviceToDevice, s));
    encode_common(m, n_sent, s_max, h_src_len, h_tgt_cap, s, beam < 1 ? 1 : beam);
    *out = &m->batch;
  });
}

nmt_status nmt_batch_encoder_output(const nmt_batch* b, float* d_dst, void* stream) {
  return guard([&] {
    NMT_REQUIRE(b && b->valid && d_dst, NMT_E_ARG, "null or invalid batch");
    nmt_model* m = b->m;
    size_t n = (size_t)b->B * b->S * m->cfg.d_model;
    if (m->prec == NMT_FP16)
      to_float<__half>((const __half*)m->enc_out, d_dst, n, (cudaStream_t)stream);
    else
      to_float<float>((const float*)m->enc_out, d_dst, n, (cudaStream_t)stream);
  });
}

nmt_status nmt_decode_step(nmt_model* m, nmt_batch* b, const int32_t* d_prev, int32_t step,
                           const nmt_step_out* out, void* stream) {
  return guard([&] {
    NMT_REQUIRE(m && b && b->valid && b->m == m, NMT_E_ARG, "null or invalid batch");
    NMT_REQUIRE(!b->pending_step_done, NMT_E_STATE, "decode_step called twice without prune");
    NMT_REQUIRE(step == b->step, NMT_E_STATE,
                "step " + std::to_string(step) + " != batch step " + std::to_string(b->step));
    NMT_REQUIRE(step < m->lim.max_tgt_len, NMT_E_STATE, "step beyond max_tgt_len");
    NMT_REQUIRE(!(d_prev && b->K > 1), NMT_E_UNSUPPORTED, "teacher forcing is greedy-only");
    decode_step_any(m, b, d_prev, out, (cudaStream_t)stream);
    b->pending_step_done = true;
  });
}

nmt_status nmt_prune_batch(nmt_model* m, nmt_batch* b, float ratio, const uint8_t* d_keep,
                           int32_t* d_new_to_old, int32_t* h_n_live, void* stream) {
  return guard([&] {
    NMT_REQUIRE(m && b && b->valid && b->m == m, NMT_E_ARG, "null or invalid batch");
    NMT_REQUIRE(b->pending_step_done, NMT_E_STATE, "prune must follow a decode step");
    NMT_REQUIRE(!(d_keep && b->K > 1), NMT_E_UNSUPPORTED, "d_keep is greedy-only");
    cudaStream_t s = (cudaStream_t)stream;
    if (d_keep)
      prune_keep(m->st, m->row_slot, m->prev_tok, m->done, d_keep, d_new_to_old, b->rows_upper, s);
    else
      prune_compact(m->st, m->row_slot, m->prev_tok, m->done, 1, ratio, d_new_to_old,
                    b->rows_upper, s, b->K > 1 ? m->bscore : nullptr);
    b->pending_step_done = false;
    b->step += 1;
    if (h_n_live) {
      poll_state(m, s);
      *h_n_live = m->hp.st->n_live;
      b->rows_upper = *h_n_live;
    }
  });
}

nmt_status nmt_batch_live(nmt_batch* b, int32_t* h_n_live, void* stream) {
  return guard([&] {
    NMT_REQUIRE(b && b->valid && h_n_live, NMT_E_ARG, "null or invalid batch");
    poll_state(b->m, (cudaStream_t)stream);
    *h_n_live = b->m->hp.st->n_live;
  });
}

nmt_status nmt_batch_results(nmt_batch* b, int32_t* h_ids, int32_t* h_len, void* stream) {
  return guard([&] {
    NMT_REQUIRE(b && b->valid && h_ids && h_len, NMT_E_ARG, "null or invalid batch");
    nmt_model* m = b->m;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t Tm = m->lim.max_tgt_len;
    NMT_CUDA(cudaMemcpyAsync(h_ids, m->out_tok, b->B * Tm * 4, cudaMemcpyDeviceToHost, s));
    NMT_CUDA(cudaMemcpyAsync(h_len, m->gen_len, b->B * 4, cudaMemcpyDeviceToHost, s));
    NMT_CUDA(cudaStreamSynchronize(s));
  });
}

void nmt_batch_free(nmt_batch* b) {
  if (b) {
    b->valid = false;
    b->pending_step_done = false;
  }
}

nmt_status nmt_ntsd_inspect(const void* h_ntsd, size_t nbytes, nmt_config* out,
                            int64_t* h_n_tensors, int32_t* h_version) {
  return guard([&] {
    NMT_REQUIRE(out, NMT_E_ARG, "null out");
    Parsed P = parse_blob(h_ntsd, nbytes);
    *out = P.cfg;
    if (h_n_tensors) *h_n_tensors = (int64_t)P.recs.size();
    if (h_version) *h_version = P.version;
  });
}

nmt_status nmt_translate(nmt_model* m, const int32_t* h_ids, const int64_t* h_off, int64_t n,
                         const nmt_translate_opts* opts, int32_t* h_out, int64_t out_cap,
                         int64_t* h_out_off, nmt_stats* stats, void* stream) {
  return guard([&] {
    NMT_REQUIRE(m && h_ids && h_off && h_out && h_out_off && n >= 0, NMT_E_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int V = m->cfg.vocab_size, eos = m->cfg.eos_id;
    const int Tm = m->lim.max_tgt_len;
    std::vector<std::vector<int>> outs(n);
    auto load_src = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B, int S,
                        const int* lens) {
      for (int j = 0; j < B; ++j) {
        const int32_t* src = h_ids + h_off[order[j]];
        const bool cut = h_off[order[j] + 1] - h_off[order[j]] > lens[j];   // truncated
        for (int p = 0; p < S; ++p) {
          int v = p < lens[j] ? src[p] : wm->cfg.pad_id;
          NMT_REQUIRE(v >= 0 && v < V, NMT_E_INPUT, "token id out of range");
          if (cut && p == lens[j] - 1) v = wm->cfg.eos_id;
          wm->hp.src[(size_t)j * S + p] = v;
        }
      }
      NMT_CUDA(cudaMemcpyAsync(wm->src, wm->hp.src, (size_t)B * S * 4, cudaMemcpyHostToDevice, ws));
    };
    auto emit = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B) -> int64_t {
      NMT_CUDA(cudaMemcpyAsync(wm->hp.out_tok, wm->out_tok, (size_t)B * Tm * 4,
                               cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaMemcpyAsync(wm->hp.gen_len, wm->gen_len, B * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaStreamSynchronize(ws));
      int64_t g = 0;
      for (int j = 0; j < B; ++j) {
        int gl = wm->hp.gen_len[j];
        g += gl;
        const int* t = wm->hp.out_tok + (size_t)j * Tm;
        int ol = (gl > 0 && t[gl - 1] == eos) ? gl - 1 : gl;
        outs[order[j]].assign(t, t + ol);
      }
      return g;
    };
    translate_core(m, h_off, n, opts, load_src, emit, stats, s);
    int64_t pos = 0;
    h_out_off[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
      NMT_REQUIRE(pos + (int64_t)outs[i].size() <= out_cap, NMT_E_SHAPE, "out_cap too small");
      std::copy(outs[i].begin(), outs[i].end(), h_out + pos);
      pos += outs[i].size();
      h_out_off[i + 1] = pos;
    }
    if (stats) stats->out_tokens = pos;
  });
}

nmt_status nmt_translate_nbest(nmt_model* m, const int32_t* h_ids, const int64_t* h_off,
                               int64_t n, const nmt_translate_opts* opts, int32_t* h_out,
                               int64_t out_cap, int64_t* h_out_off, float* h_score,
                               nmt_stats* stats, void* stream) {
  return guard([&] {
    NMT_REQUIRE(m && h_ids && h_off && h_out && h_out_off && opts && n >= 0, NMT_E_ARG,
                "null argument");
    const int K = opts->beam > 1 ? opts->beam : 1, NB = opts->nbest > 1 ? opts->nbest : 1;
    NMT_REQUIRE(NB >= 2 && NB <= K, NMT_E_ARG, "nmt_translate_nbest needs 2 <= nbest <= beam");
    cudaStream_t s = (cudaStream_t)stream;
    const int V = m->cfg.vocab_size, eos = m->cfg.eos_id;
    const int Tm = m->lim.max_tgt_len;
    std::vector<std::vector<int>> outs((size_t)n * NB);
    std::vector<float> scores((size_t)n * NB, -INFINITY);
    auto load_src = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B, int S,
                        const int* lens) {
      for (int j = 0; j < B; ++j) {
        const int32_t* src = h_ids + h_off[order[j]];
        const bool cut = h_off[order[j] + 1] - h_off[order[j]] > lens[j];   // truncated
        for (int p = 0; p < S; ++p) {
          int v = p < lens[j] ? src[p] : wm->cfg.pad_id;
          NMT_REQUIRE(v >= 0 && v < V, NMT_E_INPUT, "token id out of range");
          if (cut && p == lens[j] - 1) v = wm->cfg.eos_id;
          wm->hp.src[(size_t)j * S + p] = v;
        }
      }
      NMT_CUDA(cudaMemcpyAsync(wm->src, wm->hp.src, (size_t)B * S * 4, cudaMemcpyHostToDevice, ws));
    };
    auto emit = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B) -> int64_t {
      std::vector<int> tok((size_t)B * NB * Tm), len((size_t)B * NB), cnt(B), gl(B);
      std::vector<float> sc((size_t)B * NB);
      NMT_CUDA(cudaMemcpyAsync(tok.data(), wm->nb_tok, tok.size() * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaMemcpyAsync(len.data(), wm->nb_len, len.size() * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaMemcpyAsync(sc.data(), wm->nb_score, sc.size() * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaMemcpyAsync(cnt.data(), wm->nb_cnt, B * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaMemcpyAsync(gl.data(), wm->gen_len, B * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaStreamSynchronize(ws));
      int64_t g = 0;
      for (int j = 0; j < B; ++j) {
        g += gl[j];
        for (int r = 0; r < cnt[j] && r < NB; ++r) {
          const int L = len[(size_t)j * NB + r];
          const int* t = tok.data() + ((size_t)j * NB + r) * Tm;
          const int ol = (L > 0 && t[L - 1] == eos) ? L - 1 : L;
          outs[(size_t)order[j] * NB + r].assign(t, t + ol);
          scores[(size_t)order[j] * NB + r] = sc[(size_t)j * NB + r];
        }
      }
      return g;
    };
    translate_core(m, h_off, n, opts, load_src, emit, stats, s);
    int64_t pos = 0;
    h_out_off[0] = 0;
    for (size_t i = 0; i < outs.size(); ++i) {
      NMT_REQUIRE(pos + (int64_t)outs[i].size() <= out_cap, NMT_E_SHAPE, "out_cap too small");
      std::copy(outs[i].begin(), outs[i].end(), h_out + pos);
      pos += outs[i].size();
      h_out_off[i + 1] = pos;
      if (h_score) h_score[i] = scores[i];
    }
    if (stats) stats->out_tokens = pos;
  });
}

nmt_status nmt_ensemble_create(nmt_model* const* members, int32_t n, nmt_ensemble** out) {
  return guard([&] {
    NMT_REQUIRE(members && out && n >= 1 && n <= 8, NMT_E_ARG, "need 1..8 members");
    nmt_model* m0 = members[0];
    NMT_REQUIRE(m0, NMT_E_ARG, "null member");
    for (int k = 0; k < n; ++k) {
      const nmt_model* m = members[k];
      NMT_REQUIRE(m, NMT_E_ARG, "null member");
      NMT_REQUIRE(m->cfg.vocab_size == m0->cfg.vocab_size && m->cfg.eos_id == m0->cfg.eos_id &&
                      m->cfg.bos_id == m0->cfg.bos_id && m->cfg.pad_id == m0->cfg.pad_id &&
                      m->cfg.max_src_len == m0->cfg.max_src_len,
                  NMT_E_SHAPE, "ensemble members need one vocabulary and special ids");
      NMT_REQUIRE(m->prec == m0->prec && m->device == m0->device, NMT_E_ARG,
                  "ensemble members need one precision and device");
      NMT_REQUIRE(m->lim.max_tokens == m0->lim.max_tokens && m->lim.max_sents == m0->lim.max_sents &&
                      m->lim.max_tgt_len == m0->lim.max_tgt_len && m->lim.beam == m0->lim.beam,
                  NMT_E_SHAPE, "ensemble members need equal limits");
      NMT_REQUIRE(m->lim.beam >= 2, NMT_E_ARG, "ensembles decode with beam search (limits.beam >= 2)");
    }
    std::unique_ptr<nmt_ensemble> e(new nmt_ensemble());
    for (int k = 0; k < n; ++k) e->members.push_back(clone_worker(members[k]));
    nmt_model* c0 = e->members[0];
    for (int k = 1; k < n; ++k) {   // one search state: alias clone 0's
      nmt_model* c = e->members[k];
      c->src = c0->src; c->src_len = c0->src_len; c->tgt_cap = c0->tgt_cap;
      c->row_slot = c0->row_slot; c->prev_tok = c0->prev_tok; c->done = c0->done;
      c->out_tok = c0->out_tok; c->gen_len = c0->gen_len; c->st = c0->st; c->bad = c0->bad;
      c->keys = c0->keys; c->bscore = c0->bscore; c->anc = c0->anc; c->htok = c0->htok;
      c->best_score = c0->best_score; c->cand_v = c0->cand_v; c->cand_i = c0->cand_i;
      c->nb_score = c0->nb_score; c->nb_len = c0->nb_len; c->nb_tok = c0->nb_tok;
      c->nb_cnt = c0->nb_cnt;
    }
    const size_t R = (size_t)c0->lim.max_sents * c0->lim.beam;
    cudaError_t err = cudaMalloc(&e->ens, R * c0->cfg.vocab_size * 4);
    NMT_REQUIRE(err == cudaSuccess, NMT_E_RESOURCE, "ensemble buffer cudaMalloc failed");
    *out = e.release();
  });
}

void nmt_ensemble_free(nmt_ensemble* e) { delete e; }

nmt_status nmt_translate_ensemble(nmt_ensemble* e, const int32_t* h_ids, const int64_t* h_off,
                                  int64_t n, const nmt_translate_opts* opts, int32_t* h_out,
                                  int64_t out_cap, int64_t* h_out_off, float* h_score,
                                  nmt_stats* stats, void* stream) {
  return guard([&] {
    NMT_REQUIRE(e && h_ids && h_off && h_out && h_out_off && opts && n >= 0, NMT_E_ARG,
                "null argument");
    nmt_model* c0 = e->members[0];
    const int nm = (int)e->members.size();
    const int K = opts->beam, NB = opts->nbest > 1 ? opts->nbest : 1;
    NMT_REQUIRE(K >= 2 && K <= c0->lim.beam && K <= 4, NMT_E_ARG,
                "ensemble beam must be in [2, min(4, limits.beam)]");
    NMT_REQUIRE(NB <= K, NMT_E_ARG, "nbest must be <= beam");
    cudaStream_t s = (cudaStream_t)stream;
    const int V = c0->cfg.vocab_size, eos = c0->cfg.eos_id, Tm = c0->lim.max_tgt_len;
    const int max_tokens = opts->max_tokens > 0 ? opts->max_tokens : c0->lim.max_tokens;
    const int max_sents = opts->max_sents > 0 ? opts->max_sents : c0->lim.max_sents;
    const int every = opts->prune_every > 0 ? opts->prune_every : 1;
    const float ratio = opts->prune_ratio;
    const int sync_every = opts->sync_every > 0 ? opts->sync_every : 4;
    NMT_REQUIRE(max_tokens <= c0->lim.max_tokens && max_sents <= c0->lim.max_sents, NMT_E_ARG,
                "translate opts exceed the model limits");
    int64_t truncated = 0;
    const std::vector<int> elen = effective_lengths(c0, h_off, n, max_tokens, &truncated);
    auto t0 = std::chrono::steady_clock::now();
    Plan p = plan_batches(elen.data(), n, max_tokens, max_sents);
    const int nb = (int)p.bstart.size() - 1;
    std::vector<std::vector<int>> outs((size_t)n * NB);
    std::vector<float> scores((size_t)n * NB, -INFINITY);
    std::vector<const float*> lg(nm);
    for (int k = 0; k < nm; ++k) lg[k] = e->members[k]->blogits;
    const int R = c0->lim.max_sents * c0->lim.beam;   // row capacity (graph buckets)
    int64_t steps = 0, prunes = 0, gen = 0;
    std::vector<int> lens, caps;
    for (int bi = 0; bi < nb; ++bi) {
      const int lo = p.bstart[bi], B = p.bstart[bi + 1] - lo;
      const int S = elen[p.order[lo]];
      lens.resize(B);
      caps.resize(B);
      for (int j = 0; j < B; ++j) {
        const int sid = p.order[lo + j];
        lens[j] = elen[sid];
        caps[j] = opts->h_tgt_cap ? opts->h_tgt_cap[sid] : Tm;
        const int32_t* src = h_ids + h_off[sid];
        const bool cut = h_off[sid + 1] - h_off[sid] > lens[j];
        for (int q = 0; q < S; ++q) {
          int v = q < lens[j] ? src[q] : c0->cfg.pad_id;
          NMT_REQUIRE(v >= 0 && v < V, NMT_E_INPUT, "token id out of range");
          if (cut && q == lens[j] - 1) v = c0->cfg.eos_id;
          c0->hp.src[(size_t)j * S + q] = v;
        }
      }
      NMT_CUDA(cudaMemcpyAsync(c0->src, c0->hp.src, (size_t)B * S * 4, cudaMemcpyHostToDevice, s));
      for (auto* c : e->members) encode_common(c, B, S, lens.data(), caps.data(), s, K);
      c0->batch.NB = NB;
      const int* dR = &c0->st->n_live;
      int rows = B * K, t = 0;
      // one ensemble step for `rr` (>= live) rows: every member's decoder on its own caches,
      // the distribution average (R26), the beam update and pruning; all kernels read t, the
      // live count and S from device memory, so a captured step serves every step
      auto step = [&](int rr) {
        for (auto* c : e->members) {
          c->batch.rows_upper = rr;
          decode_step_any(c, &c->batch, nullptr, nullptr, s, /*finish=*/false);
        }
        ens_combine(lg.data(), nm, V, dR, rr, e->ens, s);
        beam_row_topk(e->ens, V, 2 * K, dR, rr, c0->cand_v, c0->cand_i, s);
        beam_select(K, c0->cand_v, c0->cand_i, c0->bscore, c0->prev_tok, c0->done, c0->row_slot,
                    c0->tgt_cap, c0->anc, c0->htok, Tm, c0->best_score, c0->out_tok, c0->gen_len,
                    c0->st, V, eos, rr, s, NB, c0->nb_score, c0->nb_len, c0->nb_tok, c0->nb_cnt);
        prune_compact(c0->st, c0->row_slot, c0->prev_tok, c0->done, every, ratio, nullptr, rr, s,
                      c0->bscore);
      };
      unsigned rb;
      memcpy(&rb, &ratio, 4);
      for (; t < c0->batch.max_cap && rows > 0; ++t) {
        const int bucket = std::min((int)R, (rows + 31) & ~31);
        const auto key = std::make_tuple(bucket, NB, every, rb);
        if (s == nullptr || !e->eager_keys.count(key)) {
          step(rows);   // legacy stream (no capture) / first use of a configuration
          e->eager_keys.insert(key);
        } else {
          auto it = e->graphs.find(key);
          if (it == e->graphs.end()) {
            cudaGraph_t g;
            NMT_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            g_pdl = pdl_enabled();
            try {
              step(bucket);
            } catch (...) {
              g_pdl = false;
              cudaStreamEndCapture(s, &g);
              throw;
            }
            g_pdl = false;
            NMT_CUDA(cudaStreamEndCapture(s, &g));
            size_t nn = 0;
            NMT_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
            std::vector<cudaGraphNode_t> ns(nn);
            if (nn) NMT_CUDA(cudaGraphGetNodes(g, ns.data(), &nn));
            int nodes = 0;
            for (auto nd : ns) {
              cudaGraphNodeType ty;
              NMT_CUDA(cudaGraphNodeGetType(nd, &ty));
              nodes += ty == cudaGraphNodeTypeKernel;
            }
            cudaGraphExec_t ex;
            NMT_CUDA(cudaGraphInstantiate(&ex, g, 0));
            NMT_CUDA(cudaGraphDestroy(g));
            it = e->graphs.emplace(key, std::make_pair(ex, nodes)).first;
          }
          NMT_CUDA(cudaGraphLaunch(it->second.first, s));
          g_launches += it->second.second;
        }
        for (auto* c : e->members) c->batch.step = t + 1;
        if ((t + 1) % sync_every == 0) {
          poll_state(c0, s);
          rows = c0->hp.st->n_live;
        }
      }
      poll_state(c0, s);
      steps += t;
      prunes += c0->hp.st->prunes;
      // results: the N-best lists (NB >= 2) or the best hypothesis
      std::vector<int> gl(B);
      NMT_CUDA(cudaMemcpyAsync(gl.data(), c0->gen_len, B * 4, cudaMemcpyDeviceToHost, s));
      if (NB >= 2) {
        std::vector<int> tok((size_t)B * NB * Tm), len((size_t)B * NB), cnt(B);
        std::vector<float> sc((size_t)B * NB);
        NMT_CUDA(cudaMemcpyAsync(tok.data(), c0->nb_tok, tok.size() * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaMemcpyAsync(len.data(), c0->nb_len, len.size() * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaMemcpyAsync(sc.data(), c0->nb_score, sc.size() * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaMemcpyAsync(cnt.data(), c0->nb_cnt, B * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < B; ++j)
          for (int r = 0; r < cnt[j] && r < NB; ++r) {
            const int L = len[(size_t)j * NB + r];
            const int* tk = tok.data() + ((size_t)j * NB + r) * Tm;
            const int ol = (L > 0 && tk[L - 1] == eos) ? L - 1 : L;
            outs[(size_t)p.order[lo + j] * NB + r].assign(tk, tk + ol);
            scores[(size_t)p.order[lo + j] * NB + r] = sc[(size_t)j * NB + r];
          }
      } else {
        std::vector<int> tok((size_t)B * Tm);
        std::vector<float> sc(B);
        NMT_CUDA(cudaMemcpyAsync(tok.data(), c0->out_tok, tok.size() * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaMemcpyAsync(sc.data(), c0->best_score, B * 4, cudaMemcpyDeviceToHost, s));
        NMT_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < B; ++j) {
          const int L = gl[j];
          const int* tk = tok.data() + (size_t)j * Tm;
          const int ol = (L > 0 && tk[L - 1] == eos) ? L - 1 : L;
          outs[p.order[lo + j]].assign(tk, tk + ol);
          scores[p.order[lo + j]] = sc[j];
        }
      }
      for (int j = 0; j < B; ++j) gen += gl[j];
      for (auto* c : e->members) c->batch.valid = false;
    }
    int64_t pos = 0;
    h_out_off[0] = 0;
    for (size_t i = 0; i < outs.size(); ++i) {
      NMT_REQUIRE(pos + (int64_t)outs[i].size() <= out_cap, NMT_E_SHAPE, "out_cap too small");
      std::copy(outs[i].begin(), outs[i].end(), h_out + pos);
      pos += outs[i].size();
      h_out_off[i + 1] = pos;
      if (h_score) h_score[i] = scores[i];
    }
    if (stats) {
      *stats = nmt_stats{};
      stats->sentences = n;
      stats->gen_tokens = gen;
      stats->out_tokens = pos;
      stats->decode_steps = steps;
      stats->prunes = prunes;
      stats->batches = nb;
      stats->truncated = truncated;
      for (auto* c : e->members) stats->arena_system_allocs += c->sys_allocs;
      stats->ms_total = std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - t0).count();
    }
  });
}

nmt_status nmt_translate_device(nmt_model* m, const int32_t* d_ids, const int64_t* h_off,
                                int64_t n, const nmt_translate_opts* opts, int32_t* d_out,
                                int32_t out_stride, int32_t* d_out_len, nmt_stats* stats,
                                void* stream) {
  return guard([&] {
    NMT_REQUIRE(m && d_ids && h_off && d_out && d_out_len && n >= 0, NMT_E_ARG, "null argument");
    NMT_REQUIRE(out_stride >= m->lim.max_tgt_len, NMT_E_ARG, "out_stride < max_tgt_len");
    cudaStream_t s = (cudaStream_t)stream;
    const int Tm = m->lim.max_tgt_len;
    NMT_CUDA(cudaMemsetAsync(m->bad, 0, 4, s));
    for (auto* w : m->workers) NMT_CUDA(cudaMemsetAsync(w->bad, 0, 4, s));
    auto load_src = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B, int S,
                        const int* lens) {
      for (int j = 0; j < B; ++j) {
        wm->hp.boff[j] = h_off[order[j]];
        const bool cut = h_off[order[j] + 1] - h_off[order[j]] > lens[j];
        wm->hp.blen[j] = cut ? -lens[j] : lens[j];   // negative: truncated, EOS last
      }
      NMT_CUDA(cudaMemcpyAsync(wm->boff, wm->hp.boff, B * 8, cudaMemcpyHostToDevice, ws));
      NMT_CUDA(cudaMemcpyAsync(wm->blen, wm->hp.blen, B * 4, cudaMemcpyHostToDevice, ws));
      pack_sources(d_ids, wm->boff, wm->blen, B, S, wm->src, wm->cfg.vocab_size, wm->bad,
                   wm->cfg.eos_id, ws);
    };
    auto emit = [&](nmt_model* wm, cudaStream_t ws, const int* order, int B) -> int64_t {
      for (int j = 0; j < B; ++j) wm->hp.sent[j] = order[j];
      NMT_CUDA(cudaMemcpyAsync(wm->sent_ids, wm->hp.sent, B * 4, cudaMemcpyHostToDevice, ws));
      scatter_outputs(wm->out_tok, Tm, wm->gen_len, wm->sent_ids, B, d_out, out_stride, d_out_len,
                      ws);
      NMT_CUDA(cudaMemcpyAsync(wm->hp.gen_len, wm->gen_len, B * 4, cudaMemcpyDeviceToHost, ws));
      NMT_CUDA(cudaStreamSynchronize(ws));  // staging buffers are reused by the next batch
      int64_t g = 0;
      for (int j = 0; j < B; ++j) g += wm->hp.gen_len[j];
      return g;
    };
    translate_core(m, h_off, n, opts, load_src, emit, stats, s);
    int bad = 0;
    for (nmt_model* wm : [&] { std::vector<nmt_model*> v{m}; for (auto* w : m->workers) v.push_back(w); return v; }()) {
      NMT_CUDA(cudaMemcpyAsync(wm->hp.bad, wm->bad, 4, cudaMemcpyDeviceToHost, s));
      NMT_CUDA(cudaStreamSynchronize(s));
      bad |= *wm->hp.bad;
    }
    NMT_REQUIRE(bad == 0, NMT_E_INPUT, "token id out of range in d_ids");
  });
}

nmt_status nmt_profile(nmt_model* m, int32_t mode, nmt_prof_entry* out, int32_t cap,
                       int32_t* n_out) {
  return guard([&] {
    NMT_REQUIRE(m, NMT_E_ARG, "null model");
    NMT_CUDA(cudaDeviceSynchronize());
    prof_flush(m);
    if (out) {
      NMT_REQUIRE(n_out, NMT_E_ARG, "null n_out");
      int n = 0;
      for (int c = 0; c < P_NCLS && n < cap; ++c) {
        if (!m->prof.n[c]) continue;
        nmt_prof_entry& e = out[n++];
        memset(&e, 0, sizeof(e));
        strncpy(e.name, kProfNames[c], sizeof(e.name) - 1);
        e.launches = m->prof.n[c];
        e.ms = m->prof.ms[c];
        e.flops = m->prof.flops[c];
        e.bytes = m->prof.bytes[c];
      }
      *n_out = n;
    }
    if (mode == 2 || mode == 0) {  // reset counters
      auto& P = m->prof;
      P.steps.clear();
      std::fill(P.ms, P.ms + 16, 0.0);
      std::fill(P.flops, P.flops + 16, 0.0);
      std::fill(P.bytes, P.bytes + 16, 0.0);
      std::fill(P.n, P.n + 16, 0ll);
    }
    if (mode == 3) m->prof.steps.clear();
    if (mode >= 0 && mode <= 3) {
      m->prof.on = (mode != 0);
      m->prof.steps_only = (mode == 3);
    }
  });
}

nmt_status nmt_debug_gemm_trace(uint64_t* h_out, int64_t cap) {
  return guard([&] {
    NMT_REQUIRE(h_out && cap > 0, NMT_E_ARG, "null argument");
    tc::gemm_trace(reinterpret_cast<unsigned long long*>(h_out),
                   (int)std::min<int64_t>(cap, 148 * 32 * 8));
  });
}

nmt_status nmt_debug_attn_trace(uint64_t* h_out, int64_t cap) {
  return guard([&] {
    NMT_REQUIRE(h_out && cap > 0, NMT_E_ARG, "null argument");
    attn_umma_trace(reinterpret_cast<unsigned long long*>(h_out), (int)std::min<int64_t>(cap, 1024));
  });
}

nmt_status nmt_debug_fused_trace(nmt_model* m, uint64_t* h_out, int64_t cap) {
  return guard([&] {
    NMT_REQUIRE(m && h_out, NMT_E_ARG, "null argument");
    NMT_REQUIRE(m->fused_trace, NMT_E_STATE, "load with NMT_FUSED_TRACE set to record the trace");
    NMT_CUDA(cudaDeviceSynchronize());
    const int64_t n = std::min<int64_t>(cap, 4 * 65536 + 1024);
    NMT_CUDA(cudaMemcpy(h_out, m->fused_trace, n * 8, cudaMemcpyDeviceToHost));
  });
}

nmt_status nmt_profile_steps(nmt_model* m, nmt_step_rec* out, int32_t cap, int32_t* n_out) {
  return guard([&] {
    NMT_REQUIRE(m && n_out && (out || cap == 0), NMT_E_ARG, "null argument");
    const auto& v = m->prof.steps;
    const int n = (int)std::min<size_t>(v.size(), (size_t)std::max(0, cap));
    for (int i = 0; i < n; ++i) out[i] = nmt_step_rec{v[i].t, v[i].live, v[i].ms};
    *n_out = (int)v.size();
  });
}

nmt_status nmt_dev_gemm(nmt_precision prec, int32_t M, int32_t N, int32_t K, const void* d_A,
                        int32_t lda, const void* d_B, int32_t ldb, const void* d_bias,
                        const void* d_R, int32_t ldr, void* d_C, int32_t ldc, int32_t relu,
                        void* stream) {
  return guard([&] {
    NMT_REQUIRE(d_A && d_B && d_C && M >= 0 && N > 0 && K > 0, NMT_E_ARG, "bad gemm args");
    NMT_REQUIRE(K % 16 == 0, NMT_E_SHAPE, "K must be a multiple of 16");
    GemmArgs a;
    a.M = M; a.N = N; a.K = K; a.A = d_A; a.lda = lda; a.B = d_B; a.ldb = ldb; a.bias = d_bias;
    a.R = d_R; a.ldr = ldr; a.C = d_C; a.ldc = ldc; a.relu = relu;
    if (prec == NMT_FP16) gemm<__half>(a, (cudaStream_t)stream);
    else gemm<float>(a, (cudaStream_t)stream);
  });
}

nmt_status nmt_dev_gemm_decode(int32_t M, int32_t N, int32_t K, const void* d_A, int32_t lda,
                               const void* d_B, int32_t ldb, const void* d_bias, const void* d_R,
                               int32_t ldr, void* d_C, int32_t ldc, int32_t relu, void* stream) {
  return guard([&] {
    NMT_REQUIRE(d_A && d_B && d_C && M > 0 && M <= 16384 && N > 0 && K > 0, NMT_E_ARG,
                "bad gemm args");
    NMT_REQUIRE(K % 16 == 0, NMT_E_SHAPE, "K must be a multiple of 16");
    static float* ws = nullptr;   // test hook scratch (not on the product path)
    static int* cnt = nullptr;
    const int sp = decode_splits(N, K);
    const size_t need = (size_t)((M + 127) / 128) * ((N + 63) / 64) * sp * 128 * 64;
    static size_t have = 0;
    if (need > have) {
      if (ws) cudaFree(ws);
      if (cnt) cudaFree(cnt);
      NMT_CUDA(cudaMalloc(&ws, need * 4));
      NMT_CUDA(cudaMalloc(&cnt, 65536 * 4));
      NMT_CUDA(cudaMemset(cnt, 0, 65536 * 4));
      have = need;
    }
    GemmArgs a;
    a.M = M; a.N = N; a.K = K; a.A = d_A; a.lda = lda; a.B = d_B; a.ldb = ldb; a.bias = d_bias;
    a.R = d_R; a.ldr = ldr; a.C = d_C; a.ldc = ldc; a.relu = relu;
    a.ws = ws; a.counters = cnt;
    decode_config(a);
    gemm<__half>(a, (cudaStream_t)stream);
  });
}

nmt_status nmt_dev_gemm_argmax(nmt_precision prec, int32_t M, int32_t N, int32_t K,
                               const void* d_A, int32_t lda, const void* d_B, int32_t ldb,
                               int32_t* d_next, float* d_logits, void* stream) {
  return guard([&] {
    NMT_REQUIRE(d_A && d_B && d_next && M > 0 && N > 0 && K > 0, NMT_E_ARG, "bad gemm args");
    NMT_REQUIRE(K % 16 == 0 && M <= 16384, NMT_E_SHAPE, "K % 16 != 0 or M > 16384");
    cudaStream_t s = (cudaStream_t)stream;
    static unsigned long long* keys = nullptr;  // test hook scratch (not on the product path)
    if (!keys) NMT_CUDA(cudaMalloc(&keys, 16384 * 8));
    NMT_CUDA(cudaMemsetAsync(keys, 0, (size_t)M * 8, s));
    GemmArgs a;
    a.M = M; a.N = N; a.K = K; a.A = d_A; a.lda = lda; a.B = d_B; a.ldb = ldb;
    a.argmax = keys; a.logits = d_logits;
    if (prec == NMT_FP16) gemm<__half>(a, s);
    else gemm<float>(a, s);
    argmax_ids(keys, d_next, M, s);
  });
}

nmt_status nmt_dev_attn_encoder(nmt_precision prec, int32_t B, int32_t S, int32_t d, int32_t H,
                                int32_t kclip, int32_t use_rpr, const void* d_qkv,
                                const int32_t* d_len, const void* d_relk, const void* d_relv,
                                void* d_out, void* stream) {
  return guard([&] {
    NMT_REQUIRE(d_qkv && d_len && d_out && B > 0 && S > 0 && H > 0 && d % H == 0, NMT_E_ARG,
                "bad attention args");
    NMT_REQUIRE(!use_rpr || (d_relk && d_relv), NMT_E_ARG, "RPR tables missing");
    NMT_REQUIRE(S <= 128 && 2 * kclip + 1 <= 31, NMT_E_SHAPE, "S > 128 or 2k+1 > 31");
    cudaStream_t s = (cudaStream_t)stream;
    if (prec == NMT_FP16)
      attn_encoder<__half>(static_cast<const __half*>(d_qkv), d_len,
                           static_cast<const __half*>(d_relk), static_cast<const __half*>(d_relv),
                           static_cast<__half*>(d_out), B, S, d, H, kclip, use_rpr, s);
    else
      attn_encoder<float>(static_cast<const float*>(d_qkv), d_len,
                          static_cast<const float*>(d_relk), static_cast<const float*>(d_relv),
                          static_cast<float*>(d_out), B, S, d, H, kclip, use_rpr, s);
  });
}

}  // extern "C"
