// forward.cu — launch sequences of the encoder (once per batch) and of one greedy decode
// step.  Every arithmetic step runs in the kernels of kernels.cu / attention.cu / gemm_*.cu.
//
// Encoder (Eq. 1-2):
//   y0 = sqrt(d) E[s] + PE;  z0 = LN^dl_0(y0);  x1 = W1_0 z0;  u = LN^a_1(x1)      [embed, dlcl]
//   per layer l: QKV = u Wqkv^T + b                                                [gemm]
//                o = RPRAttn(QKV)                                                   [attn]
//                x = x + o Wo^T + bo         (residual in the GEMM epilogue)       [gemm]
//                u = LN^f(x);  h = relu(u W1^T + b1);  x = x + h W2^T + b2          [ln, gemm x2]
//                z_l = LN^dl_l(x); x = sum_k W^{(l+1)}_k z_k; u = LN^a_{l+1}(x)     [dlcl]
//   enc = LN^enc(sum_k W^{(L+1)}_k z_k);  [CK|CV]_m = enc Wkv_m^T + b for all m     [dlcl, gemm]
// Decode step t, rows = live batch rows:
//   g = sqrt(d) E[w_t] + PE(t), u = LN^s(g)                                         [embed_dec_ln]
//   qkv = u Wqkv^T + b; cached RPR self-attn (appends k_t, v_t); g += o Wso^T + b     [gemm, attn, gemm]
//   q = LN^c(g) Wq^T + b; cross-attn over cached CK/CV; g += o Wco^T + b              [ln, gemm, attn, gemm]
//   g += relu(LN^f(g) W1^T + b1) W2^T + b2                                            [ln, gemm x2]
//   next = argmax_v LN^dec(g) . E[v]   (fused vocab GEMM + argmax)                    [ln, gemm]
//   sticky done flags, outputs per slot                                               [finish]
#include <cmath>

#include "decode_fused.h"
#include "engine.h"
#include "tc_dev.cuh"

namespace nmt {

const char* kProfNames[P_NCLS] = {"enc_gemm",  "enc_rpr_attn", "dlcl_combine", "enc_layernorm",
                                  "embed",     "dec_gemm",     "vocab_argmax", "dec_self_attn",
                                  "dec_cross_attn", "dec_layernorm", "bookkeeping", "dec_fused"};

void prof_flush(nmt_model* m) {
  auto& P = m->prof;
  for (auto& r : P.pending) {
    float ms = 0.f;
    NMT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    P.ms[r.cls] += ms;
    P.flops[r.cls] += r.flops;
    P.bytes[r.cls] += r.bytes;
    P.n[r.cls] += 1;
  }
  P.pending.clear();
  P.used = 0;
}

namespace {

double gemm_bytes(const GemmArgs& a, size_t tb) {
  double b = ((double)a.M * a.K + (double)a.N * a.K) * tb;
  if (!a.argmax) b += (double)a.M * a.N * tb;
  if (a.R) b += (double)a.M * a.N * tb;
  if (a.bias) b += (double)a.N * tb;
  return b;
}
double gemm_flops(const GemmArgs& a) { return 2.0 * a.M * a.N * a.K; }

GemmArgs mk(int M, int N, int K, const void* A, int lda, const void* B, int ldb, const void* bias,
            void* C, int ldc) {
  GemmArgs a;
  a.M = M; a.N = N; a.K = K; a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.bias = bias;
  a.C = C; a.ldc = ldc;
  return a;
}

template <class T> const T* cT(const void* p) { return static_cast<const T*>(p); }

// Decode-size GEMM (rows = live batch rows): 64-wide output tiles and a fixed split-K
// factor that depends on the weight shape only (batch invariance), see gemm_tc.cu.
GemmArgs dec_cfg(nmt_model* m, GemmArgs a) {
  decode_config(a);
  a.ws = m->gemm_ws;
  a.counters = m->gemm_cnt;
  return a;
}

template <class T>
void encode_impl(nmt_model* m, int B, int S, cudaStream_t s) {
  const nmt_config& c = m->cfg;
  const int d = c.d_model, F = c.d_ffn, H = c.n_heads, L = c.enc_layers, Ld = c.dec_layers;
  const int N = B * S;
  const float eps = c.ln_eps;
  const size_t tb = sizeof(T);
  T *x = (T*)m->x, *u = (T*)m->u, *qkv = (T*)m->qkv, *o = (T*)m->o, *h = (T*)m->h,
    *enc = (T*)m->enc_out, *hist = (T*)m->hist, *ckv = (T*)m->ckv;
  const size_t hs = (size_t)N * d;
  const double row = (double)N * d * tb;  // bytes of one [N][d] activation
  const float sq = std::sqrt((float)d);
  PROF(P_EMBED, 0, 2 * row,
       embed<T>(m->src, cT<T>(m->emb), m->pe, c.use_dlcl ? o : x, N, d, S, nullptr, nullptr, sq, s));
  const EncW& w0 = m->enc[0];
  // DLCL lookahead in blocks of `la` boundaries (kernels.h dlcl_combine): the first boundary
  // k0 of a block (combination row k0+1) also produces the partials of rows k0+2 ..
  // k0+la (those <= L+1 exist); boundary k0+i starts from partial i and the i-1 history rows
  // written since k0.  la = 1: no lookahead (NMT_NO_DLCL_LA, A/B); NMT_DLCL_LA overrides.
  const int la = dlcl_blocks(c, d);
  struct DlclStep { int mode, arg; float* P; };
  auto dlcl_step = [&](int k) -> DlclStep {
    if (la <= 1) return {0, 0, nullptr};
    const int k0 = k / la * la, i = k - k0;
    if (i == 0) {
      const int np = std::min(la - 1, L - k);   // partial i targets row k+1+i <= L+1
      return np > 0 ? DlclStep{1, np, m->dlcl_p} : DlclStep{0, 0, nullptr};
    }
    return {2, i - 1, m->dlcl_p + (size_t)(i - 1) * hs};
  };
  // bytes: y + history rows read (mode 2: arg rows) + z, x, u written; FP32 partials written
  // (mode 1: arg of them) or read (mode 2: one)
  auto dlcl_bytes = [&](int k, const DlclStep& st, bool last) {
    const int rd = st.mode == 2 ? st.arg : st.mode == 1 ? k : k;
    const int np = st.mode == 1 ? st.arg : st.mode == 2 ? 1 : 0;
    return (1 + rd + 1 + (last ? 0 : 1) + 1) * row + np * row * 4.0 / tb;
  };
  if (c.use_dlcl) {
    const DlclStep st = dlcl_step(0);
    PROF(P_DLCL, 0, dlcl_bytes(0, st, false),
         dlcl_combine<T>(o, hist, hs, 0, m->dlcl_w, cT<T>(m->dl0_g), cT<T>(m->dl0_b), c.dlcl_ln,
                         cT<T>(w0.attn_g), cT<T>(w0.attn_b), x, u, N, d, eps, s, st.mode,
                         m->dlcl_w, st.P, st.arg));
  } else {
    PROF(P_ENC_LN, 0, 2 * row,
         layernorm<T>(x, d, cT<T>(w0.attn_g), cT<T>(w0.attn_b), u, d, N, d, eps, nullptr, s));
  }
  const double attn_flops = 4.0 * B * H * (double)S * S * (d / H);
  for (int l = 0; l < L; ++l) {
    const EncW& w = m->enc[l];
    GemmArgs a = mk(N, 3 * d, d, u, d, w.qkv_w, d, w.qkv_b, qkv, 3 * d);
    PROF(P_ENC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));
    PROF(P_ENC_ATTN, attn_flops, 4 * row,
         attn_encoder<T>(qkv, m->src_len, cT<T>(w.relk), cT<T>(w.relv), o, B, S, d, H,
                         c.max_rel_pos, c.use_rpr, s));
    a = mk(N, d, d, o, d, w.out_w, d, w.out_b, x, d);
    a.R = x; a.ldr = d;
    PROF(P_ENC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));  // a = x + Attn(LN(x))
    PROF(P_ENC_LN, 0, 2 * row,
         layernorm<T>(x, d, cT<T>(w.ffn_g), cT<T>(w.ffn_b), u, d, N, d, eps, nullptr, s));
    a = mk(N, F, d, u, d, w.w1, d, w.b1, h, F);
    a.relu = 1;
    PROF(P_ENC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));
    a = mk(N, d, F, h, F, w.w2, F, w.b2, x, d);
    a.R = x; a.ldr = d;
    PROF(P_ENC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));  // y_l = a + FFN(LN(a))
    const bool last = (l == L - 1);
    const T* ng = last ? cT<T>(m->enc_fg) : cT<T>(m->enc[l + 1].attn_g);
    const T* nb = last ? cT<T>(m->enc_fb) : cT<T>(m->enc[l + 1].attn_b);
    if (c.use_dlcl) {
      const int k = l + 1;  // depth of y
      const DlclStep st = dlcl_step(k);
      PROF(P_DLCL, 0, dlcl_bytes(k, st, last),
           dlcl_combine<T>(x, hist, hs, k, m->dlcl_w + (size_t)(k + 1) * k / 2, cT<T>(w.dl_g),
                           cT<T>(w.dl_b), c.dlcl_ln, ng, nb, last ? nullptr : x,
                           last ? enc : u, N, d, eps, s, st.mode, m->dlcl_w, st.P, st.arg));
    } else {
      PROF(P_ENC_LN, 0, 2 * row,
           layernorm<T>(x, d, ng, nb, last ? enc : u, d, N, d, eps, nullptr, s));
    }
  }
  // cross K/V of every decoder layer, once per sentence
  GemmArgs a = mk(N, Ld * 2 * d, d, enc, d, m->ckv_w, d, m->ckv_b, ckv, Ld * 2 * d);
  PROF(P_ENC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));
}

// ---------------------------------------------------------------- fused decode step
// Live-row threshold of the single fused launch (embedding ... final LN in one persistent
// kernel, decode_fused.cu); above it the attention phases run as the standalone kernels
// (more warps in flight per SM for the latency-bound KV reads) between fused GEMM segments.
// (NMT_FUSE_ROWS / NMT_NO_FUSE are read when the model is loaded: nmt_model::fuse_rows)
bool fused_enabled(const nmt_model* m) {
  const nmt_config& c = m->cfg;
  return m->fuse_rows >= 0 && m->prec == NMT_FP16 && !m->fold.empty() && m->fused_ctr &&
         fused_supported(c.d_model, c.n_heads, c.d_ffn, c.dec_layers);
}

// Parameter block of the fused step (every buffer and weight is fixed after load): the six
// projections of each decoder layer with the unfused path's operands, LN folding and shape
// policy (gemm_tc.cu decode_config), their TMA descriptors over the row capacity.
const FusedParams& fused_params(nmt_model* m) {
  if (m->fused) return *m->fused;
  const nmt_config& c = m->cfg;
  const int d = c.d_model, F = c.d_ffn, Ld = c.dec_layers;
  const int Rmax = m->lim.max_sents * std::max(1, m->lim.beam);
  const int Tm = m->lim.max_tgt_len;
  std::unique_ptr<FusedParams> P(new FusedParams());
  memset(P.get(), 0, sizeof(FusedParams));
  auto H = [](const void* p) { return static_cast<const __half*>(p); };
  auto Hm = [](void* p) { return static_cast<__half*>(p); };
  for (int l = 0; l < Ld; ++l) {
    const DecW& w = m->dec[l];
    const DecFold& f = m->fold[l];
    FusedLayer& L = P->L[l];
    auto set = [&](int slot, const void* A, int K, const void* B, int N, const void* bias,
                   const void* R, void* C, int ldc, int relu, float2* st_out,
                   const float2* ln_st, const float* ln_c) {
      GemmPhase& G = L.g[slot];
      G.N = N; G.K = K; G.relu = relu; G.ldc = ldc;
      G.bias = H(bias); G.R = H(R); G.C = Hm(C);
      G.st_out = st_out; G.ln_st = ln_st; G.ln_c = ln_c;
      // decode_config: split-K 2 for K >= 2048 without LN statistics, 64-wide tiles for the
      // d x d projections, 128-wide otherwise
      G.split = (K >= 2048 && !st_out && !ln_st && ((K + 63) / 64) % 2 == 0) ? 1 : 0;
      G.bn = G.split ? 64 : (N <= 512 && K <= 512) ? 64 : 128;
      if (N % G.bn || K % 64) throw CudaError("fused decode: projection shape not tileable");
      G.nt = N / G.bn;
      L.ma[slot] = tc::make_map(A, Rmax, K, K, 128);
      L.ma32[slot] = tc::make_map(A, Rmax, K, K, 32);
      L.mb[slot] = tc::make_map(B, N, K, K, G.bn);
    };
    if (l == 0)
      set(0, m->du, d, w.qkv_w, 3 * d, w.qkv_b, nullptr, m->dqkv, 3 * d, 0, nullptr, nullptr, nullptr);
    else
      set(0, m->g, d, f.qkv.w, 3 * d, f.qkv.b, nullptr, m->dqkv, 3 * d, 0, nullptr, m->lnst, f.qkv.c);
    set(1, m->dout, d, w.so_w, d, w.so_b, m->g, m->g, d, 0, m->lnst, nullptr, nullptr);
    set(2, m->g, d, f.cq.w, d, f.cq.b, nullptr, m->dq, d, 0, nullptr, m->lnst, f.cq.c);
    set(3, m->dout, d, w.co_w, d, w.co_b, m->g, m->g, d, 0, m->lnst, nullptr, nullptr);
    set(4, m->g, d, f.w1.w, F, f.w1.b, nullptr, m->dh, F, 1, nullptr, m->lnst, f.w1.c);
    set(5, m->dh, F, w.w2, d, w.b2, m->g, m->g, d, 0, l + 1 < Ld ? m->lnst : nullptr, nullptr, nullptr);
    L.relk = H(w.relk);
    L.relv = H(w.relv);
    L.kc = Hm(m->kc) + (size_t)l * Rmax * Tm * d;
    L.vc = Hm(m->vc) + (size_t)l * Rmax * Tm * d;
    L.koff = l * 2 * d;
    L.voff = l * 2 * d + d;
  }
  P->Ld = Ld; P->Tmax = Tm; P->kclip = c.max_rel_pos; P->use_rpr = c.use_rpr;
  P->ldkv = Ld * 2 * d;
  P->eps = c.ln_eps; P->scale = std::sqrt((float)d);
  P->emb = H(m->emb); P->ln0_g = H(m->dec[0].self_g); P->ln0_b = H(m->dec[0].self_b);
  P->lnf_g = H(m->dec_fg); P->lnf_b = H(m->dec_fb); P->pe = m->pe;
  P->g = Hm(m->g); P->u = Hm(m->du); P->qkv = Hm(m->dqkv); P->attn_out = Hm(m->dout); P->q = Hm(m->dq);
  P->row_slot = m->row_slot; P->src_len = m->src_len; P->ckv = H(m->ckv); P->st = m->st;
  P->ctr = m->fused_ctr;
  P->trace = m->fused_trace;
  m->fused = std::move(P);
  return *m->fused;
}

// The decoder of one step (embedding ... final LN into du) through the fused kernel: one
// launch over every phase when the live rows are few (latency-bound step), else fused GEMM
// segments with the standalone attention kernels between them.
template <class T>
void decoder_fused(nmt_model* m, nmt_batch* b, const int* d_prev, cudaStream_t s) {
  const nmt_config& c = m->cfg;
  const int d = c.d_model, H = c.n_heads, Ld = c.dec_layers, F = c.d_ffn;
  const int R = b->rows_upper;
  const int Tm = m->lim.max_tgt_len;
  const int Rmax = m->lim.max_sents * std::max(1, m->lim.beam);
  const int nph = 2 + 8 * Ld;
  FusedParams p = fused_params(m);
  p.ids = d_prev ? d_prev : m->prev_tok;
  p.beam = b->K;
  p.anc = b->K > 1 ? m->anc : nullptr;
  const int* dR = &m->st->n_live;
  const int* dt = &m->st->t;
  const double wbytes = 2.0 * ((double)Ld * (4.0 * d * d + 2.0 * d * F + 3.0 * d * d));
  const double fl = 2.0 * R * ((double)Ld * (6.0 * d * d + 2.0 * d * F));
  auto launch = [&](int p0, int p1, double flops, double bytes) {
    p.pbeg = p0;
    p.pend = p1;
    PROF(P_DEC_FUSED, flops, bytes, decode_fused(p, d / 32, s));
  };
  if (R <= m->fuse_rows) {
    launch(0, nph, fl, wbytes + 8.0 * R * d * 2);
    return;
  }
  int p0 = 0;
  for (int l = 0; l < Ld; ++l) {
    T* kc = (T*)m->kc + (size_t)l * Rmax * Tm * d;
    T* vc = (T*)m->vc + (size_t)l * Rmax * Tm * d;
    const DecW& w = m->dec[l];
    const int a1 = 1 + 8 * l + 1, a2 = 1 + 8 * l + 4;
    launch(p0, a1, 2.0 * R * 3 * d * d, 2.0 * 3 * d * d);
    PROF(P_DEC_SELF, 4.0 * R * (b->step + 1) * d, (2.0 * (b->step + 1) + 6) * R * d * 2,
         attn_decoder_self<T>((const T*)m->dqkv, kc, vc, Tm, m->row_slot, (const T*)w.relk,
                              (const T*)w.relv, (T*)m->dout, R, d, H, c.max_rel_pos, c.use_rpr, dt,
                              dR, b->K > 1 ? m->anc : nullptr, s));
    launch(a1 + 1, a2, 2.0 * R * 2 * d * d, 2.0 * 2 * d * d);
    PROF(P_DEC_CROSS, 4.0 * R * b->S * d, (2.0 * b->S + 2) * R * d * 2,
         attn_cross<T>((const T*)m->dq, (const T*)m->ckv, Ld * 2 * d, l * 2 * d, l * 2 * d + d,
                       &m->st->S, c.max_src_len, m->src_len, m->row_slot, (T*)m->dout, R, d, H,
                       dR, b->K, s));
    p0 = a2 + 1;
  }
  launch(p0, nph, 2.0 * R * (d * d + 2.0 * d * F), 2.0 * (d * d + 2.0 * d * F));
}

template <class T>
void decode_step_impl(nmt_model* m, nmt_batch* b, const int* d_prev, const nmt_step_out* out,
                      cudaStream_t s, bool finish) {
  const nmt_config& c = m->cfg;
  const int d = c.d_model, F = c.d_ffn, H = c.n_heads, Ld = c.dec_layers;
  const int R = b->rows_upper;
  const int Tm = m->lim.max_tgt_len;
  const int Rmax = m->lim.max_sents * std::max(1, m->lim.beam);
  const float eps = c.ln_eps;
  const size_t tb = sizeof(T);
  const int* dR = &m->st->n_live;
  const int* dt = &m->st->t;
  const int t = b->step;  // host mirror (profile byte counts only)
  const double row = (double)R * d * tb;
  T *g = (T*)m->g, *du = (T*)m->du, *dqkv = (T*)m->dqkv, *dout = (T*)m->dout, *dq = (T*)m->dq,
    *dh = (T*)m->dh;
  if (sizeof(T) == 2 && fused_enabled(m)) {
    decoder_fused<T>(m, b, d_prev, s);   // embedding ... final LN -> du (decode_fused.cu)
    goto vocab;
  }
  {
  // g = sqrt(d) E[w_t] + PE(t) fused with the first layer's pre-norm
  PROF(P_EMBED, 0, 3 * row,
       embed_dec_ln<T>(d_prev ? d_prev : m->prev_tok, cT<T>(m->emb), m->pe,
                       cT<T>(m->dec[0].self_g), cT<T>(m->dec[0].self_b), g, du, R, d,
                       std::sqrt((float)d), eps, dt, dR, s));
  // FP16: the LayerNorms in front of GEMMs are folded into them:
  // residual-producing GEMMs emit row-chunk statistics, the consumers run on the raw
  // stream g with W o gamma and apply rstd (acc - mu c) + b' in their epilogue.
  static const bool no_fold = getenv("NMT_NO_FOLD") != nullptr;   // A/B experiments only
  const bool FOLD = sizeof(T) == 2 && !no_fold;
  auto folded = [&](GemmArgs a, const FoldW& f) {
    a.B = f.w; a.bias = f.b;
    a.ln_st = m->lnst; a.ln_c = f.c; a.ln_eps = eps;
    return a;
  };
  for (int l = 0; l < Ld; ++l) {
    const DecW& w = m->dec[l];
    T* kc = (T*)m->kc + (size_t)l * Rmax * Tm * d;
    T* vc = (T*)m->vc + (size_t)l * Rmax * Tm * d;
    GemmArgs a;
    if (FOLD && l > 0) {
      a = folded(mk(R, 3 * d, d, g, d, nullptr, d, nullptr, dqkv, 3 * d), m->fold[l].qkv);
    } else {
      if (l > 0)
        PROF(P_DEC_LN, 0, 2 * row,
             layernorm<T>(g, d, cT<T>(w.self_g), cT<T>(w.self_b), du, d, R, d, eps, dR, s));
      a = mk(R, 3 * d, d, du, d, w.qkv_w, d, w.qkv_b, dqkv, 3 * d);
    }
    a.dM = dR;
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
    PROF(P_DEC_SELF, 4.0 * R * (t + 1) * d, (2.0 * (t + 1) + 6) * row,
         attn_decoder_self<T>(dqkv, kc, vc, Tm, m->row_slot, cT<T>(w.relk), cT<T>(w.relv), dout,
                              R, d, H, c.max_rel_pos, c.use_rpr, dt, dR,
                              b->K > 1 ? m->anc : nullptr, s));
    a = mk(R, d, d, dout, d, w.so_w, d, w.so_b, g, d);
    a.R = g; a.ldr = d; a.dM = dR;
    if (FOLD) a.st_out = m->lnst;
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
    if (FOLD) {
      a = folded(mk(R, d, d, g, d, nullptr, d, nullptr, dq, d), m->fold[l].cq);
    } else {
      PROF(P_DEC_LN, 0, 2 * row,
           layernorm<T>(g, d, cT<T>(w.cross_g), cT<T>(w.cross_b), du, d, R, d, eps, dR, s));
      a = mk(R, d, d, du, d, w.cq_w, d, w.cq_b, dq, d);
    }
    a.dM = dR;
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
    PROF(P_DEC_CROSS, 4.0 * R * b->S * d, (2.0 * b->S + 2) * row,
         attn_cross<T>(dq, (const T*)m->ckv, Ld * 2 * d, l * 2 * d, l * 2 * d + d, &m->st->S,
                       c.max_src_len, m->src_len, m->row_slot, dout, R, d, H, dR, b->K, s));
    a = mk(R, d, d, dout, d, w.co_w, d, w.co_b, g, d);
    a.R = g; a.ldr = d; a.dM = dR;
    if (FOLD) a.st_out = m->lnst;
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
    if (FOLD) {
      a = folded(mk(R, F, d, g, d, nullptr, d, nullptr, dh, F), m->fold[l].w1);
    } else {
      PROF(P_DEC_LN, 0, 2 * row,
           layernorm<T>(g, d, cT<T>(w.ffn_g), cT<T>(w.ffn_b), du, d, R, d, eps, dR, s));
      a = mk(R, F, d, du, d, w.w1, d, w.b1, dh, F);
    }
    a.relu = 1; a.dM = dR;
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
    a = mk(R, d, F, dh, F, w.w2, F, w.b2, g, d);
    a.R = g; a.ldr = d; a.dM = dR;
    if (FOLD && l + 1 < Ld) a.st_out = m->lnst;   // for the next layer's folded QKV
    PROF(P_DEC_GEMM, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(dec_cfg(m, a), s));
  }
  // The final LN stays a kernel: the vocab GEMM's epilogue-bound K = 512 units (V / 256 per
  // row tile) would pay the folded-LN epilogue once per unit (measured +40% vocab time).
  PROF(P_DEC_LN, 0, 2 * row,
       layernorm<T>(g, d, cT<T>(m->dec_fg), cT<T>(m->dec_fb), du, d, R, d, eps, dR, s));
  }
vocab:
  // the tied vocab projection behind the final LN
  auto vocab_args = [&]() {
    GemmArgs v = mk(R, c.vocab_size, d, du, d, m->emb, d, nullptr, nullptr, 0);
    v.dM = dR;
    return v;
  };
  if (b->K == 1) {
    // vocab projection fused with argmax: logits never stored
    GemmArgs a = vocab_args();
    a.argmax = m->keys; a.logits = out ? out->d_logits : nullptr;
    PROF(P_VOCAB, gemm_flops(a), gemm_bytes(a, tb), gemm<T>(a, s));
    if (finish) {
      PROF(P_BOOK, 0, 0,
           greedy_finish(m->keys, nullptr, m->prev_tok, m->done, m->row_slot, m->tgt_cap,
                         m->out_tok, Tm, m->gen_len, m->st, R, c.eos_id,
                         out ? out->d_next : nullptr, out ? out->d_done : nullptr, s));
      if (out && out->d_parent)
        step_outputs(m->st, m->prev_tok, nullptr, m->done, nullptr, nullptr, nullptr, R, s,
                     out->d_parent);
    }
    return;
  }
  // beam
  const int K = b->K, V = c.vocab_size;
  GemmArgs a = vocab_args();
  if (sizeof(T) == 2 && finish && !(out && out->d_logits) && m->beam_epi) {
    // FP16: the vocab GEMM epilogue keeps per (row, 256-column segment) the log-sum-exp
    // partial and the top-8 candidates — the R x V logits are never written (SURVEY §2.6
    // K17) — and one warp per row merges them into the LSE and the top-2K log-probs
    const int nseg = (V + 255) / 256;   // one segment per 256-column unit (gemm_tc.cu)
    a.beam_part = m->bpart;
    PROF(P_VOCAB, gemm_flops(a), gemm_bytes(a, tb) - (double)R * V * tb + (double)R * nseg * 72,
         gemm<T>(a, s));
    PROF(P_BOOK, 0, (double)R * nseg * 72,
         beam_merge(m->bpart, nseg, 2 * K, dR, R, m->cand_v, m->cand_i, s));
  } else {
    // FP32 logits -> per-row LSE + top-2K (FP32 mode, logits dumps, and the ensemble's
    // members, whose distributions are averaged before the top-2K)
    a.logits = m->blogits;
    PROF(P_VOCAB, gemm_flops(a), gemm_bytes(a, tb) + (double)R * V * 4, gemm<T>(a, s));
    if (out && out->d_logits)
      NMT_CUDA(cudaMemcpyAsync(out->d_logits, m->blogits, (size_t)R * V * 4,
                               cudaMemcpyDeviceToDevice, s));
    if (!finish) return;
    PROF(P_BOOK, 0, (double)R * V * 4,
         beam_row_topk(m->blogits, V, 2 * K, dR, R, m->cand_v, m->cand_i, s));
  }
  PROF(P_BOOK, 0, 0,
       beam_select(K, m->cand_v, m->cand_i, m->bscore, m->prev_tok, m->done, m->row_slot,
                   m->tgt_cap, m->anc, m->htok, Tm, m->best_score, m->out_tok, m->gen_len, m->st,
                   V, c.eos_id, R, s, b->NB, m->nb_score, m->nb_len, m->nb_tok, m->nb_cnt,
                   out ? out->d_parent : nullptr));
  if (out)   // step-drivable beam (nmt_step_out): next tokens, cumulative scores, done flags
    step_outputs(m->st, m->prev_tok, m->bscore, m->done, out->d_next, out->d_score, out->d_done,
                 R, s);
}

}  // namespace

void encode_any(nmt_model* m, int B, int S, cudaStream_t s) {
  if (m->prec == NMT_FP16) encode_impl<__half>(m, B, S, s);
  else encode_impl<float>(m, B, S, s);
}

void decode_step_any(nmt_model* m, nmt_batch* b, const int* d_prev, const nmt_step_out* out,
                     cudaStream_t s, bool finish) {
  if (m->prec == NMT_FP16) decode_step_impl<__half>(m, b, d_prev, out, s, finish);
  else decode_step_impl<float>(m, b, d_prev, out, s, finish);
}

}  // namespace nmt
