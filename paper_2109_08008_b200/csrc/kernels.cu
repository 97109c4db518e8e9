// kernels.cu — bandwidth-/latency-bound kernels of the hot path (sm_100a).
// Embedding, LayerNorm, DLCL combine, RPR attention (encoder / cached decoder),
// cross-attention, greedy bookkeeping, batch-pruning compaction.
// All reductions (LN statistics, softmax, DLCL sums) run in FP32.
#include "common.cuh"
#include "kernels.h"
#include "rowops.cuh"

namespace nmt {

constexpr int kMaxLaneElems = 16;  // d <= 512 with one warp per row

// ------------------------------------------------------------------- embedding
template <class T>
__global__ void k_embed(const int* __restrict__ ids, const T* __restrict__ E,
                        const float* __restrict__ pe, T* __restrict__ out, int rows, int d, int S,
                        const int* __restrict__ d_t, const int* __restrict__ dR, float scale) {
  int r = blockIdx.x;
  if (dR && r >= *dR) return;
  if (r >= rows) return;
  int pos = d_t ? *d_t : (r % S);
  int id = ids[r];
  const T* e = E + (size_t)id * d;
  const float* p = pe + (size_t)pos * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    out[(size_t)r * d + c] = from_f<T>(to_f(e[c]) * scale + p[c]);
}

template <class T>
void embed(const int* ids, const T* E, const float* pe, T* out, int rows, int d, int S,
           const int* d_t, const int* dR, float scale, cudaStream_t s) {
  if (rows <= 0) return;
  k_embed<T><<<rows, 128, 0, s>>>(ids, E, pe, out, rows, d, S, d_t, dR, scale);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- layer norm
// Warp per row; lane owns columns c = lane + 32 i (coalesced).  Two-pass FP32 stats.
template <class T>
__device__ __forceinline__ void ln_regs(float* v, int E, int d, const T* g, const T* b, float eps,
                                        int lane) {
  float s = 0.f;
  for (int i = 0; i < E; ++i) s += v[i];
  float mu = warp_sum(s) / d;
  float q = 0.f;
  for (int i = 0; i < E; ++i) { float t = v[i] - mu; q += t * t; }
  float rstd = rsqrtf(warp_sum(q) / d + eps);
  for (int i = 0; i < E; ++i) {
    int c = lane + 32 * i;
    v[i] = (v[i] - mu) * rstd * to_f(g[c]) + to_f(b[c]);
  }
}

template <class T>
__global__ void k_layernorm(const T* __restrict__ in, int ldi, const T* __restrict__ g,
                            const T* __restrict__ b, T* __restrict__ out, int ldo, int rows, int d,
                            float eps, const int* __restrict__ dR) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nrows = dR ? min(rows, *dR) : rows;
  if (warp >= nrows) return;
  const int E = d >> 5;
  float v[kMaxLaneElems];
  const T* x = in + (size_t)warp * ldi;
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) v[i] = to_f(x[lane + 32 * i]);
  ln_regs(v, E, d, g, b, eps, lane);
  T* y = out + (size_t)warp * ldo;
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) y[lane + 32 * i] = from_f<T>(v[i]);
}

template <class T>
bool layernorm_vec(const T* in, int ldi, const T* g, const T* b, T* out, int ldo, int rows, int d,
                   float eps, const int* dR, cudaStream_t s);

template <class T>
void layernorm(const T* in, int ldi, const T* g, const T* b, T* out, int ldo, int rows, int d,
               float eps, const int* dR, cudaStream_t s) {
  if (rows <= 0) return;
  if (layernorm_vec<T>(in, ldi, g, b, out, ldo, rows, d, eps, dR, s)) return;  // d = 256 / 512
  k_layernorm<T><<<ceil_div(rows, 8), 256, 0, s>>>(in, ldi, g, b, out, ldo, rows, d, eps, dR);
  NMT_LAUNCH_CHECK();
}

template <class T>
__global__ void k_embed_dec_ln(const int* __restrict__ ids, const T* __restrict__ E,
                               const float* __restrict__ pe, const T* __restrict__ gam,
                               const T* __restrict__ bet, T* __restrict__ g, T* __restrict__ u,
                               int rows, int d, float scale, float eps, const int* __restrict__ d_t,
                               const int* __restrict__ dR) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= min(rows, *dR)) return;
  const int E_ = d >> 5;
  const T* e = E + (size_t)ids[row] * d;
  const float* p = pe + (size_t)(*d_t) * d;
  float v[kMaxLaneElems];
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E_) {
      const int c = lane + 32 * i;
      const T gt = from_f<T>(to_f(e[c]) * scale + p[c]);
      g[(size_t)row * d + c] = gt;
      v[i] = to_f(gt);
    }
  ln_regs(v, E_, d, gam, bet, eps, lane);
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E_) u[(size_t)row * d + lane + 32 * i] = from_f<T>(v[i]);
}

template <class T>
bool embed_dec_ln_vec(const int* ids, const T* E, const float* pe, const T* gam, const T* bet, T* g,
                      T* u, int rows, int d, float scale, float eps, const int* d_t, const int* dR,
                      cudaStream_t s);

template <class T>
void embed_dec_ln(const int* ids, const T* E, const float* pe, const T* gam, const T* bet, T* g,
                  T* u, int rows, int d, float scale, float eps, const int* d_t, const int* dR,
                  cudaStream_t s) {
  if (rows <= 0) return;
  if (embed_dec_ln_vec<T>(ids, E, pe, gam, bet, g, u, rows, d, scale, eps, d_t, dR, s)) return;
  k_embed_dec_ln<T><<<ceil_div(rows, 8), 256, 0, s>>>(ids, E, pe, gam, bet, g, u, rows, d, scale,
                                                      eps, d_t, dR);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- DLCL combine
// Eq. 2: x_{l+1} = sum_{k=0..l} W^{(l+1)}_k LN(y_k).  z_k = LN^dl_k(y_k)
// is written once into the history when y_k is produced and re-read by every later
// combine (reading A2).
template <class T>
__global__ void k_dlcl(const T* __restrict__ y, T* __restrict__ hist, size_t hist_stride, int l,
                       const float* __restrict__ w, const T* __restrict__ gdl,
                       const T* __restrict__ bdl, int dlcl_ln, const T* __restrict__ g2,
                       const T* __restrict__ b2, T* __restrict__ xout, T* __restrict__ uout,
                       int rows, int d, float eps) {
  int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int E = d >> 5;
  float z[kMaxLaneElems], x[kMaxLaneElems];
  const T* yr = y + (size_t)row * d;
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) z[i] = to_f(yr[lane + 32 * i]);
  if (dlcl_ln) ln_regs(z, E, d, gdl, bdl, eps, lane);
  T* hl = hist + (size_t)l * hist_stride + (size_t)row * d;
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) {
      T zt = from_f<T>(z[i]);
      hl[lane + 32 * i] = zt;
      x[i] = 0.f;
      z[i] = to_f(zt);
    }
  for (int k = 0; k < l; ++k) {
    const float wk = w[k];
    const T* hk = hist + (size_t)k * hist_stride + (size_t)row * d;
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i)
      if (i < E) x[i] += wk * to_f(hk[lane + 32 * i]);
  }
  const float wl = w[l];
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) x[i] += wl * z[i];
  if (xout) {
    T* xr = xout + (size_t)row * d;
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i)
      if (i < E) xr[lane + 32 * i] = from_f<T>(x[i]);
  }
  ln_regs(x, E, d, g2, b2, eps, lane);
  T* ur = uout + (size_t)row * d;
#pragma unroll
  for (int i = 0; i < kMaxLaneElems; ++i)
    if (i < E) ur[lane + 32 * i] = from_f<T>(x[i]);
}

template <class T>
void dlcl_combine(const T* y, T* hist, size_t hist_stride, int l, const float* w, const T* gdl,
                  const T* bdl, int dlcl_ln, const T* g2, const T* b2, T* xout, T* uout, int rows,
                  int d, float eps, cudaStream_t s, int mode, const float* wP, float* P);

// MODE (m-boundary lookahead): boundaries are taken in blocks of
// m; the block's first boundary l reads every history row once and also accumulates, from
// the same rows, the FP32 partials of the block's later combinations (their weight rows
// l + 1 + i are known), so the later boundaries read one partial plus the few history rows
// written since the block started instead of l + 1 rows:
//   MODE 0: x = sum_{k<=l} w[k] z_k                                 (every history row read)
//   MODE 1: as 0, and P_i = sum_{k<=l} W^(l+1+i)[k] z_k -> FP32 partial i, i = 1..NP
//   MODE 2: x = P + sum_{k=l-nx}^{l-1} w[k] z_k + w[l] z_l           (P: this boundary's partial)
// The FP32 sums run in the same k order in every mode, so x is bit-identical to MODE 0.
template <class T, int E, int MODE, int NP>
__global__ void __launch_bounds__(256) k_dlcl_vec(
    const T* __restrict__ y, T* __restrict__ hist, size_t hist_stride, int l,
    const float* __restrict__ w, const T* __restrict__ gdl, const T* __restrict__ bdl, int dlcl_ln,
    const T* __restrict__ g2, const T* __restrict__ b2, T* __restrict__ xout, T* __restrict__ uout,
    int rows, float eps, const float* __restrict__ wall, float* __restrict__ P, int nx) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  constexpr int d = 32 * E;
  constexpr int NPA = MODE == 1 ? NP : 1;
  const size_t off = (size_t)row * d + lane * E;
  const size_t pstride = (size_t)rows * d;   // partial i at P + (i - 1) * rows * d
  float z[E], x[E], pa[NPA][E];
  const float* wp[NPA];
  if constexpr (MODE == 1) {
#pragma unroll
    for (int i = 0; i < NP; ++i) wp[i] = wall + (size_t)(l + 2 + i) * (l + 1 + i) / 2;   // row l+1+(i+1)
  }
  if constexpr (MODE == 2) {   // the partial, issued before the y row's LN
#pragma unroll
    for (int i = 0; i < E; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(P + off + i);
      x[i] = q.x; x[i + 1] = q.y; x[i + 2] = q.z; x[i + 3] = q.w;
    }
  }
  ldrow<T, E>(y + off, z);
  if (dlcl_ln) ln_contig<T, E>(z, d, gdl, bdl, eps, lane);
  // z_l rounded to storage precision: later combines re-read exactly this value
  strow<T, E>(hist + (size_t)l * hist_stride + off, z);
#pragma unroll
  for (int i = 0; i < E; ++i) z[i] = to_f(from_f<T>(z[i]));
  if constexpr (MODE != 2) {
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = 0.f;
    if constexpr (MODE == 1) {
#pragma unroll
      for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int i = 0; i < E; ++i) pa[q][i] = 0.f;
    }
    // U history rows in flight per lane (raw 16-B loads issued before any arithmetic): the
    // combine is bound by HBM bandwidth, not by one memory latency per history row
    constexpr int U = sizeof(T) == 2 ? (NP >= 2 && MODE == 1 ? 4 : 8) : 4;
    int k = 0;
    for (; k + U <= l; k += U) {
      RawRow<T, E> a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].load(hist + (size_t)(k + u) * hist_stride + off);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u].fma_into(w[k + u], x);
        if constexpr (MODE == 1) {
#pragma unroll
          for (int q = 0; q < NP; ++q) a[u].fma_into(wp[q][k + u], pa[q]);
        }
      }
    }
    for (; k < l; ++k) {
      float a[E];
      ldrow<T, E>(hist + (size_t)k * hist_stride + off, a);
      const float wa = w[k];
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = fmaf(wa, a[i], x[i]);
      if constexpr (MODE == 1) {
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const float wb = wp[q][k];
#pragma unroll
          for (int i = 0; i < E; ++i) pa[q][i] = fmaf(wb, a[i], pa[q][i]);
        }
      }
    }
    if constexpr (MODE == 1) {
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const float wb = wp[q][l];
#pragma unroll
        for (int i = 0; i < E; i += 4) {
          float4 o;
          o.x = fmaf(wb, z[i], pa[q][i]); o.y = fmaf(wb, z[i + 1], pa[q][i + 1]);
          o.z = fmaf(wb, z[i + 2], pa[q][i + 2]); o.w = fmaf(wb, z[i + 3], pa[q][i + 3]);
          *reinterpret_cast<float4*>(P + q * pstride + off + i) = o;
        }
      }
    }
  } else {
    // the rows written since the block's partial was formed (k = l - nx .. l - 1, nx <= 2),
    // all loads in flight before the in-order FMAs
    RawRow<T, E> a[2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (u < nx) a[u].load(hist + (size_t)(l - nx + u) * hist_stride + off);
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (u < nx) a[u].fma_into(w[l - nx + u], x);
  }
  const float wl = w[l];
#pragma unroll
  for (int i = 0; i < E; ++i) x[i] = fmaf(wl, z[i], x[i]);
  if (xout) strow<T, E>(xout + off, x);
  ln_contig<T, E>(x, d, g2, b2, eps, lane);
  strow<T, E>(uout + off, x);
}

bool dlcl_lookahead_ok(int d) { return d == 512 || d == 256; }

template <class T>
void dlcl_combine(const T* y, T* hist, size_t hist_stride, int l, const float* w, const T* gdl,
                  const T* bdl, int dlcl_ln, const T* g2, const T* b2, T* xout, T* uout, int rows,
                  int d, float eps, cudaStream_t s, int mode, const float* wall, float* P, int arg) {
  if (rows <= 0) return;
  if (mode != 0 && !dlcl_lookahead_ok(d)) throw CudaError("dlcl_combine: lookahead needs d = 256 / 512");
  if ((mode == 1 && (arg < 1 || arg > 3)) || (mode == 2 && (arg < 0 || arg > 2)))
    throw CudaError("dlcl_combine: 1..3 partials, 0..2 extra rows");
#define NMT_DV(E, MODE, NP)                                                                     \
  k_dlcl_vec<T, E, MODE, NP><<<ceil_div(rows, 8), 256, 0, s>>>(y, hist, hist_stride, l, w, gdl,   \
                                                               bdl, dlcl_ln, g2, b2, xout, uout, \
                                                               rows, eps, wall, P, arg)
#define NMT_DVE(E)                                       \
  if (mode == 1 && arg == 1) NMT_DV(E, 1, 1);            \
  else if (mode == 1 && arg == 2) NMT_DV(E, 1, 2);       \
  else if (mode == 1) NMT_DV(E, 1, 3);                   \
  else if (mode == 2) NMT_DV(E, 2, 1);                   \
  else NMT_DV(E, 0, 1);
  if (d == 512) {
    NMT_DVE(16)
  } else if (d == 256) {
    NMT_DVE(8)
  } else {
    k_dlcl<T><<<ceil_div(rows, 8), 256, 0, s>>>(y, hist, hist_stride, l, w, gdl, bdl, dlcl_ln, g2,
                                                 b2, xout, uout, rows, d, eps);
  }
#undef NMT_DVE
#undef NMT_DV
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- vectorised row kernels
// One warp per row, lane owns E contiguous columns: 16-B loads/stores (d = 32*E).
template <class T, int E>
__global__ void __launch_bounds__(256) k_layernorm_vec(const T* __restrict__ in, int ldi,
                                                       const T* __restrict__ g,
                                                       const T* __restrict__ b,
                                                       T* __restrict__ out, int ldo, int rows,
                                                       float eps, const int* __restrict__ dR) {
  pdl_trigger();
  pdl_wait();
  // grid-stride over rows with the next row's load issued before this row's reductions (a
  // bounded grid instead of one short-lived warp per row)
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nrows = dR ? min(rows, *dR) : rows;
  if (row >= nrows) return;
  float v[E], nx[E];
  ldrow<T, E>(in + (size_t)row * ldi + lane * E, v);
  for (;;) {
    const int nr = row + nw;
    if (nr < nrows) ldrow<T, E>(in + (size_t)nr * ldi + lane * E, nx);
    ln_contig<T, E>(v, 32 * E, g, b, eps, lane);
    strow<T, E>(out + (size_t)row * ldo + lane * E, v);
    if (nr >= nrows) break;
    row = nr;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = nx[i];
  }
}

template <class T>
bool layernorm_vec(const T* in, int ldi, const T* g, const T* b, T* out, int ldo, int rows, int d,
                   float eps, const int* dR, cudaStream_t s) {
  const bool al = (ldi % 8 == 0) && (ldo % 8 == 0);
  static const int cap = [] {   // one wave of resident 256-thread CTAs
    int dev = 0, sms = 0, occ16 = 0;
    NMT_CUDA(cudaGetDevice(&dev));
    NMT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    NMT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ16, k_layernorm_vec<T, 16>, 256, 0));
    return std::max(1, occ16) * sms;
  }();
  const int grid = std::min(ceil_div(rows, 8), cap);
  if (d == 512 && al)
    launch_k(k_layernorm_vec<T, 16>, grid, 256, 0, s, in, ldi, g, b, out, ldo, rows, eps, dR);
  else if (d == 256 && al)
    launch_k(k_layernorm_vec<T, 8>, grid, 256, 0, s, in, ldi, g, b, out, ldo, rows, eps, dR);
  else
    return false;
  NMT_LAUNCH_CHECK();
  return true;
}

template <class T, int E>
__global__ void __launch_bounds__(256) k_embed_dec_ln_vec(
    const int* __restrict__ ids, const T* __restrict__ Em, const float* __restrict__ pe,
    const T* __restrict__ gam, const T* __restrict__ bet, T* __restrict__ g, T* __restrict__ u,
    int rows, float scale, float eps, const int* __restrict__ d_t, const int* __restrict__ dR) {
  pdl_trigger();
  pdl_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= min(rows, *dR)) return;
  constexpr int d = 32 * E;
  float v[E];
  ldrow<T, E>(Em + (size_t)ids[row] * d + lane * E, v);
  const float* p = pe + (size_t)(*d_t) * d + lane * E;
#pragma unroll
  for (int i = 0; i < E; i += 4) {
    const float4 q = *reinterpret_cast<const float4*>(p + i);
    v[i] = to_f(from_f<T>(v[i] * scale + q.x));
    v[i + 1] = to_f(from_f<T>(v[i + 1] * scale + q.y));
    v[i + 2] = to_f(from_f<T>(v[i + 2] * scale + q.z));
    v[i + 3] = to_f(from_f<T>(v[i + 3] * scale + q.w));
  }
  strow<T, E>(g + (size_t)row * d + lane * E, v);   // g (residual stream) in storage precision
  ln_contig<T, E>(v, d, gam, bet, eps, lane);
  strow<T, E>(u + (size_t)row * d + lane * E, v);
}

template <class T>
bool embed_dec_ln_vec(const int* ids, const T* E, const float* pe, const T* gam, const T* bet, T* g,
                      T* u, int rows, int d, float scale, float eps, const int* d_t, const int* dR,
                      cudaStream_t s) {
  if (d == 512)
    launch_k(k_embed_dec_ln_vec<T, 16>, ceil_div(rows, 8), 256, 0, s, ids, E, pe, gam, bet, g, u,
             rows, scale, eps, d_t, dR);
  else if (d == 256)
    launch_k(k_embed_dec_ln_vec<T, 8>, ceil_div(rows, 8), 256, 0, s, ids, E, pe, gam, bet, g, u,
             rows, scale, eps, d_t, dR);
  else
    return false;
  NMT_LAUNCH_CHECK();
  return true;
}

// ------------------------------------------------------------------- greedy bookkeeping
__global__ void k_greedy_finish(unsigned long long* __restrict__ keys, int* __restrict__ prev_tok,
                                uint8_t* __restrict__ done, const int* __restrict__ row_slot,
                                const int* __restrict__ cap, int* __restrict__ out_tok,
                                int out_stride, int* __restrict__ gen_len, DevState* st, int eos,
                                int* __restrict__ d_next, uint8_t* __restrict__ d_done) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= st->n_live) return;
  const int t = st->t;
  unsigned long long k = keys[r];
  keys[r] = 0ull;
  const int tok = unpack_argmax_id(k);
  prev_tok[r] = tok;
  if (!done[r]) {
    const int slot = row_slot[r];
    out_tok[(size_t)slot * out_stride + t] = tok;
    gen_len[slot] = t + 1;
    if (tok == eos || t + 1 >= cap[slot]) {
      done[r] = 1;
      atomicAdd(&st->n_done, 1);
    }
  }
  if (d_next) d_next[r] = tok;
  if (d_done) d_done[r] = done[r];
}

void greedy_finish(unsigned long long* keys, const int* /*force_next*/, int* prev_tok,
                   uint8_t* done, const int* row_slot, const int* cap, int* out_tok,
                   int out_stride, int* gen_len, DevState* st, int rows_upper, int eos,
                   int* d_next_copy, uint8_t* d_done_copy, cudaStream_t s) {
  if (rows_upper <= 0) return;
  k_greedy_finish<<<ceil_div(rows_upper, 128), 128, 0, s>>>(keys, prev_tok, done, row_slot, cap,
                                                            out_tok, out_stride, gen_len, st, eos,
                                                            d_next_copy, d_done_copy);
  NMT_LAUNCH_CHECK();
}

// Block-wide exclusive scan of one int per thread (blockDim.x == 1024).
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_tot[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = warp_tot[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    warp_tot[lane] = wi - w;  // exclusive prefix of warp totals
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  return warp_tot[warp] + incl - v;
}

constexpr int kPrunePer = 16;                   // rows per thread held in registers
constexpr int kPruneMaxRows = 1024 * kPrunePer;  // 16384

__device__ void prune_body(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, int every,
                           float ratio, int* new_to_old, float* score);

__global__ void __launch_bounds__(1024) k_prune(DevState* st, int* row_slot, int* prev_tok,
                                                uint8_t* done, int every, float ratio,
                                                int* new_to_old, float* score) {
  pdl_wait();
  prune_body(st, row_slot, prev_tok, done, every, ratio, new_to_old, score);
}

// Greedy finish (k_greedy_finish) + pruning decision/compaction (k_prune) in one CTA: the
// decode step's bookkeeping tail as a single launch.
__global__ void __launch_bounds__(1024) k_finish_prune(
    unsigned long long* __restrict__ keys, int* __restrict__ prev_tok, uint8_t* __restrict__ done,
    int* __restrict__ row_slot, const int* __restrict__ cap, int* __restrict__ out_tok,
    int out_stride, int* __restrict__ gen_len, DevState* st, int eos, int every, float ratio) {
  pdl_wait();
  __shared__ int s_new;
  if (threadIdx.x == 0) s_new = 0;
  __syncthreads();
  const int n = st->n_live, t = st->t;
  int cnt = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const unsigned long long k = keys[r];
    keys[r] = 0ull;
    const int tok = unpack_argmax_id(k);
    prev_tok[r] = tok;
    if (!done[r]) {
      const int slot = row_slot[r];
      out_tok[(size_t)slot * out_stride + t] = tok;
      gen_len[slot] = t + 1;
      if (tok == eos || t + 1 >= cap[slot]) {
        done[r] = 1;
        ++cnt;
      }
    }
  }
  cnt = (int)warp_sum((float)cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_new, cnt);
  __syncthreads();
  if (threadIdx.x == 0) st->n_done += s_new;
  __syncthreads();
  prune_body(st, row_slot, prev_tok, done, every, ratio, nullptr, nullptr);
}

void finish_prune(unsigned long long* keys, int* prev_tok, uint8_t* done, int* row_slot,
                  const int* cap, int* out_tok, int out_stride, int* gen_len, DevState* st,
                  int eos, int every, float ratio, int rows_upper, cudaStream_t s) {
  if (rows_upper > kPruneMaxRows) throw CudaError("finish_prune: too many rows");
  launch_k(k_finish_prune, 1, 1024, 0, s, keys, prev_tok, done, row_slot, cap, out_tok, out_stride,
           gen_len, st, eos, every, ratio);
  NMT_LAUNCH_CHECK();
}

__device__ void prune_body(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, int every,
                           float ratio, int* new_to_old, float* score) {
  __shared__ int s_total;
  const int n = st->n_live, nd = st->n_done, t = st->t;
  bool all_done = (n > 0 && nd == n);
  bool decide = false;
  if (ratio >= 0.f && (t + 1) % every == 0 && n > 0) {
    int need = (int)ceilf(ratio * (float)n);
    need = need < 1 ? 1 : need;
    decide = nd >= need;
  }
  const bool compact = all_done || decide;
  if (!compact) {
    if (new_to_old)
      for (int i = threadIdx.x; i < n; i += blockDim.x) new_to_old[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) st->t = t + 1;
    return;
  }
  // each thread owns a contiguous chunk of <= kPrunePer rows, read into registers before
  // the scan's barrier so the stable in-place compaction cannot overwrite unread rows
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  int r_slot[kPrunePer], r_tok[kPrunePer];
  float r_sc[kPrunePer];
  unsigned keepmask = 0;
  int keep = 0;
#pragma unroll
  for (int k = 0; k < kPrunePer; ++k) {
    const int i = lo + k;
    if (i < hi) {
      r_slot[k] = row_slot[i];
      r_tok[k] = prev_tok[i];
      r_sc[k] = score ? score[i] : 0.f;
      if (!done[i]) {
        keepmask |= 1u << k;
        ++keep;
      }
    }
  }
  int base = block_excl_scan(keep, &s_total);
  __syncthreads();
  int o = base;
#pragma unroll
  for (int k = 0; k < kPrunePer; ++k) {
    if (keepmask & (1u << k)) {
      row_slot[o] = r_slot[k];
      prev_tok[o] = r_tok[k];
      if (score) score[o] = r_sc[k];
      if (new_to_old) new_to_old[o] = lo + k;
      ++o;
    }
  }
  __syncthreads();
  const int nn = s_total;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i < nn) done[i] = 0;
    else if (new_to_old) new_to_old[i] = -1;
  }
  if (threadIdx.x == 0) {
    st->n_live = nn;
    st->n_done = 0;
    if (!all_done) st->prunes += 1;
    st->t = t + 1;
  }
}

void prune_compact(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, int every,
                   float ratio, int* new_to_old, int rows_upper, cudaStream_t s, float* score) {
  if (rows_upper > kPruneMaxRows) throw CudaError("prune_compact: too many rows");
  launch_k(k_prune, 1, 1024, 0, s, st, row_slot, prev_tok, done, every, ratio, new_to_old, score);
  NMT_LAUNCH_CHECK();
}

// Caller-driven pruning (nmt_prune_batch with d_keep, greedy): rows with keep[r] == 0 leave
// the live batch, the others stay in order with their sticky done flags.
__global__ void __launch_bounds__(1024) k_prune_keep(DevState* st, int* row_slot, int* prev_tok,
                                                     uint8_t* done, const uint8_t* keep,
                                                     int* new_to_old) {
  __shared__ int s_total, s_done;
  const int n = st->n_live, t = st->t;
  if (threadIdx.x == 0) s_done = 0;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  int r_slot[kPrunePer], r_tok[kPrunePer];
  unsigned keepmask = 0, donemask = 0;
  int kept = 0, kdone = 0;
#pragma unroll
  for (int k = 0; k < kPrunePer; ++k) {
    const int i = lo + k;
    if (i < hi) {
      r_slot[k] = row_slot[i];
      r_tok[k] = prev_tok[i];
      if (keep[i]) {
        keepmask |= 1u << k;
        ++kept;
        if (done[i]) { donemask |= 1u << k; ++kdone; }
      }
    }
  }
  const int base = block_excl_scan(kept, &s_total);
  if (kdone) atomicAdd(&s_done, kdone);
  __syncthreads();
  int o = base;
#pragma unroll
  for (int k = 0; k < kPrunePer; ++k) {
    if (keepmask & (1u << k)) {
      row_slot[o] = r_slot[k];
      prev_tok[o] = r_tok[k];
      done[o] = (donemask >> k) & 1u;
      if (new_to_old) new_to_old[o] = lo + k;
      ++o;
    }
  }
  __syncthreads();
  const int nn = s_total;
  if (new_to_old)
    for (int i = nn + threadIdx.x; i < n; i += blockDim.x) new_to_old[i] = -1;
  if (threadIdx.x == 0) {
    if (nn < n) st->prunes += 1;
    st->n_live = nn;
    st->n_done = s_done;
    st->t = t + 1;
  }
}

void prune_keep(DevState* st, int* row_slot, int* prev_tok, uint8_t* done, const uint8_t* keep,
                int* new_to_old, int rows_upper, cudaStream_t s) {
  if (rows_upper > kPruneMaxRows) throw CudaError("prune_keep: too many rows");
  k_prune_keep<<<1, 1024, 0, s>>>(st, row_slot, prev_tok, done, keep, new_to_old);
  NMT_LAUNCH_CHECK();
}

// Per-row step outputs of a beam step (nmt_step_out): next token, cumulative score, done.
__global__ void k_step_outputs(const DevState* st, const int* prev_tok, const float* score,
                               const uint8_t* done, int* d_next, float* d_score,
                               uint8_t* d_done, int* d_parent_id) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= st->n_live) return;
  if (d_next) d_next[r] = prev_tok[r];
  if (d_score) d_score[r] = score[r];
  if (d_done) d_done[r] = done[r];
  if (d_parent_id) d_parent_id[r] = r;
}

void step_outputs(const DevState* st, const int* prev_tok, const float* score, const uint8_t* done,
                  int* d_next, float* d_score, uint8_t* d_done, int rows_upper, cudaStream_t s,
                  int* d_parent_identity) {
  if (rows_upper <= 0 || (!d_next && !d_score && !d_done && !d_parent_identity)) return;
  k_step_outputs<<<ceil_div(rows_upper, 128), 128, 0, s>>>(st, prev_tok, score, done, d_next,
                                                           d_score, d_done, d_parent_identity);
  NMT_LAUNCH_CHECK();
}

__global__ void k_batch_init(int* row_slot, int* prev_tok, uint8_t* done, int* gen_len,
                             DevState* st, int B, int S, int bos) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < B) {
    row_slot[r] = r;
    prev_tok[r] = bos;
    done[r] = 0;
    gen_len[r] = 0;
  }
  if (r == 0) {
    st->t = 0;
    st->n_live = B;
    st->n_done = 0;
    st->prunes = 0;
    st->S = S;
  }
}

void batch_init(int* row_slot, int* prev_tok, uint8_t* done, int* gen_len, DevState* st, int B,
                int S, int bos, cudaStream_t s) {
  k_batch_init<<<ceil_div(B > 0 ? B : 1, 128), 128, 0, s>>>(row_slot, prev_tok, done, gen_len, st,
                                                            B, S, bos);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- batch I/O
__global__ void k_scatter(const int* __restrict__ out_tok, int out_stride,
                          const int* __restrict__ gen_len, const int* __restrict__ sent_ids,
                          int* __restrict__ d_out, int d_out_stride, int* __restrict__ d_out_len) {
  const int b = blockIdx.x;
  const int sid = sent_ids[b], n = gen_len[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    d_out[(size_t)sid * d_out_stride + j] = out_tok[(size_t)b * out_stride + j];
  if (threadIdx.x == 0) d_out_len[sid] = n;
}

void scatter_outputs(const int* out_tok, int out_stride, const int* gen_len, const int* sent_ids,
                     int B, int* d_out, int d_out_stride, int* d_out_len, cudaStream_t s) {
  if (B <= 0) return;
  k_scatter<<<B, 64, 0, s>>>(out_tok, out_stride, gen_len, sent_ids, d_out, d_out_stride,
                             d_out_len);
  NMT_LAUNCH_CHECK();
}

__global__ void k_pack(const int* __restrict__ ids, const long long* __restrict__ boff,
                       const int* __restrict__ blen, int S, int* __restrict__ out, int vocab,
                       int* bad, int eos) {
  const int b = blockIdx.x;
  const long long o = boff[b];
  const int nb = blen[b];
  const bool cut = nb < 0;            // truncated source: keep |blen| - 1 ids, then EOS
  const int n = cut ? -nb : nb;
  for (int p = threadIdx.x; p < S; p += blockDim.x) {
    int v = p < n ? ((cut && p == n - 1) ? eos : ids[o + p]) : 0;
    if (v < 0 || v >= vocab) {
      atomicOr(bad, 1);
      v = 0;
    }
    out[(size_t)b * S + p] = v;
  }
}

void pack_sources(const int* ids, const long long* boff, const int* blen, int B, int S, int* out,
                  int vocab, int* bad, int eos, cudaStream_t s) {
  if (B <= 0) return;
  k_pack<<<B, 128, 0, s>>>(ids, boff, blen, S, out, vocab, bad, eos);
  NMT_LAUNCH_CHECK();
}

template <class T>
__global__ void k_to_float(const T* __restrict__ in, float* __restrict__ out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = to_f(in[i]);
}
template <class T> void to_float(const T* in, float* out, size_t n, cudaStream_t s) {
  if (!n) return;
  k_to_float<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n);
  NMT_LAUNCH_CHECK();
}

__global__ void k_argmax_ids(unsigned long long* keys, int* ids, int rows) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) {
    ids[r] = unpack_argmax_id(keys[r]);
    keys[r] = 0ull;
  }
}
void argmax_ids(unsigned long long* keys, int* ids, int rows, cudaStream_t s) {
  if (rows <= 0) return;
  k_argmax_ids<<<ceil_div(rows, 128), 128, 0, s>>>(keys, ids, rows);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- instantiations
#define NMT_INST(T)                                                                             \
  template void embed<T>(const int*, const T*, const float*, T*, int, int, int, const int*,     \
                         const int*, float, cudaStream_t);                                      \
  template void layernorm<T>(const T*, int, const T*, const T*, T*, int, int, int, float,       \
                             const int*, cudaStream_t);                                         \
  template void dlcl_combine<T>(const T*, T*, size_t, int, const float*, const T*, const T*,    \
                                int, const T*, const T*, T*, T*, int, int, float, cudaStream_t, \
                                int, const float*, float*, int);                                \
  template void to_float<T>(const T*, float*, size_t, cudaStream_t);                          \
  template void embed_dec_ln<T>(const int*, const T*, const float*, const T*, const T*, T*, T*, \
                                int, int, float, float, const int*, const int*, cudaStream_t);
NMT_INST(float)
NMT_INST(__half)

// ------------------------------------------------------------------- LN folding (load time)
// For y = LN(x) W^T + b with LN(x)_k = (x_k - mu) rstd g_k + beta_k:
//   y_n = rstd (sum_k x_k W'_nk - mu c_n) + b'_n,   W' = W o g (FP16),
//   c_n = sum_k W'_nk (of the rounded W'),           b'_n = b_n + sum_k W_nk beta_k.
// One warp per output row n; fixed reduction order (deterministic).
__global__ void k_fold_ln(const __half* __restrict__ W, const __half* __restrict__ g,
                          const __half* __restrict__ beta, const __half* __restrict__ bias, int N,
                          int K, __half* __restrict__ Wf, float* __restrict__ c,
                          __half* __restrict__ bf) {
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (n >= N) return;
  double cs = 0.0, bs = 0.0;
  for (int k = lane; k < K; k += 32) {
    const float w = __half2float(W[(size_t)n * K + k]);
    const __half wf = __float2half_rn(w * __half2float(g[k]));
    Wf[(size_t)n * K + k] = wf;
    cs += (double)__half2float(wf);
    bs += (double)w * (double)__half2float(beta[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cs += __shfl_xor_sync(0xffffffffu, cs, o);
    bs += __shfl_xor_sync(0xffffffffu, bs, o);
  }
  if (lane == 0) {
    c[n] = (float)cs;
    bf[n] = __float2half_rn((float)((bias ? (double)__half2float(bias[n]) : 0.0) + bs));
  }
}

void fold_ln(const void* W, const void* g, const void* beta, const void* bias, int N, int K,
             void* Wf, float* c, void* bf, cudaStream_t s) {
  k_fold_ln<<<ceil_div(N, 8), 256, 0, s>>>((const __half*)W, (const __half*)g,
                                          (const __half*)beta, (const __half*)bias, N, K,
                                          (__half*)Wf, c, (__half*)bf);
  NMT_LAUNCH_CHECK();
}

}  // namespace nmt
