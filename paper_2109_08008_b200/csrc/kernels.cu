// kernels.cu — bandwidth-/latency-bound kernels of the hot path (sm_100a).
// Embedding, LayerNorm, DLCL combine, RPR attention (encoder / cached decoder),
// cross-attention, greedy bookkeeping, batch-pruning compaction.
// All reductions (LN statistics, softmax, DLCL sums) run in FP32.
#include "common.cuh"
#include "kernels.h"

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
void layernorm(const T* in, int ldi, const T* g, const T* b, T* out, int ldo, int rows, int d,
               float eps, const int* dR, cudaStream_t s) {
  if (rows <= 0) return;
  k_layernorm<T><<<ceil_div(rows, 8), 256, 0, s>>>(in, ldi, g, b, out, ldo, rows, d, eps, dR);
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
                  int d, float eps, cudaStream_t s) {
  if (rows <= 0) return;
  k_dlcl<T><<<ceil_div(rows, 8), 256, 0, s>>>(y, hist, hist_stride, l, w, gdl, bdl, dlcl_ln, g2,
                                               b2, xout, uout, rows, d, eps);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- attention helpers
template <class T>
__device__ __forceinline__ float dot_gs(const T* __restrict__ row, const float* __restrict__ q,
                                        int dh) {
  float acc = 0.f;
  for (int c = 0; c < dh; ++c) acc += to_f(row[c]) * q[c];
  return acc;
}
template <>
__device__ __forceinline__ float dot_gs<__half>(const __half* __restrict__ row,
                                                const float* __restrict__ q, int dh) {
  float acc = 0.f;
  if ((dh & 7) == 0) {
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
    for (int c8 = 0; c8 < (dh >> 3); ++c8) {
      uint4 u = r4[c8];
      const __half2* h2 = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __half22float2(h2[e]);
        acc += f.x * q[c8 * 8 + 2 * e] + f.y * q[c8 * 8 + 2 * e + 1];
      }
    }
  } else {
    for (int c = 0; c < dh; ++c) acc += __half2float(row[c]) * q[c];
  }
  return acc;
}

// ------------------------------------------------------------------- encoder RPR attention
// grid (B, H), 4 warps; Q, K, V of one (sentence, head) staged in shared memory as FP32.
//   e_ij = (q_i . k_j + q_i . A^K[r(i,j)]) / sqrt(dh)   masked j >= len
//   o_i  = sum_j a_ij v_j + sum_r (sum_{j: r(i,j)=r} a_ij) A^V[r]
template <class T>
__global__ void k_attn_enc(const T* __restrict__ qkv, const int* __restrict__ len,
                           const T* __restrict__ relk, const T* __restrict__ relv,
                           T* __restrict__ out, int S, int d, int H, int kclip, int use_rpr) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, h = blockIdx.y;
  const int dh = d / H, R = 2 * kclip + 1, ld = dh + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* sQ = sm;                 // [S][dh+1]
  float* sK = sQ + S * ld;        // [S][dh+1]
  float* sV = sK + S * ld;        // [S][dh]
  float* sAK = sV + S * dh;       // [R][dh]
  float* sAV = sAK + R * dh;      // [R][dh]
  float* sP = sAV + R * dh;       // [nw][S]
  float* sX = sP + nw * S;        // [nw][32]  (qa, then bucket sums)
  const int n = len[b];
  const size_t rs = 3 * (size_t)d;
  for (int idx = threadIdx.x; idx < n * dh; idx += blockDim.x) {
    int j = idx / dh, c = idx % dh;
    const T* rp = qkv + ((size_t)b * S + j) * rs + h * dh + c;
    sQ[j * ld + c] = to_f(rp[0]);
    sK[j * ld + c] = to_f(rp[d]);
    sV[j * dh + c] = to_f(rp[2 * d]);
  }
  if (use_rpr)
    for (int idx = threadIdx.x; idx < R * dh; idx += blockDim.x) {
      sAK[idx] = to_f(relk[idx]);
      sAV[idx] = to_f(relv[idx]);
    }
  __syncthreads();
  const float scale = rsqrtf((float)dh);
  float* p = sP + warp * S;
  float* x = sX + warp * 32;
  for (int i = warp; i < S; i += nw) {
    T* orow = out + ((size_t)b * S + i) * d + h * dh;
    if (i >= n) {  // padding query rows: zero output
      for (int c = lane; c < dh; c += 32) orow[c] = from_f<T>(0.f);
      continue;
    }
    const float* qi = sQ + i * ld;
    if (use_rpr) {
      if (lane < R) {
        float a = 0.f;
        for (int c = 0; c < dh; ++c) a += qi[c] * sAK[lane * dh + c];
        x[lane] = a;
      }
      __syncwarp();
    }
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) {
      const float* kj = sK + j * ld;
      float e = 0.f;
      for (int c = 0; c < dh; ++c) e += qi[c] * kj[c];
      if (use_rpr) e += x[min(max(j - i, -kclip), kclip) + kclip];
      e *= scale;
      p[j] = e;
      mx = fmaxf(mx, e);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < n; j += 32) {
      float e = __expf(p[j] - mx);
      p[j] = e;
      sum += e;
    }
    const float inv = 1.f / warp_sum(sum);
    __syncwarp();
    if (use_rpr) {
      if (lane < R) {  // bucket sums of the normalised weights
        float bs = 0.f;
        int r = lane;
        if (r == 0) {
          for (int j = 0; j <= min(i - kclip, n - 1); ++j) bs += p[j];
        } else if (r == R - 1) {
          for (int j = max(i + kclip, 0); j < n; ++j) bs += p[j];
        } else {
          int j = i + r - kclip;
          if (j >= 0 && j < n) bs = p[j];
        }
        x[lane] = bs * inv;
      }
      __syncwarp();
    }
    for (int c = lane; c < dh; c += 32) {
      float o = 0.f;
      for (int j = 0; j < n; ++j) o += p[j] * sV[j * dh + c];
      o *= inv;
      if (use_rpr)
        for (int r = 0; r < R; ++r) o += x[r] * sAV[r * dh + c];
      orow[c] = from_f<T>(o);
    }
    __syncwarp();
  }
}

template <class T>
void attn_encoder(const T* qkv, const int* len, const T* relk, const T* relv, T* out, int B, int S,
                  int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  if (B <= 0) return;
  const int dh = d / H, R = 2 * kclip + 1, nw = 4;
  size_t smem = sizeof(float) * (2 * S * (dh + 1) + S * dh + 2 * R * dh + nw * S + nw * 32);
  static bool attr_set[2] = {false, false};
  bool& set = attr_set[sizeof(T) == 2];
  if (!set) {
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    set = true;
  }
  k_attn_enc<T><<<dim3(B, H), nw * 32, smem, s>>>(qkv, len, relk, relv, out, S, d, H, kclip,
                                                  use_rpr);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- decoder self-attention
// One warp per (live row, head).  Step t: write k_t, v_t to the cache slot, then attend
// over j = 0..t; only buckets 0..k occur (j <= t) and every j <= t-k shares bucket 0.
template <class T>
__global__ void k_attn_dec_self(const T* __restrict__ qkv, T* __restrict__ kc, T* __restrict__ vc,
                                int Tmax, const int* __restrict__ row_slot,
                                const T* __restrict__ relk, const T* __restrict__ relv,
                                T* __restrict__ out, int rows, int d, int H, int kclip,
                                int use_rpr, const int* __restrict__ d_t,
                                const int* __restrict__ dR) {
  extern __shared__ float sm[];
  const int dh = d / H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw % H;
  const int nrows = min(rows, *dR);
  if (row >= nrows) return;
  const int t = *d_t;
  float* q = sm + warp * (dh + 32 + Tmax);
  float* x = q + dh;
  float* p = x + 32;
  const int slot = row_slot[row];
  const T* src = qkv + (size_t)row * 3 * d + h * dh;
  T* krow = kc + ((size_t)slot * Tmax + t) * d + h * dh;
  T* vrow = vc + ((size_t)slot * Tmax + t) * d + h * dh;
  for (int c = lane; c < dh; c += 32) {
    q[c] = to_f(src[c]);
    krow[c] = src[d + c];
    vrow[c] = src[2 * d + c];
  }
  __syncwarp();
  if (use_rpr && lane <= kclip) {
    float a = 0.f;
    for (int c = 0; c < dh; ++c) a += q[c] * to_f(relk[lane * dh + c]);
    x[lane] = a;
  }
  __syncwarp();
  const float scale = rsqrtf((float)dh);
  float mx = -INFINITY;
  const T* kbase = kc + (size_t)slot * Tmax * d + h * dh;
  for (int j = lane; j <= t; j += 32) {
    float e = dot_gs<T>(kbase + (size_t)j * d, q, dh);
    if (use_rpr) e += x[max(j - t, -kclip) + kclip];
    e *= scale;
    p[j] = e;
    mx = fmaxf(mx, e);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j <= t; j += 32) {
    float e = __expf(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  const float inv = 1.f / warp_sum(sum);
  __syncwarp();
  if (use_rpr) {
    float bs = 0.f;
    if (lane == 0) {
      for (int j = 0; j <= t - kclip; ++j) bs += p[j];
    } else if (lane <= kclip) {
      int j = t - kclip + lane;
      if (j >= 0) bs = p[j];
    }
    __syncwarp();
    if (lane <= kclip) x[lane] = bs * inv;
    __syncwarp();
  }
  const T* vbase = vc + (size_t)slot * Tmax * d + h * dh;
  T* orow = out + (size_t)row * d + h * dh;
  for (int c = lane; c < dh; c += 32) {
    float o = 0.f;
    for (int j = 0; j <= t; ++j) o += p[j] * to_f(vbase[(size_t)j * d + c]);
    o *= inv;
    if (use_rpr)
      for (int r = 0; r <= kclip; ++r) o += x[r] * to_f(relv[r * dh + c]);
    orow[c] = from_f<T>(o);
  }
}

template <class T>
void attn_decoder_self(const T* qkv, T* kc, T* vc, int Tmax, const int* row_slot, const T* relk,
                       const T* relv, T* out, int rows, int d, int H, int kclip, int use_rpr,
                       const int* d_t, const int* dR, cudaStream_t s) {
  if (rows <= 0) return;
  const int nw = 4, dh = d / H;
  size_t smem = sizeof(float) * nw * (dh + 32 + Tmax);
  k_attn_dec_self<T><<<ceil_div(rows * H, nw), nw * 32, smem, s>>>(
      qkv, kc, vc, Tmax, row_slot, relk, relv, out, rows, d, H, kclip, use_rpr, d_t, dR);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- cross-attention
template <class T>
__global__ void k_attn_cross(const T* __restrict__ qb, const T* __restrict__ ckv, int ldkv,
                             int koff, int voff, int S, const int* __restrict__ src_len,
                             const int* __restrict__ row_slot, T* __restrict__ out, int rows,
                             int d, int H, const int* __restrict__ dR) {
  extern __shared__ float sm[];
  const int dh = d / H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw % H;
  const int nrows = min(rows, *dR);
  if (row >= nrows) return;
  float* q = sm + warp * (dh + S);
  float* p = q + dh;
  const int slot = row_slot[row];
  const int n = src_len[slot];
  for (int c = lane; c < dh; c += 32) q[c] = to_f(qb[(size_t)row * d + h * dh + c]);
  __syncwarp();
  const float scale = rsqrtf((float)dh);
  const T* base = ckv + (size_t)slot * S * ldkv + h * dh;
  float mx = -INFINITY;
  for (int j = lane; j < n; j += 32) {
    float e = dot_gs<T>(base + (size_t)j * ldkv + koff, q, dh) * scale;
    p[j] = e;
    mx = fmaxf(mx, e);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < n; j += 32) {
    float e = __expf(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  const float inv = 1.f / warp_sum(sum);
  __syncwarp();
  T* orow = out + (size_t)row * d + h * dh;
  for (int c = lane; c < dh; c += 32) {
    float o = 0.f;
    for (int j = 0; j < n; ++j) o += p[j] * to_f(base[(size_t)j * ldkv + voff + c]);
    orow[c] = from_f<T>(o * inv);
  }
}

template <class T>
void attn_cross(const T* q, const T* ckv, int ldkv, int koff, int voff, int S, const int* src_len,
                const int* row_slot, T* out, int rows, int d, int H, const int* dR, cudaStream_t s) {
  if (rows <= 0) return;
  const int nw = 4, dh = d / H;
  size_t smem = sizeof(float) * nw * (dh + S);
  k_attn_cross<T><<<ceil_div(rows * H, nw), nw * 32, smem, s>>>(q, ckv, ldkv, koff, voff, S,
                                                                 src_len, row_slot, out, rows, d,
                                                                 H, dR);
  NMT_LAUNCH_CHECK();
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

constexpr int kPruneMaxRows = 4096;

__global__ void __launch_bounds__(1024) k_prune(DevState* st, int* row_slot, int* prev_tok,
                                                uint8_t* done, int every, float ratio,
                                                int* new_to_old) {
  __shared__ int s_slot[kPruneMaxRows];
  __shared__ int s_tok[kPruneMaxRows];
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
  // each thread owns a contiguous chunk of rows
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  int keep = 0;
  for (int i = lo; i < hi; ++i) {
    s_slot[i] = row_slot[i];
    s_tok[i] = prev_tok[i];
    keep += done[i] ? 0 : 1;
  }
  int base = block_excl_scan(keep, &s_total);
  __syncthreads();
  int o = base;
  for (int i = lo; i < hi; ++i) {
    if (!done[i]) {
      row_slot[o] = s_slot[i];
      prev_tok[o] = s_tok[i];
      if (new_to_old) new_to_old[o] = i;
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
                   float ratio, int* new_to_old, int rows_upper, cudaStream_t s) {
  if (rows_upper > kPruneMaxRows) throw CudaError("prune_compact: too many rows");
  k_prune<<<1, 1024, 0, s>>>(st, row_slot, prev_tok, done, every, ratio, new_to_old);
  NMT_LAUNCH_CHECK();
}

__global__ void k_batch_init(int* row_slot, int* prev_tok, uint8_t* done, int* gen_len,
                             DevState* st, int B, int bos) {
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
  }
}

void batch_init(int* row_slot, int* prev_tok, uint8_t* done, int* gen_len, DevState* st, int B,
                int bos, cudaStream_t s) {
  k_batch_init<<<ceil_div(B > 0 ? B : 1, 128), 128, 0, s>>>(row_slot, prev_tok, done, gen_len, st,
                                                            B, bos);
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
                       int* bad) {
  const int b = blockIdx.x;
  const long long o = boff[b];
  const int n = blen[b];
  for (int p = threadIdx.x; p < S; p += blockDim.x) {
    int v = p < n ? ids[o + p] : 0;
    if (v < 0 || v >= vocab) {
      atomicOr(bad, 1);
      v = 0;
    }
    out[(size_t)b * S + p] = v;
  }
}

void pack_sources(const int* ids, const long long* boff, const int* blen, int B, int S, int* out,
                  int vocab, int* bad, cudaStream_t s) {
  if (B <= 0) return;
  k_pack<<<B, 128, 0, s>>>(ids, boff, blen, S, out, vocab, bad);
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
                                int, const T*, const T*, T*, T*, int, int, float, cudaStream_t); \
  template void attn_encoder<T>(const T*, const int*, const T*, const T*, T*, int, int, int,    \
                                int, int, int, cudaStream_t);                                   \
  template void attn_decoder_self<T>(const T*, T*, T*, int, const int*, const T*, const T*, T*, \
                                     int, int, int, int, int, const int*, const int*,           \
                                     cudaStream_t);                                             \
  template void attn_cross<T>(const T*, const T*, int, int, int, int, const int*, const int*,   \
                              T*, int, int, int, const int*, cudaStream_t);                     \
  template void to_float<T>(const T*, float*, size_t, cudaStream_t);
NMT_INST(float)
NMT_INST(__half)

}  // namespace nmt
