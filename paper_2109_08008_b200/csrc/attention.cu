// attention.cu — RPR self-attention (Shaw et al.; "maximum relative
// length was 8"), cached decoder self-attention and cross-attention
// over the once-per-sentence encoder K/V.
//
// Bandwidth/latency-bound at these shapes (S <= 120, dh = 64): SIMT FP32 with every
// (query, key) pair and every (query, channel) pair in parallel; reductions by warp
// shuffle; no serial dependency chains.  Keys and values carry the clipped relative
// embeddings A^K[r], A^V[r], r(i,j) = clip(j - i, -k, k) + k (reading R7/R24):
//   e_ij = (q_i . k_j + q_i . A^K[r(i,j)]) / sqrt(dh)
//   o_i  = sum_j a_ij v_j + sum_r (sum_{j: r(i,j) = r} a_ij) A^V[r]
// The second form of o_i needs only the 2k+1 bucket sums: buckets 1..2k-1 hold one key
// each, buckets 0 and 2k the tails j <= i-k and j >= i+k.
#include "common.cuh"
#include "kernels.h"
#include "warp_attn.cuh"

namespace nmt {

template <class T> struct Vec8;   // 8 consecutive elements -> float[8]
template <> struct Vec8<__half> {
  static __device__ __forceinline__ void load(const __half* p, float* f) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 x = __half22float2(h[e]);
      f[2 * e] = x.x;
      f[2 * e + 1] = x.y;
    }
  }
};
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* f) {
    float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

template <int DH>
__device__ __forceinline__ float dot_ss(const float* __restrict__ a, const float* __restrict__ b) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int c = 0; c < DH; c += 4) {
    s0 = fmaf(a[c], b[c], s0);
    s1 = fmaf(a[c + 1], b[c + 1], s1);
    s2 = fmaf(a[c + 2], b[c + 2], s2);
    s3 = fmaf(a[c + 3], b[c + 3], s3);
  }
  return (s0 + s1) + (s2 + s3);
}

// ----------------------------------------------------------------- encoder (per sentence, head)
template <class T, int DH>
__global__ void __launch_bounds__(256) k_attn_enc(const T* __restrict__ qkv,
                                                  const int* __restrict__ len,
                                                  const T* __restrict__ relk,
                                                  const T* __restrict__ relv, T* __restrict__ out,
                                                  int S, int d, int kclip, int use_rpr) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, h = blockIdx.y;
  const int R = 2 * kclip + 1, LQ = DH + 1, LP = S + 1, LB = R + 1;
  float* sQ = sm;                  // [S][DH+1]
  float* sK = sQ + S * LQ;         // [S][DH+1]
  float* sV = sK + S * LQ;         // [S][DH]
  float* sAK = sV + S * DH;        // [R][DH+1]
  float* sAV = sAK + R * LQ;       // [R][DH]
  float* sQA = sAV + R * DH;       // [S][R+1]   q_i . A^K[r]
  float* sP = sQA + S * LB;        // [S][S+1]   scores -> probabilities
  float* sB = sP + S * LP;         // [S][R+1]   bucket sums
  const int n = len[b];
  const int tid = threadIdx.x, nt = blockDim.x;
  const size_t rs = 3 * (size_t)d;
  const T* base = qkv + (size_t)b * S * rs + h * DH;
  // phase 0: stage Q, K, V (8 elements per thread-iteration) and the relative tables
  for (int idx = tid; idx < n * (DH / 8); idx += nt) {
    const int j = idx / (DH / 8), c = (idx % (DH / 8)) * 8;
    float f[8];
    const T* rp = base + (size_t)j * rs + c;
    Vec8<T>::load(rp, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) sQ[j * LQ + c + e] = f[e];
    Vec8<T>::load(rp + d, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) sK[j * LQ + c + e] = f[e];
    Vec8<T>::load(rp + 2 * d, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) sV[j * DH + c + e] = f[e];
  }
  if (use_rpr)
    for (int idx = tid; idx < R * DH; idx += nt) {
      const int r = idx / DH, c = idx % DH;
      sAK[r * LQ + c] = to_f(relk[idx]);
      sAV[r * DH + c] = to_f(relv[idx]);
    }
  __syncthreads();
  // phase 1: raw scores q_i . k_j for every pair, 4x4 register tiles (rows i = ib + r*n4,
  // cols j = jb + s*n4 so a warp's K rows are consecutive -> conflict-free) and
  // q_i . A^K[r] for every (i, r)
  const int n4 = (n + 3) >> 2;
  for (int idx = tid; idx < n4 * n4; idx += nt) {
    const int ib = idx / n4, jb = idx - ib * n4;
    const float* qa[4];
    const float* kb[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      qa[r] = sQ + min(ib + r * n4, n - 1) * LQ;
      kb[r] = sK + min(jb + r * n4, n - 1) * LQ;
    }
    float acc[4][4] = {};
#pragma unroll 8
    for (int c = 0; c < DH; ++c) {
      float a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a[r] = qa[r][c];
        b[r] = kb[r][c];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) acc[r][s2] = fmaf(a[r], b[s2], acc[r][s2]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = ib + r * n4;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        const int j = jb + s2 * n4;
        if (i < n && j < n) sP[i * LP + j] = acc[r][s2];
      }
    }
  }
  if (use_rpr)
    for (int idx = tid; idx < n * R; idx += nt) {
      const int i = idx / R, r = idx - i * R;
      sQA[i * LB + r] = dot_ss<DH>(sQ + i * LQ, sAK + r * LQ);
    }
  __syncthreads();
  // phase 2: masked FP32 softmax per query row (warp per row) + bucket sums
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const float scale = rsqrtf((float)DH);
  for (int i = warp; i < n; i += nw) {
    float* p = sP + i * LP;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) {
      float e = p[j];
      if (use_rpr) e += sQA[i * LB + min(max(j - i, -kclip), kclip) + kclip];
      e *= scale;
      p[j] = e;
      mx = fmaxf(mx, e);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float e = __expf(p[j] - mx);
      p[j] = e;
      sum += e;
    }
    const float inv = 1.f / warp_sum(sum);
    float lo = 0.f, hi = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float a = p[j] * inv;
      p[j] = a;
      if (j - i <= -kclip) lo += a;
      if (j - i >= kclip) hi += a;
    }
    if (use_rpr) {
      lo = warp_sum(lo);
      hi = warp_sum(hi);
      __syncwarp();
      if (lane < R) {
        float v;
        if (lane == 0) v = lo;
        else if (lane == R - 1) v = hi;
        else {
          const int j = i + lane - kclip;
          v = (j >= 0 && j < n) ? p[j] : 0.f;
        }
        sB[i * LB + lane] = v;
      }
    }
  }
  __syncthreads();
  // phase 3: o_i[c] = sum_j a_ij v_j[c] + sum_r B_ir A^V[r][c]; 4 rows x 4 channels per
  // thread (rows i = ib + r*n4, channels c = cb + k*DH/4: a warp reads consecutive V columns)
  T* obase = out + (size_t)b * S * d + h * DH;
  constexpr int CQ = DH / 4;
  for (int idx = tid; idx < n4 * CQ; idx += nt) {
    const int ib = idx / CQ, cb = idx - ib * CQ;
    const float* pr[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) pr[r] = sP + min(ib + r * n4, n - 1) * LP;
    float acc[4][4] = {};
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
      float pv[4], vv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pv[r] = pr[r][j];
#pragma unroll
      for (int k = 0; k < 4; ++k) vv[k] = sV[j * DH + cb + k * CQ];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[r][k] = fmaf(pv[r], vv[k], acc[r][k]);
    }
    if (use_rpr) {
      for (int rr = 0; rr < R; ++rr) {
        float bv[4], av[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) bv[r] = sB[min(ib + r * n4, n - 1) * LB + rr];
#pragma unroll
        for (int k = 0; k < 4; ++k) av[k] = sAV[rr * DH + cb + k * CQ];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[r][k] = fmaf(bv[r], av[k], acc[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = ib + r * n4;
      if (i < n) {
#pragma unroll
        for (int k = 0; k < 4; ++k) obase[(size_t)i * d + cb + k * CQ] = from_f<T>(acc[r][k]);
      }
    }
  }
  // padding query rows -> 0 (finite inputs for the following GEMM / LN)
  for (int idx = n * DH + tid; idx < S * DH; idx += nt) {
    const int i = idx / DH, c = idx - i * DH;
    obase[(size_t)i * d + c] = from_f<T>(0.f);
  }
}

template <class T, int DH>
void launch_enc(const T* qkv, const int* len, const T* relk, const T* relv, T* out, int B, int S,
                int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  const int R = 2 * kclip + 1;
  size_t fl = 2 * S * (DH + 1) + S * DH + R * (DH + 1) + R * DH + S * (R + 1) + S * (S + 1) +
              S * (R + 1);
  size_t smem = fl * sizeof(float);
  // thread-safe one-time attribute setup (C++11 static initialisation)
  static const bool attr = [&] {
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    return true;
  }();
  (void)attr;
  k_attn_enc<T, DH><<<dim3(B, H), 256, smem, s>>>(qkv, len, relk, relv, out, S, d, kclip, use_rpr);
  NMT_LAUNCH_CHECK();
}

template <class T>
void attn_encoder(const T* qkv, const int* len, const T* relk, const T* relv, T* out, int B, int S,
                  int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  if (B <= 0) return;
  if constexpr (sizeof(T) == 2) {  // FP16 mode: all contractions on tensor cores
    attn_encoder_tc(reinterpret_cast<const __half*>(qkv), len,
                    reinterpret_cast<const __half*>(relk), reinterpret_cast<const __half*>(relv),
                    reinterpret_cast<__half*>(out), B, S, d, H, kclip, use_rpr, s);
    return;
  }
  switch (d / H) {
    case 16: launch_enc<T, 16>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 32: launch_enc<T, 32>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 64: launch_enc<T, 64>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    default: throw CudaError("attn_encoder: head dim must be 16, 32 or 64");
  }
}

// ----------------------------------------------------------------- decoder attention
// One warp per (live row, head).  The keys are split over lane groups: G = DH/8 lanes hold
// the 8-channel slices of one key (one 16-B load each, a group reads the key's contiguous
// DH-element head slice), KP = 32/G keys per warp pass, U passes per chunk of CH = KP*U
// keys.  A chunk issues all of its K and V loads before any arithmetic (2U independent
// loads per lane in flight), so a step costs about one memory round trip per chunk instead
// of a dependent chain per key.  Softmax is online over chunks (running max and sum,
// FP32, rescaled per chunk).  The RPR value term is folded per key, v_j + A^V[r(j)], which
// is the same sum as the bucket form sum_r (sum_{j in r} a_j) A^V[r] above.
// ----------------------------------------------------------------- decoder self-attention
// Step t = *d_t: k_t, v_t are appended to the row's cache slot and
// positions 0..t attended; key t is taken from the fresh projection.  Only buckets
// r = clip(j - t, -k, k) + k in 0..k occur (j <= t).  Beam rows read their ancestors'
// cached positions j < t through the ancestry table (no K/V copies).
// Occupancy: 6 CTAs (24 warps) per SM; a warp's keys are short dependent load chains, so
// the step time at thousands of rows is the number of warp waves times that latency.  The
// relative tables are read per lane from global memory (L1-resident, 2 x (k+1) x dh
// elements): no per-CTA staging barrier.
template <class T, int DH>
__global__ void __launch_bounds__(128, sizeof(T) == 2 ? 6 : 4) k_attn_dec_self(
    const T* __restrict__ qkv, T* __restrict__ kc, T* __restrict__ vc, int Tmax,
    const int* __restrict__ row_slot, const T* __restrict__ relk, const T* __restrict__ relv,
    T* __restrict__ out, int rows, int d, int H, int kclip, int use_rpr, const int* __restrict__ d_t,
    const int* __restrict__ dR, const int* __restrict__ anc) {
  __shared__ float s_x[4][16];      // per warp: q . A^K[r] / sqrt(dh), r = 0..k
  using WA = WarpAttn<T, DH>;
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw - (gw / H) * H;
  // one memory round trip for everything that does not depend on the cache slot: the
  // device scalars, this row's slot, q / k_t / v_t (row clamped to the host bound so the
  // loads stay in bounds) and the relative tables
  const int nlive = *dR, t = *d_t;
  const int rowc = min(row, rows - 1);
  const int slot = row_slot[rowc];
  const T* src = qkv + (size_t)rowc * 3 * d + h * DH;
  WA w;
  w.init(lane, src, rsqrtf((float)DH));
  Raw8<T> kt, vt;
  if (w.kq == 0) {
    kt.load(src + d + w.sub * 8);
    vt.load(src + 2 * d + w.sub * 8);
  }
  if (row >= min(rows, nlive)) return;
  if (w.kq == 0) {  // KV-cache append at position t
    kt.store(kc + ((size_t)slot * Tmax + t) * d + h * DH + w.sub * 8);
    vt.store(vc + ((size_t)slot * Tmax + t) * d + h * DH + w.sub * 8);
  }
  float* x = s_x[warp];
  if (use_rpr) {
    for (int b0 = 0; b0 <= kclip; b0 += WA::KP) {
      const int b = b0 + w.kq;
      float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (b <= kclip) {
        Raw8<T> r;
        r.load(relk + b * DH + w.sub * 8);
        r.to_f(f);
      }
      const float e = w.group_dot(f);
      if (b <= kclip && w.sub == 0) x[b] = e;
    }
    __syncwarp();
  }
  const int* anc_row = anc ? anc + (size_t)slot * Tmax : nullptr;
  const size_t hoff = (size_t)h * DH;
  auto addr = [&](int j, const T*& kp, const T*& vp) {
    if (j == t) {
      kp = src + d;
      vp = src + 2 * d;
    } else {
      const int sl = anc_row ? anc_row[j] : slot;
      const size_t o = ((size_t)sl * Tmax + j) * d + hoff;
      kp = kc + o;
      vp = vc + o;
    }
  };
  const int n = t + 1;
  if (use_rpr) {
    auto bias = [&](int j) { return x[max(j - t, -kclip) + kclip]; };
    auto vadd = [&](int j, float* f) {
      Raw8<T> r;
      r.load(relv + (max(j - t, -kclip) + kclip) * DH + w.sub * 8);
      float rv[8];
      r.to_f(rv);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] += rv[e];
    };
    for (int j0 = 0; j0 < n; j0 += WA::CH) w.chunk(j0, n, n, addr, bias, vadd);
  } else {
    auto bias = [](int) { return 0.f; };
    auto vadd = [](int, float*) {};
    for (int j0 = 0; j0 < n; j0 += WA::CH) w.chunk(j0, n, n, addr, bias, vadd);
  }
  float o[8];
  w.finish(o);
  if (w.kq == 0) store8(out + (size_t)row * d + hoff + w.sub * 8, o);
}

template <class T>
void attn_decoder_self(const T* qkv, T* kc, T* vc, int Tmax, const int* row_slot, const T* relk,
                       const T* relv, T* out, int rows, int d, int H, int kclip, int use_rpr,
                       const int* d_t, const int* dR, const int* anc, cudaStream_t s) {
  if (rows <= 0) return;
  const int nw = 4, dh = d / H;
  dim3 grid(ceil_div(rows * H, nw));
#define NMT_DS(DH)                                                                           \
  launch_k(k_attn_dec_self<T, DH>, grid, nw * 32, 0, s, qkv, kc, vc, Tmax, row_slot, relk, \
           relv, out, rows, d, H, kclip, use_rpr, d_t, dR, anc)
  switch (dh) {
    case 16: NMT_DS(16); break;
    case 32: NMT_DS(32); break;
    case 64: NMT_DS(64); break;
    default: throw CudaError("attn_decoder_self: head dim must be 16, 32 or 64");
  }
#undef NMT_DS
  NMT_LAUNCH_CHECK();
}

// ----------------------------------------------------------------- cross-attention
// One warp per (live row, head) over the sentence's once-computed encoder K/V:
// keys at ckv + (slot*S + j)*ldkv + koff + h*dh, values at + voff; mask j < src_len[slot].
// S = *dS (device) so a captured step graph serves every batch.  Beam rows share their
// sentence's K/V (slot = row slot / beam).
// 8 CTAs per SM (64 registers): at 8192 rows 110 -> 98 us per step; the self-attention keeps
// 6 (at 8 its long-history steps slow down: 319 -> 385 us at t = 56..120)
template <class T, int DH>
__global__ void __launch_bounds__(128, sizeof(T) == 2 ? 8 : 4) k_attn_cross(
    const T* __restrict__ qb, const T* __restrict__ ckv, int ldkv, int koff, int voff,
    const int* __restrict__ dS, const int* __restrict__ src_len,
    const int* __restrict__ row_slot, T* __restrict__ out, int rows, int d, int H,
    const int* __restrict__ dR, int beam) {
  using WA = WarpAttn<T, DH>;
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw - (gw / H) * H;
  if (row >= rows) return;
  // round trip 1: scalars, slot, q; round trip 2: the source length together with the
  // first key chunk (loaded up to S, the batch's padded length, and masked by n)
  const int nlive = *dR, S = *dS;
  const int slot = row_slot[row] / beam;
  WA w;
  w.init(lane, qb + (size_t)row * d + h * DH, rsqrtf((float)DH));
  if (row >= nlive) return;
  const int n = src_len[slot];
  const T* base = ckv + (size_t)slot * S * ldkv + h * DH;
  auto addr = [&](int j, const T*& kp, const T*& vp) {
    kp = base + (size_t)j * ldkv + koff;
    vp = base + (size_t)j * ldkv + voff;
  };
  auto bias = [](int) { return 0.f; };
  auto vadd = [](int, float*) {};
  w.chunk(0, n, S, addr, bias, vadd);
  for (int j0 = WA::CH; j0 < n; j0 += WA::CH) w.chunk(j0, n, n, addr, bias, vadd);
  float o[8];
  w.finish(o);
  if (w.kq == 0) store8(out + (size_t)row * d + h * DH + w.sub * 8, o);
}

template <class T>
void attn_cross(const T* q, const T* ckv, int ldkv, int koff, int voff, const int* dS, int Smax,
                const int* src_len, const int* row_slot, T* out, int rows, int d, int H,
                const int* dR, int beam, cudaStream_t s) {
  if (rows <= 0) return;
  (void)Smax;
  const int nw = 4, dh = d / H;
  dim3 grid(ceil_div(rows * H, nw));
#define NMT_CS(DH)                                                                          \
  launch_k(k_attn_cross<T, DH>, grid, nw * 32, 0, s, q, ckv, ldkv, koff, voff, dS, src_len, \
           row_slot, out, rows, d, H, dR, beam)
  switch (dh) {
    case 16: NMT_CS(16); break;
    case 32: NMT_CS(32); break;
    case 64: NMT_CS(64); break;
    default: throw CudaError("attn_cross: head dim must be 16, 32 or 64");
  }
#undef NMT_CS
  NMT_LAUNCH_CHECK();
}

#define NMT_INST_ATT(T)                                                                         \
  template void attn_encoder<T>(const T*, const int*, const T*, const T*, T*, int, int, int,    \
                                int, int, int, cudaStream_t);                                   \
  template void attn_decoder_self<T>(const T*, T*, T*, int, const int*, const T*, const T*, T*, \
                                     int, int, int, int, int, const int*, const int*,           \
                                     const int*, cudaStream_t);                                 \
  template void attn_cross<T>(const T*, const T*, int, int, int, const int*, int, const int*,   \
                              const int*, T*, int, int, int, const int*, int, cudaStream_t);
NMT_INST_ATT(float)
NMT_INST_ATT(__half)

}  // namespace nmt
