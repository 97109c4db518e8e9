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
  static bool attr = false;
  if (!attr) {
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    attr = true;
  }
  k_attn_enc<T, DH><<<dim3(B, H), 256, smem, s>>>(qkv, len, relk, relv, out, S, d, kclip, use_rpr);
  NMT_LAUNCH_CHECK();
}

// ----------------------------------------------------------------- encoder, FP16 tensor cores
// Same computation for the FP16 path with warp-level mma.sync (m16n8k16, FP16 in / FP32
// accumulate): S = Q K^T and O = P V on tensor cores, the RPR terms q . A^K[r] and
// sum_r B_ir A^V[r] in FP32 SIMT.  Scores, softmax and bucket sums stay in registers
// (FP32); P is rounded to FP16 only as the A operand of P V (within the FP16-mode
// tolerance).  One CTA per (sentence, head), 4 warps, each owning 16-query blocks.
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int DH, int NT>  // NT = number of 8-wide key tiles (Sp = 8*NT, multiple of 16)
__global__ void __launch_bounds__(128) k_attn_enc_mma(const __half* __restrict__ qkv,
                                                      const int* __restrict__ len,
                                                      const __half* __restrict__ relk,
                                                      const __half* __restrict__ relv,
                                                      __half* __restrict__ out, int S, int d,
                                                      int kclip, int use_rpr) {
  constexpr int SP = NT * 8, LDH = DH + 8;  // padded row (16-B multiple, conflict-free ldmatrix)
  extern __shared__ __align__(16) uint8_t smraw[];
  __half* sQ = reinterpret_cast<__half*>(smraw);   // [SP][LDH]
  __half* sK = sQ + SP * LDH;                       // [SP][LDH]
  __half* sV = sK + SP * LDH;                       // [SP][LDH]
  float* sAK = reinterpret_cast<float*>(sV + SP * LDH);  // [R][DH]
  float* sAV = sAK + 32 * (DH + 1);                       // [R][DH]  (sAK rows padded: DH+1)
  float* sQA = sAV + 32 * DH;                             // [SP][R+1]
  float* sB = sQA + SP * 33;                              // [SP][R+1]
  const int b = blockIdx.x, h = blockIdx.y;
  const int R = 2 * kclip + 1, LB = 33;
  const int n = len[b];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t rs = 3 * (size_t)d;
  const __half* base = qkv + (size_t)b * S * rs + h * DH;
  // stage Q, K, V (zero rows >= n) and the relative tables
  for (int idx = tid; idx < SP * (DH / 8); idx += 128) {
    const int j = idx / (DH / 8), c = (idx % (DH / 8)) * 8;
    uint4 q = make_uint4(0, 0, 0, 0), k = q, v = q;
    if (j < n) {
      const __half* rp = base + (size_t)j * rs + c;
      q = *reinterpret_cast<const uint4*>(rp);
      k = *reinterpret_cast<const uint4*>(rp + d);
      v = *reinterpret_cast<const uint4*>(rp + 2 * d);
    }
    *reinterpret_cast<uint4*>(sQ + j * LDH + c) = q;
    *reinterpret_cast<uint4*>(sK + j * LDH + c) = k;
    *reinterpret_cast<uint4*>(sV + j * LDH + c) = v;
  }
  if (use_rpr) {
    for (int idx = tid; idx < R * DH; idx += 128) {
      sAK[(idx / DH) * (DH + 1) + idx % DH] = __half2float(relk[idx]);
      sAV[idx] = __half2float(relv[idx]);
    }
    for (int idx = tid; idx < SP * LB; idx += 128) sB[idx] = 0.f;
  }
  __syncthreads();
  if (use_rpr)  // q_i . A^K[r] (FP32 SIMT)
    for (int idx = tid; idx < n * R; idx += 128) {
      const int i = idx / R, r = idx - i * R;
      float a = 0.f;
#pragma unroll 8
      for (int c = 0; c < DH; ++c) a = fmaf(__half2float(sQ[i * LDH + c]), sAK[r * (DH + 1) + c], a);
      sQA[i * LB + r] = a;
    }
  __syncthreads();
  const float scale = rsqrtf((float)DH);
  const int g = lane >> 2, tig = lane & 3;
  const int nblk = (n + 15) >> 4;
  for (int mb = warp; mb < nblk; mb += 4) {
    const int m0 = mb * 16;
    // ---- S = Q K^T for rows m0..m0+15, all SP key columns
    float sc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < DH; k0 += 16) {
      uint32_t af[4];
      {
        const int mi = lane >> 3, rr = lane & 7;
        ldsm_x4(af, sQ + (m0 + rr + (mi & 1) * 8) * LDH + k0 + (mi >> 1) * 8);
      }
#pragma unroll
      for (int t = 0; t < NT; t += 2) {
        uint32_t bf[4];  // matrices (t, k0) (t, k0+8) (t+1, k0) (t+1, k0+8)
        const int mi = lane >> 3, rr = lane & 7;
        ldsm_x4(bf, sK + ((t + (mi >> 1)) * 8 + rr) * LDH + k0 + (mi & 1) * 8);
        mma16816(sc[t], af, bf[0], bf[1]);
        mma16816(sc[t + 1], af, bf[2], bf[3]);
      }
    }
    // ---- RPR key term, mask, scale, softmax (rows r0 = m0+g, r1 = m0+g+8)
    const int r0 = m0 + g, r1 = r0 + 8;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = e < 2 ? r0 : r1, j = t * 8 + 2 * tig + (e & 1);
        float v = sc[t][e];
        if (j < n && i < n) {
          if (use_rpr) v += sQA[i * LB + min(max(j - i, -kclip), kclip) + kclip];
          v *= scale;
        } else {
          v = -INFINITY;
        }
        sc[t][e] = v;
        if (e < 2) mx0 = fmaxf(mx0, v);
        else mx1 = fmaxf(mx1, v);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    if (mx0 == -INFINITY) mx0 = 0.f;  // padding query rows
    if (mx1 == -INFINITY) mx1 = 0.f;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = __expf(sc[t][e] - (e < 2 ? mx0 : mx1));
        sc[t][e] = v;
        if (e < 2) s0 += v;
        else s1 += v;
      }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    const float inv0 = s0 > 0.f ? 1.f / s0 : 0.f, inv1 = s1 > 0.f ? 1.f / s1 : 0.f;
    float lo0 = 0.f, hi0 = 0.f, lo1 = 0.f, hi1 = 0.f;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool top = e < 2;
        const int i = top ? r0 : r1, j = t * 8 + 2 * tig + (e & 1);
        const float p = sc[t][e] * (top ? inv0 : inv1);
        sc[t][e] = p;
        if (use_rpr && i < n && j < n) {
          const int dj = j - i;
          if (dj <= -kclip) { if (top) lo0 += p; else lo1 += p; }
          else if (dj >= kclip) { if (top) hi0 += p; else hi1 += p; }
          else sB[i * LB + dj + kclip] = p;  // unique writer per (i, middle bucket)
        }
      }
    if (use_rpr) {
      lo0 += __shfl_xor_sync(0xffffffffu, lo0, 1); lo0 += __shfl_xor_sync(0xffffffffu, lo0, 2);
      hi0 += __shfl_xor_sync(0xffffffffu, hi0, 1); hi0 += __shfl_xor_sync(0xffffffffu, hi0, 2);
      lo1 += __shfl_xor_sync(0xffffffffu, lo1, 1); lo1 += __shfl_xor_sync(0xffffffffu, lo1, 2);
      hi1 += __shfl_xor_sync(0xffffffffu, hi1, 1); hi1 += __shfl_xor_sync(0xffffffffu, hi1, 2);
      if (tig == 0) {
        if (r0 < n) { sB[r0 * LB] = lo0; sB[r0 * LB + R - 1] = hi0; }
        if (r1 < n) { sB[r1 * LB] = lo1; sB[r1 * LB + R - 1] = hi1; }
      }
    }
    // ---- O = P V (P from registers as FP16 A fragments)
    float oc[DH / 8][4];
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) oc[t][0] = oc[t][1] = oc[t][2] = oc[t][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NT / 2; ++kk) {
      uint32_t af[4];
      af[0] = pack_h2(sc[2 * kk][0], sc[2 * kk][1]);
      af[1] = pack_h2(sc[2 * kk][2], sc[2 * kk][3]);
      af[2] = pack_h2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
      af[3] = pack_h2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 16) {
        uint32_t bf[4];  // .trans: (j0,c0) (j0+8,c0) (j0,c0+8) (j0+8,c0+8)
        const int mi = lane >> 3, rr = lane & 7;
        ldsm_x4_t(bf, sV + (kk * 16 + (mi & 1) * 8 + rr) * LDH + c0 + (mi >> 1) * 8);
        mma16816(oc[c0 / 8], af, bf[0], bf[1]);
        mma16816(oc[c0 / 8 + 1], af, bf[2], bf[3]);
      }
    }
    __syncwarp();
    // ---- + sum_r B_ir A^V[r][c], store (rows >= n written as 0)
    __half* orow0 = out + ((size_t)b * S + r0) * d + h * DH;
    __half* orow1 = out + ((size_t)b * S + r1) * d + h * DH;
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) {
      const int c = t * 8 + 2 * tig;
      float o00 = oc[t][0], o01 = oc[t][1], o10 = oc[t][2], o11 = oc[t][3];
      if (use_rpr) {
        for (int r = 0; r < R; ++r) {
          const float b0 = r0 < n ? sB[r0 * LB + r] : 0.f, b1 = r1 < n ? sB[r1 * LB + r] : 0.f;
          const float a0 = sAV[r * DH + c], a1 = sAV[r * DH + c + 1];
          o00 = fmaf(b0, a0, o00); o01 = fmaf(b0, a1, o01);
          o10 = fmaf(b1, a0, o10); o11 = fmaf(b1, a1, o11);
        }
      }
      if (r0 < S)
        *reinterpret_cast<__half2*>(orow0 + c) =
            r0 < n ? __floats2half2_rn(o00, o01) : __floats2half2_rn(0.f, 0.f);
      if (r1 < S)
        *reinterpret_cast<__half2*>(orow1 + c) =
            r1 < n ? __floats2half2_rn(o10, o11) : __floats2half2_rn(0.f, 0.f);
    }
  }
  // query rows beyond the last 16-block are padding: zero them
  for (int idx = nblk * 16 * DH + tid; idx < S * DH; idx += 128) {
    const int i = idx / DH, c = idx - i * DH;
    out[((size_t)b * S + i) * d + h * DH + c] = __float2half(0.f);
  }
}

template <int DH>
void launch_enc_mma(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                    __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  const int sp = (S + 15) / 16 * 16;
  auto smem_for = [](int SP) {
    return (size_t)3 * SP * (DH + 8) * 2 + 32 * (2 * DH + 1) * 4 + 2 * SP * 33 * 4;
  };
#define NMT_EM(NTV)                                                                          \
  {                                                                                          \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      NMT_CUDA(cudaFuncSetAttribute(k_attn_enc_mma<DH, NTV>,                                \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
      attr = true;                                                                           \
    }                                                                                        \
    k_attn_enc_mma<DH, NTV><<<dim3(B, H), 128, smem_for(NTV * 8), s>>>(qkv, len, relk, relv, \
                                                                      out, S, d, kclip,       \
                                                                      use_rpr);               \
  }
  if (sp <= 16) NMT_EM(2)
  else if (sp <= 32) NMT_EM(4)
  else if (sp <= 48) NMT_EM(6)
  else if (sp <= 64) NMT_EM(8)
  else if (sp <= 80) NMT_EM(10)
  else if (sp <= 96) NMT_EM(12)
  else if (sp <= 112) NMT_EM(14)
  else if (sp <= 128) NMT_EM(16)
  else throw CudaError("attn_encoder: S > 128");
#undef NMT_EM
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

// o[0..8) = sum_{j < n} p[j] * V[j][c0 .. c0+8) for this lane's 8-channel group (lanes
// 0..DH/8-1 hold the result).  G = DH/8 lanes share a value row (one 16-B load each), a
// warp covers 32/G rows per iteration; the row groups are combined by xor-shuffles.
// Row j lives in slot (anc_row && j < t_own ? anc_row[j] : own_slot): beam hypotheses read
// their ancestors' cached positions through the ancestry table (no K/V copies).
template <class T, int DH>
__device__ __forceinline__ void pv_accumulate(const float* __restrict__ p,
                                              const T* __restrict__ v0, size_t slot_stride,
                                              int own_slot, const int* __restrict__ anc_row,
                                              int t_own, int stride, int n, int lane, float* o) {
  constexpr int G = DH / 8, KP = 32 / G;
  const int sub = lane % G, kq = lane / G;
  float a[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) a[e] = 0.f;
#pragma unroll 2
  for (int j0 = 0; j0 < n; j0 += KP) {
    const int j = j0 + kq;
    if (j < n) {
      float v[8];
      const int sl = (anc_row && j < t_own) ? anc_row[j] : own_slot;
      Vec8<T>::load(v0 + (size_t)sl * slot_stride + (size_t)j * stride + sub * 8, v);
      const float pj = p[j];
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = fmaf(pj, v[e], a[e]);
    }
  }
#pragma unroll
  for (int off = G; off < 32; off <<= 1)
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += __shfl_xor_sync(0xffffffffu, a[e], off);
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = a[e];
}

// ----------------------------------------------------------------- decoder self-attention
// One warp per (live row, head) at step t = *d_t: k_t, v_t are appended to the cache slot,
// then positions 0..t are attended; only buckets 0..k occur (j <= t) and every
// j <= t - k falls in bucket 0.
template <class T, int DH>
__global__ void __launch_bounds__(128) k_attn_dec_self(
    const T* __restrict__ qkv, T* __restrict__ kc, T* __restrict__ vc, int Tmax,
    const int* __restrict__ row_slot, const T* __restrict__ relk, const T* __restrict__ relv,
    T* __restrict__ out, int rows, int d, int H, int kclip, int use_rpr, const int* __restrict__ d_t,
    const int* __restrict__ dR, const int* __restrict__ anc) {
  extern __shared__ float sm[];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw - (gw / H) * H;
  if (row >= min(rows, *dR)) return;
  const int t = *d_t;
  float* q = sm + warp * (DH + 32 + Tmax);
  float* x = q + DH;   // q . A^K[r], then bucket sums
  float* p = x + 32;
  const int slot = row_slot[row];
  const T* src = qkv + (size_t)row * 3 * d + h * DH;
  T* kbase = kc + (size_t)slot * Tmax * d + h * DH;
  T* vbase = vc + (size_t)slot * Tmax * d + h * DH;
  for (int c = lane; c < DH; c += 32) {
    q[c] = to_f(src[c]);
    kbase[(size_t)t * d + c] = src[d + c];        // KV-cache append
    vbase[(size_t)t * d + c] = src[2 * d + c];
  }
  __syncwarp();
  if (use_rpr && lane <= kclip) {
    float a = 0.f;
#pragma unroll 8
    for (int c = 0; c < DH; ++c) a = fmaf(q[c], to_f(relk[lane * DH + c]), a);
    x[lane] = a;
  }
  __syncwarp();
  const float scale = rsqrtf((float)DH);
  float mx = -INFINITY;
  const int* anc_row = anc ? anc + (size_t)slot * Tmax : nullptr;
  for (int j = lane; j <= t; j += 32) {
    const int sl = (anc_row && j < t) ? anc_row[j] : slot;
    const T* kr = kc + ((size_t)sl * Tmax + j) * d + h * DH;
    float e0 = 0.f, e1 = 0.f;
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      float f[8];
      Vec8<T>::load(kr + c, f);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        e0 = fmaf(f[u], q[c + u], e0);
        e1 = fmaf(f[u + 1], q[c + u + 1], e1);
      }
    }
    float e = e0 + e1;
    if (use_rpr) e += x[max(j - t, -kclip) + kclip];
    e *= scale;
    p[j] = e;
    mx = fmaxf(mx, e);
  }
  mx = warp_max(mx);
  float sum = 0.f, lo = 0.f;
  for (int j = lane; j <= t; j += 32) {
    const float e = __expf(p[j] - mx);
    p[j] = e;
    sum += e;
    if (j <= t - kclip) lo += e;
  }
  const float inv = 1.f / warp_sum(sum);
  lo = warp_sum(lo);
  __syncwarp();
  if (use_rpr) {
    if (lane <= kclip) {
      float bsum;
      if (lane == 0) bsum = lo;
      else {
        const int j = t - kclip + lane;
        bsum = j >= 0 ? p[j] : 0.f;
      }
      x[lane] = bsum;  // (unnormalised)
    }
    __syncwarp();
  }
  float o[8];
  pv_accumulate<T, DH>(p, vc + h * DH, (size_t)Tmax * d, slot, anc_row, t, d, t + 1, lane, o);
  constexpr int G = DH / 8;
  if (lane < G) {
    const int c0 = lane * 8;
    if (use_rpr)
      for (int b = 0; b <= kclip; ++b) {
        float rv[8];
        Vec8<T>::load(relv + b * DH + c0, rv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = fmaf(x[b], rv[e], o[e]);
      }
    T* orow = out + (size_t)row * d + h * DH + c0;
#pragma unroll
    for (int e = 0; e < 8; ++e) orow[e] = from_f<T>(o[e] * inv);
  }
}

template <class T>
void attn_decoder_self(const T* qkv, T* kc, T* vc, int Tmax, const int* row_slot, const T* relk,
                       const T* relv, T* out, int rows, int d, int H, int kclip, int use_rpr,
                       const int* d_t, const int* dR, const int* anc, cudaStream_t s) {
  if (rows <= 0) return;
  const int nw = 4, dh = d / H;
  size_t smem = sizeof(float) * nw * (dh + 32 + Tmax);
  dim3 grid(ceil_div(rows * H, nw));
#define NMT_DS(DH)                                                                             \
  launch_k(k_attn_dec_self<T, DH>, grid, nw * 32, smem, s, qkv, kc, vc, Tmax, row_slot, relk, \
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
// One warp per (live row, head); keys at ckv + (slot*S + j)*ldkv + koff + h*dh, values at
// + voff; mask j < src_len[slot].  S = *dS (device) so a captured step graph serves every
// batch; Smax sizes shared memory.
template <class T, int DH>
__global__ void __launch_bounds__(128) k_attn_cross(
    const T* __restrict__ qb, const T* __restrict__ ckv, int ldkv, int koff, int voff,
    const int* __restrict__ dS, int Smax, const int* __restrict__ src_len,
    const int* __restrict__ row_slot, T* __restrict__ out, int rows, int d, int H,
    const int* __restrict__ dR, int beam) {
  extern __shared__ float sm[];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const int row = gw / H, h = gw - (gw / H) * H;
  if (row >= min(rows, *dR)) return;
  const int S = *dS;
  float* q = sm + warp * (DH + Smax);
  float* p = q + DH;
  const int slot = row_slot[row] / beam;  // sentence slot (beam rows share the encoder K/V)
  const int n = src_len[slot];
  for (int c = lane; c < DH; c += 32) q[c] = to_f(qb[(size_t)row * d + h * DH + c]);
  __syncwarp();
  const float scale = rsqrtf((float)DH);
  const T* base = ckv + (size_t)slot * S * ldkv + h * DH;
  float mx = -INFINITY;
  for (int j = lane; j < n; j += 32) {
    const T* kr = base + (size_t)j * ldkv + koff;
    float e0 = 0.f, e1 = 0.f;
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      float f[8];
      Vec8<T>::load(kr + c, f);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        e0 = fmaf(f[u], q[c + u], e0);
        e1 = fmaf(f[u + 1], q[c + u + 1], e1);
      }
    }
    const float e = (e0 + e1) * scale;
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
  __syncwarp();
  float o[8];
  pv_accumulate<T, DH>(p, base + voff, 0, 0, nullptr, 0, ldkv, n, lane, o);
  constexpr int G = DH / 8;
  if (lane < G) {
    T* orow = out + (size_t)row * d + h * DH + lane * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) orow[e] = from_f<T>(o[e] * inv);
  }
}

template <class T>
void attn_cross(const T* q, const T* ckv, int ldkv, int koff, int voff, const int* dS, int Smax,
                const int* src_len, const int* row_slot, T* out, int rows, int d, int H,
                const int* dR, int beam, cudaStream_t s) {
  if (rows <= 0) return;
  const int nw = 4, dh = d / H;
  size_t smem = sizeof(float) * nw * (dh + Smax);
  dim3 grid(ceil_div(rows * H, nw));
#define NMT_CS(DH)                                                                          \
  launch_k(k_attn_cross<T, DH>, grid, nw * 32, smem, s, q, ckv, ldkv, koff, voff, dS, Smax, \
           src_len, row_slot, out, rows, d, H, dR, beam)
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
