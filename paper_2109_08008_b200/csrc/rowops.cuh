// rowops.cuh — row-wise device helpers shared by kernels.cu and decode_fused.cu: 16-B
// vector row I/O (lane owns E contiguous columns) and the warp LayerNorm (FP32 statistics,
// PAPER.md:123).  No kernels here.
#pragma once
#include "common.cuh"

namespace nmt {

// Vectorised variant: lane owns E contiguous columns [lane*E, lane*E + E) so every row
// access is 16-B vector loads/stores (one 1 KB row per warp-instruction pair at d = 512).
template <class T> struct VecIO;
template <> struct VecIO<__half> {
  static constexpr int W = 8;  // elements per 16 B
  static __device__ __forceinline__ void ld(const __half* p, float* f) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 x = __half22float2(h[e]);
      f[2 * e] = x.x;
      f[2 * e + 1] = x.y;
    }
  }
  static __device__ __forceinline__ void st(__half* p, const float* f) {
    uint4 u;
    __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __halves2half2(from_f<__half>(f[2 * e]), from_f<__half>(f[2 * e + 1]));
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct VecIO<float> {
  static constexpr int W = 4;
  static __device__ __forceinline__ void ld(const float* p, float* f) {
    float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  static __device__ __forceinline__ void st(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
};

template <class T, int E>
__device__ __forceinline__ void ldrow(const T* p, float* v) {
#pragma unroll
  for (int i = 0; i < E; i += VecIO<T>::W) VecIO<T>::ld(p + i, v + i);
}
// E contiguous elements of a row held raw (16-B vectors) until their fma into x.
template <class T, int E>
struct RawRow {
  static constexpr int NV = E * (int)sizeof(T) / 16;
  uint4 u[NV];
  __device__ __forceinline__ void load(const T* p) {
#pragma unroll
    for (int i = 0; i < NV; ++i) u[i] = reinterpret_cast<const uint4*>(p)[i];
  }
  __device__ __forceinline__ void fma_into(float wk, float* x) const {
    if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const __half2* h = reinterpret_cast<const __half2*>(&u[i]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h[e]);
          x[8 * i + 2 * e] = fmaf(wk, f.x, x[8 * i + 2 * e]);
          x[8 * i + 2 * e + 1] = fmaf(wk, f.y, x[8 * i + 2 * e + 1]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        x[4 * i] = fmaf(wk, __uint_as_float(u[i].x), x[4 * i]);
        x[4 * i + 1] = fmaf(wk, __uint_as_float(u[i].y), x[4 * i + 1]);
        x[4 * i + 2] = fmaf(wk, __uint_as_float(u[i].z), x[4 * i + 2]);
        x[4 * i + 3] = fmaf(wk, __uint_as_float(u[i].w), x[4 * i + 3]);
      }
    }
  }
};
template <class T, int E>
__device__ __forceinline__ void strow(T* p, const float* v) {
#pragma unroll
  for (int i = 0; i < E; i += VecIO<T>::W) VecIO<T>::st(p + i, v + i);
}
template <class T, int E>
__device__ __forceinline__ void ln_contig(float* v, int d, const T* g, const T* b, float eps,
                                          int lane) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < E; ++i) s += v[i];
  const float mu = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const float t = v[i] - mu;
    q += t * t;
  }
  const float rstd = rsqrtf(warp_sum(q) / d + eps);
  float gv[E], bv[E];
  ldrow<T, E>(g + lane * E, gv);
  ldrow<T, E>(b + lane * E, bv);
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = (v[i] - mu) * rstd * gv[i] + bv[i];
}


}  // namespace nmt
