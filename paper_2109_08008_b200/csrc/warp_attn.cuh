// warp_attn.cuh — one-warp attention for a single query (decoder self / cross attention):
// 8-channel lane slices, all key / value loads of a chunk in flight, online FP32 softmax.
// Shared by attention.cu and decode_fused.cu (CG = loads through L2 only, for data written
// earlier in the same launch by other SMs).
#pragma once
#include "common.cuh"

namespace nmt {

template <class T> struct Raw8;   // 8 consecutive elements in their storage type
__device__ __forceinline__ uint4 ld_cg16(const void* p) {   // L2 only: sees other SMs' writes
  uint4 u;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p));
  return u;
}
template <> struct Raw8<__half> {
  uint4 u;
  __device__ __forceinline__ void load(const __half* p) { u = *reinterpret_cast<const uint4*>(p); }
  __device__ __forceinline__ void load_cg(const __half* p) { u = ld_cg16(p); }
  __device__ __forceinline__ void store(__half* p) const { *reinterpret_cast<uint4*>(p) = u; }
  __device__ __forceinline__ void zero() { u = make_uint4(0u, 0u, 0u, 0u); }
  __device__ __forceinline__ void to_f(float* f) const {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __half22float2(h[e]);
      f[2 * e] = x.x;
      f[2 * e + 1] = x.y;
    }
  }
};
template <> struct Raw8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = reinterpret_cast<const float4*>(p)[0];
    b = reinterpret_cast<const float4*>(p)[1];
  }
  __device__ __forceinline__ void load_cg(const float* p) {
    const uint4 x = ld_cg16(p), y = ld_cg16(p + 4);
    a = make_float4(__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z), __uint_as_float(x.w));
    b = make_float4(__uint_as_float(y.x), __uint_as_float(y.y), __uint_as_float(y.z), __uint_as_float(y.w));
  }
  __device__ __forceinline__ void store(float* p) const {
    reinterpret_cast<float4*>(p)[0] = a;
    reinterpret_cast<float4*>(p)[1] = b;
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void to_f(float* f) const {
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

template <class T, int DH, bool CG = false>
struct WarpAttn {
  static constexpr int G = DH / 8, KP = 32 / G;
  // keys per lane per chunk: 4 for FP16 dh = 64 (16 keys in flight per warp, 32 registers of
  // raw K / V), small enough for 6 CTAs (24 warps) per SM
  static constexpr int U = sizeof(T) == 2 ? (G >= 2 ? G / 2 : 1) : (G >= 2 ? G / 2 : 1);
  static constexpr int CH = KP * U;
  int sub, kq;
  float q[8], m, l, acc[8];

  // q (this lane's 8 channels) pre-multiplied by 1/sqrt(dh)
  __device__ __forceinline__ void init(int lane, const T* qhead, float scale) {
    sub = lane % G;
    kq = lane / G;
    Raw8<T> r;
    if constexpr (CG) r.load_cg(qhead + sub * 8);
    else r.load(qhead + sub * 8);
    r.to_f(q);
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] *= scale, acc[e] = 0.f;
    m = -INFINITY;
    l = 0.f;
  }
  // q . x over the head, x given as this lane's 8 channels (all lanes must call)
  __device__ __forceinline__ float group_dot(const float* x) const {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      s0 = fmaf(q[e], x[e], s0);
      s1 = fmaf(q[e + 1], x[e + 1], s1);
    }
    float s = s0 + s1;
#pragma unroll
    for (int off = 1; off < G; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
  }
  // Keys [j0, j0 + CH) with j < n (requires j0 < n).  addr(j, kp, vp) sets the head-slice
  // pointers of key j; bias(j) is added to the scaled score; vadd(j, v) adds to v_j.
  // Keys j < nload (>= n, readable memory) are loaded: the loads need not wait for n.
  template <class ADDR, class BIAS, class VADD>
  __device__ __forceinline__ void chunk(int j0, int n, int nload, ADDR addr, BIAS bias, VADD vadd) {
    Raw8<T> kr[U], vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * KP + kq;
      if (j < nload) {
        const T *kp, *vp;
        addr(j, kp, vp);
        if constexpr (CG) {
          kr[u].load_cg(kp + sub * 8);
          vr[u].load_cg(vp + sub * 8);
        } else {
          kr[u].load(kp + sub * 8);
          vr[u].load(vp + sub * 8);
        }
      } else {
        kr[u].zero();
        vr[u].zero();
      }
    }
    float s[U], cm = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * KP + kq;
      float f[8];
      kr[u].to_f(f);
      const float e = group_dot(f);
      s[u] = j < n ? e + bias(j) : -INFINITY;
      cm = fmaxf(cm, s[u]);
    }
#pragma unroll
    for (int off = G; off < 32; off <<= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
    const float mn = fmaxf(m, cm);
    const float corr = __expf(m - mn);
    l *= corr;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= corr;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * KP + kq;
      if (j < n) {
        const float p = __expf(s[u] - mn);
        float f[8];
        vr[u].to_f(f);
        vadd(j, f);
        l += p;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(p, f[e], acc[e]);
      }
    }
    m = mn;
  }
  // Sum over the KP key groups; every lane ends with the normalised output of its channels.
  __device__ __forceinline__ void finish(float* o) {
#pragma unroll
    for (int off = G; off < 32; off <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
    }
    const float inv = 1.f / l;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = acc[e] * inv;
  }
};

template <class T>
__device__ __forceinline__ void store8(T* p, const float* o) {
  if constexpr (sizeof(T) == 2) {
    uint4 u;
    __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2half2_rn(o[2 * e], o[2 * e + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    reinterpret_cast<float4*>(p)[0] = make_float4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(o[4], o[5], o[6], o[7]);
  }
}


}  // namespace nmt
