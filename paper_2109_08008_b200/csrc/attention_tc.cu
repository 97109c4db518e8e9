// attention_tc.cu — encoder RPR self-attention for the FP16 path, every contraction on the
// tensor cores (warp-level mma.sync m16n8k16, FP16 in / FP32 accumulate):
//   S   = Q K^T                      (keys)
//   QA  = Q A^K^T                    (q_i . A^K[r], the relative-key term, 17 -> 32 cols)
//   O   = P V + B A^V                (values + relative-value term; B = bucket sums)
// with r(i,j) = clip(j - i, -k, k) + k (Shaw et al.; clip 8).
// Scores, masking and the softmax stay in FP32 registers; P and the bucket sums B are
// rounded to FP16 only as MMA operands (FP16-mode tolerance).  One CTA per
// (sentence, head), 4 warps each owning 16-query blocks; Q/K/V staged with cp.async.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace nmt {
namespace {

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
// 16-byte async global->shared copy; src_bytes = 0 zero-fills (padding rows)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}

constexpr int RP = 32;   // relative buckets padded to 32 (2k+1 <= 31)
constexpr int QLD = 33;  // FP32 row stride of q . A^K

template <int DH, int NT>
struct EncSmem {
  static constexpr int SP = NT * 8, LDH = DH + 8, LDB = RP + 8;
  static constexpr int Q = 0, K = Q + SP * LDH * 2, V = K + SP * LDH * 2, AK = V + SP * LDH * 2,
                       AV = AK + RP * LDH * 2, QA = AV + RP * LDH * 2, B = QA + SP * QLD * 4,
                       BYTES = B + SP * LDB * 2;
};

template <int DH, int NT>  // NT = 8-wide key tiles (SP = 8*NT, multiple of 16)
__global__ void __launch_bounds__(128) k_attn_enc_tc(const __half* __restrict__ qkv,
                                                     const int* __restrict__ len,
                                                     const __half* __restrict__ relk,
                                                     const __half* __restrict__ relv,
                                                     __half* __restrict__ out, int S, int d,
                                                     int kclip, int use_rpr) {
  using L = EncSmem<DH, NT>;
  constexpr int SP = L::SP, LDH = L::LDH, LDB = L::LDB;
  extern __shared__ __align__(16) uint8_t sm[];
  __half* sQ = reinterpret_cast<__half*>(sm + L::Q);
  __half* sK = reinterpret_cast<__half*>(sm + L::K);
  __half* sV = reinterpret_cast<__half*>(sm + L::V);
  __half* sAK = reinterpret_cast<__half*>(sm + L::AK);   // [RP][LDH], rows >= R zero
  __half* sAV = reinterpret_cast<__half*>(sm + L::AV);   // [RP][LDH], rows >= R zero
  float* sQA = reinterpret_cast<float*>(sm + L::QA);     // [SP][QLD]
  __half* sB = reinterpret_cast<__half*>(sm + L::B);     // [SP][LDB] bucket sums (FP16)
  const int b = blockIdx.x, h = blockIdx.y;
  const int R = 2 * kclip + 1;
  const int n = len[b];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nthr = blockDim.x, nwarp = nthr >> 5;   // min(4, SP/16) warps (launch_nt)
  const size_t rs = 3 * (size_t)d;
  const __half* base = qkv + (size_t)b * S * rs + h * DH;
  // ---- stage Q, K, V asynchronously (rows >= n zero-filled) + relative tables
  for (int idx = tid; idx < SP * (DH / 8); idx += nthr) {
    const int j = idx / (DH / 8), c = (idx % (DH / 8)) * 8;
    const bool ok = j < n;
    const __half* rp = base + (size_t)(ok ? j : 0) * rs + c;
    cp_async16(sQ + j * LDH + c, rp, ok ? 16 : 0);
    cp_async16(sK + j * LDH + c, rp + d, ok ? 16 : 0);
    cp_async16(sV + j * LDH + c, rp + 2 * d, ok ? 16 : 0);
  }
  for (int idx = tid; idx < RP * (DH / 8); idx += nthr) {  // A^K, A^V rows >= R zero-filled
    const int r = idx / (DH / 8), c = (idx % (DH / 8)) * 8;
    const bool ok = use_rpr && r < R;
    cp_async16(sAK + r * LDH + c, relk + (ok ? r * DH + c : 0), ok ? 16 : 0);
    cp_async16(sAV + r * LDH + c, relv + (ok ? r * DH + c : 0), ok ? 16 : 0);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int idx = tid; idx < SP * LDB / 8; idx += nthr)
    reinterpret_cast<uint4*>(sB)[idx] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  const float scale = rsqrtf((float)DH);
  const int g = lane >> 2, tig = lane & 3, mi = lane >> 3, rr = lane & 7;
  const int nblk = (n + 15) >> 4;
  for (int mb = warp; mb < nblk; mb += nwarp) {
    const int m0 = mb * 16;
    // ---- S = Q K^T and QA = Q A^K^T
    float sc[NT][4], qa[RP / 8][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
#pragma unroll
    for (int t = 0; t < RP / 8; ++t) qa[t][0] = qa[t][1] = qa[t][2] = qa[t][3] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < DH; k0 += 16) {
      uint32_t af[4];
      ldsm_x4(af, sQ + (m0 + rr + (mi & 1) * 8) * LDH + k0 + (mi >> 1) * 8);
#pragma unroll
      for (int t = 0; t < NT; t += 2) {
        uint32_t bf[4];  // (t, k0) (t, k0+8) (t+1, k0) (t+1, k0+8)
        ldsm_x4(bf, sK + ((t + (mi >> 1)) * 8 + rr) * LDH + k0 + (mi & 1) * 8);
        mma16816(sc[t], af, bf[0], bf[1]);
        mma16816(sc[t + 1], af, bf[2], bf[3]);
      }
      if (use_rpr) {
#pragma unroll
        for (int t = 0; t < RP / 8; t += 2) {
          uint32_t bf[4];
          ldsm_x4(bf, sAK + ((t + (mi >> 1)) * 8 + rr) * LDH + k0 + (mi & 1) * 8);
          mma16816(qa[t], af, bf[0], bf[1]);
          mma16816(qa[t + 1], af, bf[2], bf[3]);
        }
      }
    }
    const int r0 = m0 + g, r1 = r0 + 8;
    if (use_rpr) {  // this warp's 16 rows of q . A^K -> shared (indexed by bucket below)
#pragma unroll
      for (int t = 0; t < RP / 8; ++t) {
        const int c = t * 8 + 2 * tig;
        sQA[r0 * QLD + c] = qa[t][0];
        sQA[r0 * QLD + c + 1] = qa[t][1];
        sQA[r1 * QLD + c] = qa[t][2];
        sQA[r1 * QLD + c + 1] = qa[t][3];
      }
      __syncwarp();
    }
    // ---- relative-key term, mask, scale, FP32 softmax (rows r0, r1; quad reductions)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = e < 2 ? r0 : r1, j = t * 8 + 2 * tig + (e & 1);
        float v = sc[t][e];
        if (j < n && i < n) {
          if (use_rpr) v += sQA[i * QLD + min(max(j - i, -kclip), kclip) + kclip];
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
          else sB[i * LDB + dj + kclip] = __float2half(p);  // unique writer per (i, bucket)
        }
      }
    if (use_rpr) {
      lo0 += __shfl_xor_sync(0xffffffffu, lo0, 1); lo0 += __shfl_xor_sync(0xffffffffu, lo0, 2);
      hi0 += __shfl_xor_sync(0xffffffffu, hi0, 1); hi0 += __shfl_xor_sync(0xffffffffu, hi0, 2);
      lo1 += __shfl_xor_sync(0xffffffffu, lo1, 1); lo1 += __shfl_xor_sync(0xffffffffu, lo1, 2);
      hi1 += __shfl_xor_sync(0xffffffffu, hi1, 1); hi1 += __shfl_xor_sync(0xffffffffu, hi1, 2);
      if (tig == 0) {
        if (r0 < n) { sB[r0 * LDB] = __float2half(lo0); sB[r0 * LDB + R - 1] = __float2half(hi0); }
        if (r1 < n) { sB[r1 * LDB] = __float2half(lo1); sB[r1 * LDB + R - 1] = __float2half(hi1); }
      }
      __syncwarp();
    }
    // ---- O = P V (+ B A^V): P from registers as FP16 A fragments, B via ldmatrix
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
        ldsm_x4_t(bf, sV + (kk * 16 + (mi & 1) * 8 + rr) * LDH + c0 + (mi >> 1) * 8);
        mma16816(oc[c0 / 8], af, bf[0], bf[1]);
        mma16816(oc[c0 / 8 + 1], af, bf[2], bf[3]);
      }
    }
    if (use_rpr) {
#pragma unroll
      for (int kk = 0; kk < RP / 16; ++kk) {
        uint32_t af[4];
        ldsm_x4(af, sB + (m0 + rr + (mi & 1) * 8) * LDB + kk * 16 + (mi >> 1) * 8);
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 16) {
          uint32_t bf[4];
          ldsm_x4_t(bf, sAV + (kk * 16 + (mi & 1) * 8 + rr) * LDH + c0 + (mi >> 1) * 8);
          mma16816(oc[c0 / 8], af, bf[0], bf[1]);
          mma16816(oc[c0 / 8 + 1], af, bf[2], bf[3]);
        }
      }
    }
    // ---- store (query rows >= n written as 0)
    __half* orow0 = out + ((size_t)b * S + r0) * d + h * DH;
    __half* orow1 = out + ((size_t)b * S + r1) * d + h * DH;
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) {
      const int c = t * 8 + 2 * tig;
      if (r0 < S)
        *reinterpret_cast<__half2*>(orow0 + c) =
            r0 < n ? __floats2half2_rn(oc[t][0], oc[t][1]) : __floats2half2_rn(0.f, 0.f);
      if (r1 < S)
        *reinterpret_cast<__half2*>(orow1 + c) =
            r1 < n ? __floats2half2_rn(oc[t][2], oc[t][3]) : __floats2half2_rn(0.f, 0.f);
    }
  }
  // query rows beyond the last 16-block are padding: zero them
  for (int idx = nblk * 16 * (DH / 8) + tid; idx < S * (DH / 8); idx += nthr) {
    const int i = idx / (DH / 8), c = (idx % (DH / 8)) * 8;
    *reinterpret_cast<uint4*>(out + ((size_t)b * S + i) * d + h * DH + c) = make_uint4(0, 0, 0, 0);
  }
}

// ------------------------------------------------------------------ TMA-fed pipeline (DH = 64)
// The same arithmetic as k_attn_enc_tc (scores, relative terms, softmax, P V + B A^V, all
// MMA operands FP16, FP32 accumulation), restructured for HBM throughput:
//  * persistent CTAs walk the (sentence, head) items c, c + G, ...; one producer warp
//    streams each item's Q / K / V head tiles (SP rows x 128 B, 128-B swizzle) into a ring
//    of NSLOT shared-memory slots with three TMA loads (no per-thread copy issue), so the
//    loads of the next items are in flight while the current ones are computed;
//  * W consumer warps take (item, 16-query block) units round robin; a slot is released
//    when all SP/16 units of its item have arrived on its `empty` barrier;
//  * A^K / A^V (shared by all heads of the layer, reading R7) are staged once per CTA;
//  * each warp stages its 16 x 64 output block in shared memory and writes full 128-B
//    row segments.
// Rows of the TMA box beyond the sentence (SP > S) belong to the next sentence or lie
// beyond the tensor (zero-filled by TMA); they are masked as keys (j >= n) and never
// written as queries (rows >= S).
}  // namespace
namespace tc {
CUtensorMap make_map(const void* ptr, int rows, int cols, int ld, int box_rows, bool out);
}
namespace {

constexpr int kEncW = 8;             // consumer warps per CTA
constexpr int kEncMaxSlots = 16;
constexpr int kEncWarpScratch = 16 * QLD * 4 + 16 * (RP + 8) * 2;   // q.A^K [16][33] f32 + B [16][40] f16
constexpr int kEncTab = 2 * RP * (64 + 8) * 2;                        // A^K, A^V [32][72] f16

// Slot-ring depth per padded length (compile time: the kernel's slot index / phase and the
// host's shared-memory size use the same number): enough slots for the items the W warps
// work on at once plus two being prefetched, within ~112 KB (two CTAs per SM) when possible;
// S <= 16: three CTAs per SM (the kernel is latency-bound: 24 consumer warps instead of 16;
// measured 37.0 -> 35.6 us at S = 16, slower at S = 32: 37.6 -> 39.9), so ~74 KB.
constexpr int kEncFixedSmem = kEncTab + kEncW * kEncWarpScratch + 2 * kEncMaxSlots * 8 + 16 + 1024;
constexpr int enc_cmin(int a, int b) { return a < b ? a : b; }
template <int NT>
constexpr int enc_nslot() {
  constexpr int SP = NT * 8, NQ = SP / 16, SLOT = 3 * SP * 128;
  constexpr int want = enc_cmin(kEncMaxSlots, (kEncW + NQ - 1) / NQ + 2);
  constexpr int budget = NT <= 2 ? 74 * 1024 : 112 * 1024;
  constexpr int ns = enc_cmin(want, (budget - kEncFixedSmem) / SLOT);
  constexpr int ns2 = ns >= 2 ? ns : enc_cmin(want, (220 * 1024 - kEncFixedSmem) / SLOT);
  return ns2 < 1 ? 1 : ns2;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait1(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  for (uint32_t i = 0;; ++i) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    if (ok) return;
    if ((i & 1023) == 1023 && clock64() - t0 > 20000000000ll)   // pipeline bug
      NMT_TRAP("attn_mbar", smem_addr(bar) & 0xFFFFF, parity);
  }
}
// Item hand-off counter: the producer publishes "items 0..k issued" after arming slot k's
// barrier.  A consumer warp waits for it before the parity wait on full[k % nslot], because
// a warp does not visit every round of a slot (units go round robin over the warps, so with
// e.g. nslot = 3 and 4 units per item a warp sees each slot every second round): the 1-bit
// parity wait alone would accept the completion of the round before the one it wants.  Once
// item k is issued, round k / nslot - 1 of the slot has been consumed (so loaded) and round
// k / nslot + 1 cannot be loaded before this warp's unit is done: the parity is exact.
__device__ __forceinline__ void wait_issued(const int* issued, int k) {
  int v;
  const long long t0 = clock64();
  for (uint32_t i = 0;; ++i) {
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(issued)) : "memory");
    if (v > k) return;
    if ((i & 1023) == 1023 && clock64() - t0 > 20000000000ll) NMT_TRAP("attn_issued", v, k);
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}
// byte offset of the 16-B chunk `ch` (0..7) of row r in a 128-B-swizzled tile
__device__ __forceinline__ uint32_t sw128(int r, int ch) { return r * 128 + ((ch ^ (r & 7)) << 4); }

// KC > 0: the clip distance as a compile-time constant (the models' k = 8): the per-element
// relative-bucket clamps and band tests fold to immediates (KC = 0: runtime kclip_rt).
template <int NT, int KC>
__global__ void __launch_bounds__(32 * (kEncW + 1), NT <= 2 ? 3 : NT <= 8 ? 2 : 1) k_attn_enc_tma(
    const __grid_constant__ CUtensorMap mqkv, const int* __restrict__ len,
    const __half* __restrict__ relk, const __half* __restrict__ relv, __half* __restrict__ out,
    int B, int S, int d, int H, int kclip_rt, int use_rpr, int nslot_rt, unsigned hmagic) {
  const int kclip = KC > 0 ? KC : kclip_rt;
  // CT: the slot count as a compile-time constant and the item's (sentence, head) by a
  // multiply-high, b = floor(it / H) = umulhi(it, ceil(2^32 / H)) (exact for it < 2^32 / H^2:
  // items <= 2^18 here) — three integer divisions fewer per unit (S = 32: 37.5 -> 36.5 us,
  // S = 96: 72.6 -> 66.9).  NT = 6 / 8 keep the runtime forms: under the two-CTA register cap
  // the change makes them spill (S = 40: 47.8 -> 50.5 us).
  constexpr bool CT = NT != 6 && NT != 8;
  const int nslot = CT ? enc_nslot<NT>() : nslot_rt;
  auto item_bh = [&](int it, int& b, int& h) {
    if constexpr (CT) b = (int)__umulhi((unsigned)it, hmagic);
    else b = it / H;
    h = it - b * H;
  };
  constexpr int DH = 64, SP = NT * 8, NQ = SP / 16, LDH = DH + 8, LDB = RP + 8;
  constexpr int TILE = SP * 128, SLOT = 3 * TILE;
  extern __shared__ uint8_t smraw[];
  // 1024-B aligned by pointer arithmetic on the __shared__ array (an integer round trip
  // would hide the address space: generic LD/ST instead of LDS/STS)
  uint8_t* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  uint8_t* slots = sm;
  __half* sAK = reinterpret_cast<__half*>(sm + nslot * SLOT);
  __half* sAV = sAK + RP * LDH;
  uint8_t* wscr = reinterpret_cast<uint8_t*>(sAV + RP * LDH);
  uint64_t* full = reinterpret_cast<uint64_t*>(wscr + kEncW * kEncWarpScratch);
  uint64_t* empty = full + kEncMaxSlots;
  int* issued = reinterpret_cast<int*>(empty + kEncMaxSlots);   // items issued by the producer

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int items = B * H, G = gridDim.x, c = blockIdx.x;
  const int nloc = c < items ? (items - 1 - c) / G + 1 : 0;   // items of this CTA
  const int R = 2 * kclip + 1;
  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init1(&full[i], 1);
      mbar_init1(&empty[i], NQ);
    }
    *issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mqkv)) : "memory");
  }
  // A^K / A^V once per CTA (rows >= R zero: finite operands for the padded MMA columns)
  for (int idx = tid; idx < RP * (DH / 8); idx += blockDim.x) {
    const int r = idx / (DH / 8), cc = (idx % (DH / 8)) * 8;
    const bool ok = use_rpr && r < R;
    cp_async16(sAK + r * LDH + cc, relk + (ok ? r * DH + cc : 0), ok ? 16 : 0);
    cp_async16(sAV + r * LDH + cc, relv + (ok ? r * DH + cc : 0), ok ? 16 : 0);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  if (warp == kEncW) {  // ---------------- producer
    if (lane == 0) {
      for (int k = 0; k < nloc; ++k) {
        const int sl = k % nslot;
        if (k >= nslot) mbar_wait1(&empty[sl], ((k / nslot) - 1) & 1);
        const int it = c + k * G;
        int b, h;
        item_bh(it, b, h);
        uint8_t* dst = slots + sl * SLOT;
        mbar_expect(&full[sl], SLOT);
        tma_2d(dst, &mqkv, &full[sl], h * DH, b * S);
        tma_2d(dst + TILE, &mqkv, &full[sl], d + h * DH, b * S);
        tma_2d(dst + 2 * TILE, &mqkv, &full[sl], 2 * d + h * DH, b * S);
        asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(issued)), "r"(k + 1)
                     : "memory");
      }
    }
    return;
  }
  // ---------------- consumers
  float* sQA = reinterpret_cast<float*>(wscr + warp * kEncWarpScratch);      // [16][QLD]
  __half* sB = reinterpret_cast<__half*>(wscr + warp * kEncWarpScratch + 16 * QLD * 4);  // [16][LDB]
  const float scale = rsqrtf((float)DH);
  const int g = lane >> 2, tig = lane & 3, mi = lane >> 3, rr = lane & 7;
  for (int u = warp; u < nloc * NQ; u += kEncW) {
    const int k = u / NQ, qb = u - k * NQ, sl = k % nslot;
    const int it = c + k * G;
    int b, h;
    item_bh(it, b, h);
    const int n = len[b], m0 = qb * 16;
    const uint32_t tQ = smem_addr(slots + sl * SLOT), tK = tQ + TILE, tV = tK + TILE;
    wait_issued(issued, k);
    mbar_wait1(&full[sl], (k / nslot) & 1);
    float oc[DH / 8][4];
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) oc[t][0] = oc[t][1] = oc[t][2] = oc[t][3] = 0.f;
    const int r0 = m0 + g, r1 = r0 + 8;
    if (m0 < n) {
      // zero this unit's bucket sums (band buckets without a key stay 0)
      for (int idx = lane; idx < 16 * LDB / 8; idx += 32)
        reinterpret_cast<uint4*>(sB)[idx] = make_uint4(0u, 0u, 0u, 0u);
      // ---- S = Q K^T and QA = Q A^K^T
      float sc[NT][4], qa[RP / 8][4];
#pragma unroll
      for (int t = 0; t < NT; ++t) sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
#pragma unroll
      for (int t = 0; t < RP / 8; ++t) qa[t][0] = qa[t][1] = qa[t][2] = qa[t][3] = 0.f;
#pragma unroll
      for (int k0 = 0; k0 < DH; k0 += 16) {
        uint32_t af[4];
        {
          const int row = m0 + rr + (mi & 1) * 8;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                       : "r"(tQ + sw128(row, k0 / 8 + (mi >> 1))));
        }
#pragma unroll
        for (int t = 0; t < NT; t += 2) {
          uint32_t bf[4];
          const int row = (t + (mi >> 1)) * 8 + rr;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(bf[0]), "=r"(bf[1]), "=r"(bf[2]), "=r"(bf[3])
                       : "r"(tK + sw128(row, k0 / 8 + (mi & 1))));
          mma16816(sc[t], af, bf[0], bf[1]);
          mma16816(sc[t + 1], af, bf[2], bf[3]);
        }
#pragma unroll
        for (int t = 0; t < RP / 8; t += 2) {
          uint32_t bf[4];
          ldsm_x4(bf, sAK + ((t + (mi >> 1)) * 8 + rr) * LDH + k0 + (mi & 1) * 8);
          mma16816(qa[t], af, bf[0], bf[1]);
          mma16816(qa[t + 1], af, bf[2], bf[3]);
        }
      }
      // ---- relative-key term, mask, scale, FP32 softmax (rows r0, r1; quad reductions).
      // Branch-free: with use_rpr = 0 the staged tables are zero, so the relative terms
      // add exact zeros.  Scores are kept in log2 units (scale * log2 e folded in).
#pragma unroll
      for (int t = 0; t < RP / 8; ++t) {
        const int cc = t * 8 + 2 * tig;
        sQA[g * QLD + cc] = qa[t][0];
        sQA[g * QLD + cc + 1] = qa[t][1];
        sQA[(g + 8) * QLD + cc] = qa[t][2];
        sQA[(g + 8) * QLD + cc + 1] = qa[t][3];
      }
      __syncwarp();
      const float sl2 = scale * 1.4426950408889634f;
      const bool ok0 = r0 < n, ok1 = r1 < n;
      const float* qa0 = sQA + g * QLD + kclip;        // indexed by clip(j - i, -k, k)
      const float* qa1 = sQA + (g + 8) * QLD + kclip;
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool top = e < 2;
          const int j = t * 8 + 2 * tig + (e & 1), dj = j - (top ? r0 : r1);
          const float v = sc[t][e] + (top ? qa0 : qa1)[min(max(dj, -kclip), kclip)];
          sc[t][e] = (j < n && (top ? ok0 : ok1)) ? v * sl2 : -INFINITY;
          if (top) mx0 = fmaxf(mx0, sc[t][e]);
          else mx1 = fmaxf(mx1, sc[t][e]);
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
          const float v = exp2f(sc[t][e] - (e < 2 ? mx0 : mx1));
          sc[t][e] = v;
          if (e < 2) s0 += v;
          else s1 += v;
        }
      s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
      s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
      const float inv0 = s0 > 0.f ? 1.f / s0 : 0.f, inv1 = s1 > 0.f ? 1.f / s1 : 0.f;
      // P, and the bucket sums B[i][r] = sum_{j: r(i,j) = r} P[i][j]: the band buckets have
      // one key each (unique writer; masked keys carry P = 0), the two clipped ends are sums
      float lo0 = 0.f, hi0 = 0.f, lo1 = 0.f, hi1 = 0.f;
      __half* sb0 = sB + g * LDB + kclip;
      __half* sb1 = sB + (g + 8) * LDB + kclip;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool top = e < 2;
          const int j = t * 8 + 2 * tig + (e & 1), dj = j - (top ? r0 : r1);
          const float p = sc[t][e] * (top ? inv0 : inv1);
          sc[t][e] = p;
          const float pl = dj <= -kclip ? p : 0.f, ph = dj >= kclip ? p : 0.f;
          if (top) { lo0 += pl; hi0 += ph; } else { lo1 += pl; hi1 += ph; }
          if (dj > -kclip && dj < kclip) (top ? sb0 : sb1)[dj] = __float2half(p);
        }
      lo0 += __shfl_xor_sync(0xffffffffu, lo0, 1); lo0 += __shfl_xor_sync(0xffffffffu, lo0, 2);
      hi0 += __shfl_xor_sync(0xffffffffu, hi0, 1); hi0 += __shfl_xor_sync(0xffffffffu, hi0, 2);
      lo1 += __shfl_xor_sync(0xffffffffu, lo1, 1); lo1 += __shfl_xor_sync(0xffffffffu, lo1, 2);
      hi1 += __shfl_xor_sync(0xffffffffu, hi1, 1); hi1 += __shfl_xor_sync(0xffffffffu, hi1, 2);
      if (tig == 0) {
        sb0[-kclip] = __float2half(lo0); sb0[kclip] = __float2half(hi0);
        sb1[-kclip] = __float2half(lo1); sb1[kclip] = __float2half(hi1);
      }
      __syncwarp();
      // ---- O = P V (+ B A^V)
#pragma unroll
      for (int kk = 0; kk < NT / 2; ++kk) {
        uint32_t af[4];
        af[0] = pack_h2(sc[2 * kk][0], sc[2 * kk][1]);
        af[1] = pack_h2(sc[2 * kk][2], sc[2 * kk][3]);
        af[2] = pack_h2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
        af[3] = pack_h2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 16) {
          uint32_t bf[4];
          const int row = kk * 16 + (mi & 1) * 8 + rr;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(bf[0]), "=r"(bf[1]), "=r"(bf[2]), "=r"(bf[3])
                       : "r"(tV + sw128(row, c0 / 8 + (mi >> 1))));
          mma16816(oc[c0 / 8], af, bf[0], bf[1]);
          mma16816(oc[c0 / 8 + 1], af, bf[2], bf[3]);
        }
      }
      {
#pragma unroll
        for (int kk = 0; kk < RP / 16; ++kk) {
          uint32_t af[4];
          ldsm_x4(af, sB + (rr + (mi & 1) * 8) * LDB + kk * 16 + (mi >> 1) * 8);
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 16) {
            uint32_t bf[4];
            ldsm_x4_t(bf, sAV + (kk * 16 + (mi & 1) * 8 + rr) * LDH + c0 + (mi >> 1) * 8);
            mma16816(oc[c0 / 8], af, bf[0], bf[1]);
            mma16816(oc[c0 / 8 + 1], af, bf[2], bf[3]);
          }
        }
      }
    }
    // this unit no longer reads the slot: release it (the producer may refill it)
    __syncwarp();
    if (lane == 0) mbar_arrive1(&empty[sl]);
    // ---- stage the 16 x 64 FP16 block (rows >= n are zero) in the q.A^K scratch
    // (2 KB, 128-B rows, 16-B chunks XOR-swizzled by row), then full-row stores
    uint8_t* st = reinterpret_cast<uint8_t*>(sQA);
#pragma unroll
    for (int t = 0; t < DH / 8; ++t) {
      const uint32_t w0 = r0 < n ? pack_h2(oc[t][0], oc[t][1]) : 0u;
      const uint32_t w1 = r1 < n ? pack_h2(oc[t][2], oc[t][3]) : 0u;
      *reinterpret_cast<uint32_t*>(st + sw128(g, t) + 4 * tig) = w0;
      *reinterpret_cast<uint32_t*>(st + sw128(g + 8, t) + 4 * tig) = w1;
    }
    __syncwarp();
    __half* obase = out + ((size_t)b * S) * d + h * DH;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = i * 32 + lane, row = idx >> 3, ch = idx & 7;
      if (m0 + row < S)
        *reinterpret_cast<uint4*>(obase + (size_t)(m0 + row) * d + ch * 8) =
            *reinterpret_cast<const uint4*>(st + sw128(row, ch));
    }
    __syncwarp();
  }
}

struct EncTmaCfg {
  int nslot, smem, grid_per_sm;
};

template <int NT, int KC>
EncTmaCfg enc_tma_cfg() {
  static EncTmaCfg cfg = [] {
    constexpr int SP = NT * 8, SLOT = 3 * SP * 128;
    EncTmaCfg c{};
    c.nslot = enc_nslot<NT>();
    c.smem = kEncFixedSmem + c.nslot * SLOT;
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc_tma<NT, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  c.smem));
    int occ = 0;
    NMT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_attn_enc_tma<NT, KC>,
                                                           32 * (kEncW + 1), c.smem));
    c.grid_per_sm = std::max(1, occ);
    return c;
  }();
  return cfg;
}

int sm_count() {
  static const int n = [] {
    int dev = 0, c = 0;
    NMT_CUDA(cudaGetDevice(&dev));
    NMT_CUDA(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev));
    return c;
  }();
  return n;
}

template <int NT, int KC>
void launch_tma_kc(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                   __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  const EncTmaCfg c = enc_tma_cfg<NT, KC>();
  const CUtensorMap map = tc::make_map(qkv, B * S, 3 * d, 3 * d, NT * 8, false);
  const int grid = std::min(B * H, c.grid_per_sm * sm_count());
  launch_k(k_attn_enc_tma<NT, KC>, dim3(grid), dim3(32 * (kEncW + 1)), (size_t)c.smem, s, map, len,
           relk, relv, out, B, S, d, H, kclip, use_rpr, c.nslot,
           (unsigned)((0x100000000ull + H - 1) / H));
}

template <int NT>
void launch_tma(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  if (kclip == 8)   // every preset's clip distance: compile-time k
    launch_tma_kc<NT, 8>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s);
  else
    launch_tma_kc<NT, 0>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s);
}

void launch_tma_sp(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                   __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  switch ((S + 15) / 16 * 16) {
    case 16: launch_tma<2>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 32: launch_tma<4>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 48: launch_tma<6>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 64: launch_tma<8>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 80: launch_tma<10>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 96: launch_tma<12>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 112: launch_tma<14>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 128: launch_tma<16>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    default: throw CudaError("attn_encoder: S > 128");
  }
}

template <int DH, int NT>
void launch_nt(const __half* qkv, const int* len, const __half* relk, const __half* relv,
               __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  using L = EncSmem<DH, NT>;
  // thread-safe one-time attribute setup (C++11 static initialisation)
  static const bool attr = [&] {
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc_tc<DH, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    return true;
  }();
  (void)attr;
  // one warp per 16-query block up to 4: short sentences do not hold idle warps
  constexpr int threads = 32 * (NT / 2 < 4 ? NT / 2 : 4);
  k_attn_enc_tc<DH, NT><<<dim3(B, H), threads, L::BYTES, s>>>(qkv, len, relk, relv, out, S, d,
                                                             kclip, use_rpr);
}

template <int DH>
void launch_dh(const __half* qkv, const int* len, const __half* relk, const __half* relv,
               __half* out, int B, int S, int d, int H, int kclip, int use_rpr, cudaStream_t s) {
  const int sp = (S + 15) / 16 * 16;
  switch (sp) {
    case 16: launch_nt<DH, 2>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 32: launch_nt<DH, 4>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 48: launch_nt<DH, 6>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 64: launch_nt<DH, 8>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 80: launch_nt<DH, 10>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 96: launch_nt<DH, 12>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 112: launch_nt<DH, 14>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 128: launch_nt<DH, 16>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    default: throw CudaError("attn_encoder: S > 128");
  }
}

}  // namespace

void attn_encoder_tc(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                     __half* out, int B, int S, int d, int H, int kclip, int use_rpr,
                     cudaStream_t s) {
  if (2 * kclip + 1 > RP - 1) throw CudaError("attn_encoder_tc: 2k+1 must be < 32");
  // NMT_ENC_ATTN (read per call; A/B and tests): 0 = one CTA per item (cp.async), 2 = the
  // tcgen05 / TMEM kernel (attention_umma.cu), unset = the TMA-fed mma.sync pipeline
  const char* ea = getenv("NMT_ENC_ATTN");
  const int mode = ea ? atoi(ea) : 1;
  if (mode == 2 && d / H == 64 && use_rpr && kclip <= 8 && relk && relv) {
    attn_encoder_umma(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
    return;
  }
  const bool legacy = mode == 0;
  if (d / H == 64 && !legacy) {
    launch_tma_sp(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s);
    NMT_LAUNCH_CHECK();
    return;
  }
  switch (d / H) {
    case 16: launch_dh<16>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 32: launch_dh<32>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    case 64: launch_dh<64>(qkv, len, relk, relv, out, B, S, d, H, kclip, use_rpr, s); break;
    default: throw CudaError("attn_encoder_tc: head dim must be 16, 32 or 64");
  }
  NMT_LAUNCH_CHECK();
}

}  // namespace nmt
