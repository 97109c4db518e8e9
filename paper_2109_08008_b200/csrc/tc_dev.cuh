// tc_dev.cuh — tcgen05 / TMEM / TMA / mbarrier device helpers and the fused GEMM epilogue
// math (bias, residual, ReLU, folded LayerNorm, argmax packing), shared by gemm_tc.cu and
// decode_fused.cu.  Inline PTX for sm_100a only.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace nmt {
namespace tc {

constexpr int BM = 128;       // UMMA M (cta_group::1): one TMEM lane per output row
constexpr int BK = 64;        // 64 halves = 128 B = one swizzle-128B atom row
constexpr int UMMA_K = 16;    // K per tcgen05.mma for 16-bit inputs
constexpr int kThreads = 384;
constexpr int kBiasMax = 2048;   // bias vectors up to this length are staged whole per CTA  // warps 0-3: TMA / MMA / TMEM alloc / idle; 4-11: epilogue

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe (mbarrier.test_wait): for issuers that poll several barriers —
// try_wait may suspend the thread for a system-dependent time before failing.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (clean launch failure) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (mbar_try(bar, parity)) return;
    if ((i & 1023) == 0 && clock64() - t0 > 20000000000ll)
      NMT_TRAP("mbar_wait", smem_u32(bar) & 0xFFFFF, parity);
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// K-major, 128B-swizzled operand tile: rows of 128 B, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t make_desc_sw128(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) /*LBO (unused for SW128 K-major)*/ |
         ((1024ull >> 4) << 32) /*SBO*/ | (1ull << 46) /*sm100 version*/ |
         (2ull << 61) /*SWIZZLE_128B*/;
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// ---- thread-block cluster / CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(const void* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
// TMA into this CTA's shared memory, completion counted on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar,
                                                 int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// M = 256 MMA over the CTA pair: A rows 0-127 / 128-255 and B rows 0-N/2 / N/2-N from the
// two CTAs' shared memory at the same offsets; D rows split the same way over their TMEM.
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t a, uint64_t b,
                                             uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// arrive on the mbarrier at this offset in BOTH CTAs of the pair when the MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// Asynchronous variant: the registers are valid only after tmem_wait_ld (whose operands tie
// them to the wait) or, for further loads issued before that wait, tmem_touch after it.
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
#define NMT_R32(r)                                                                           \
  "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),        \
      "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), \
      "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),           \
      "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),           \
      "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
__device__ __forceinline__ void tmem_wait_ld(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : NMT_R32(r)::"memory");
}
__device__ __forceinline__ void tmem_touch(uint32_t* r) { asm volatile("" : NMT_R32(r)::"memory"); }
// Plain (coherent) load: the residual may alias the output (in-place x += f(x)).
__device__ __forceinline__ void load8h(const __half* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 x = __half22float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}

struct Params {
  int M, N, K;
  const __half* bias;
  const __half* R;
  int ldr;
  __half* C;
  int ldc;
  int relu;
  const int* dM;
  unsigned long long* argmax;
  float* logits;
  float* bpart;       // beam epilogue (logits never stored): per (row, HALF-column segment)
                      // {max, sum exp(x - max), top-8 values, top-8 ids} (kBeamRec floats)
  int splits;         // split-K factor (kb_total % splits == 0)
  float* ws;          // split-K partials [tile][split][BM][BN]
  int* counters;      // split-K arrival counters [tile] (self-resetting)
  int dbg;            // tuning experiments only (NMT_GEMM_DBG bits): 1 = drain TMEM only,
                      // 2 = no TMA stores, 4 = no staging / stores, 8 = no epilogue math,
                      // 32 = operand TMA only for the first STAGES k-blocks (MMA rate)
  int tstore;         // FP16 C written by TMA stores (mapC), see k_gemm_tc
  int rtma;           // residual 32 x 32 blocks TMA-loaded into the staging tiles (mapR)
  int bpre;           // first-unit weight tiles requested before the PDL wait
  int trace;          // NMT_GEMM_TRACE: per (CTA, local unit < 32) globaltimer stamps (g_gemm_trace)
  int nfast;          // unit order: 1 = column tiles of one row block on consecutive CTAs
                      // (the A row block is read from DRAM once and shared through L2)
  float2* st_out;     // LN folding, producer side (GemmArgs)
  const float2* ln_st;
  const float* ln_c;
  float ln_eps;
};

// (mean, M2) of 32 values as stored (FP16-rounded), two-pass in registers
__device__ __forceinline__ float2 chunk_stats(const float* v) {
  float r[32], s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const uint32_t h = pack_half2_sat(v[j], v[j + 1]);
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h));
    r[j] = f.x;
    r[j + 1] = f.y;
    s += f.x + f.y;
  }
  const float mu = s * (1.f / 32.f);
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) q = fmaf(r[j] - mu, r[j] - mu, q);
  return make_float2(mu, q);
}
// Row mean / rstd from NCH chunk partials of 32 columns each (Chan et al. merge of
// equal-size groups).  All partials are loaded at once (16-B vectors) before the merge.
template <int NCH>
__device__ __forceinline__ float2 merge_stats_n(const float2* st, float eps) {
  float4 q[NCH / 2];
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) q[i] = reinterpret_cast<const float4*>(st)[i];
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) sm += q[i].x + q[i].z;
  const float mu = sm * (1.f / NCH);
  float m2 = 0.f;
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) {
    const float a = q[i].x - mu, b = q[i].z - mu;
    m2 += q[i].y + q[i].w + 32.f * (a * a + b * b);
  }
  return make_float2(mu, rsqrtf(m2 * (1.f / (32 * NCH)) + eps));
}
__device__ __forceinline__ float2 merge_stats(const float2* st, int nch, float eps) {
  switch (nch) {
    case 16: return merge_stats_n<16>(st, eps);   // d = 512
    case 8: return merge_stats_n<8>(st, eps);     // d = 256
    case 32: return merge_stats_n<32>(st, eps);   // d = 1024
    default: break;
  }
  float sm = 0.f;
  for (int i = 0; i < nch; ++i) sm += st[i].x;
  const float mu = sm / nch;
  float m2 = 0.f;
  for (int i = 0; i < nch; ++i) {
    const float dm = st[i].x - mu;
    m2 += st[i].y + 32.f * dm * dm;
  }
  return make_float2(mu, rsqrtf(m2 / (32.f * nch) + eps));
}

template <int BN, int STAGES, bool PAIR = false, int EW = 8, int NSTG = 1>
struct Smem {
  static constexpr int BROWS = PAIR ? BN / 2 : BN;   // B rows staged by one CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BROWS * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // epilogue: per warp a 32 x 32 FP16 staging tile (TMA store) and its FP32 bias slice
  static constexpr int STG = 2048;
  // per epilogue warp: a 32 x 32 staging tile (TMA store) + bias and LN c[n] slices
  // NSTG staging tiles per warp (2: the residual of chunk i + 1 is TMA-loaded while chunk i
  // is processed), the whole bias vector (N <= kBiasMax) and per-unit bias / LN c slices
  static constexpr int BIAS = kBiasMax * 4;
  static constexpr int EPI = EW * NSTG * STG + BIAS + 2 * 4 * BN * 4;
  static constexpr int BYTES = STAGES * STAGE + EPI + 1024 /*align slack*/ + 512 /*barriers*/;
};

// Epilogue math on 32 consecutive columns nb..nb+31 of row m (v = FP32 accumulators):
// bias (from the warp's shared-memory slice, zero beyond N), residual (prefetched `pre` or
// loaded here), ReLU.
// a.lo/hi (FP16 pair) added to two FP32 values, one mixed-precision add each (FHADD)
__device__ __forceinline__ void add_h2(uint32_t pair, float& lo, float& hi) {
  asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
      "add.rn.f32.f16 %0, l, %0;\n\tadd.rn.f32.f16 %1, h, %1;\n\t}"
      : "+f"(lo), "+f"(hi)
      : "r"(pair));
}
// (lo, hi) -> max(., 0) rounded to a saturating half2 in one instruction
__device__ __forceinline__ uint32_t pack_half2_sat_relu(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void epi_math(const Params& p, int m, int nb, float* v,
                                         const float* sb, const uint4* pre, bool row_ok,
                                         const float* sc = nullptr, float2 ln = {0.f, 0.f},
                                         bool relu_in_pack = false) {
  const int nv = min(32, p.N - nb);
  const bool full = nv == 32;
  if (p.ln_st) {  // folded LayerNorm: rstd * (acc - mu * c[n])
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 c = *reinterpret_cast<const float4*>(sc + j);
      v[j] = ln.y * fmaf(-ln.x, c.x, v[j]);
      v[j + 1] = ln.y * fmaf(-ln.x, c.y, v[j + 1]);
      v[j + 2] = ln.y * fmaf(-ln.x, c.z, v[j + 2]);
      v[j + 3] = ln.y * fmaf(-ln.x, c.w, v[j + 3]);
    }
  }
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 b = *reinterpret_cast<const float4*>(sb + j);
      v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
    }
  }
  if (p.R && row_ok && nv > 0) {
    const __half* rr = p.R + (size_t)m * p.ldr + nb;
    if (pre) {  // residual prefetched before the accumulator wait; FP16 + FP32 adds
#pragma unroll
      for (int j8 = 0; j8 < 4; ++j8) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&pre[j8]);
#pragma unroll
        for (int e = 0; e < 4; ++e) add_h2(w[e], v[j8 * 8 + 2 * e], v[j8 * 8 + 2 * e + 1]);
      }
    } else if (full && ((reinterpret_cast<uintptr_t>(rr) & 15) == 0)) {
#pragma unroll
      for (int j8 = 0; j8 < 4; ++j8) {
        float f[8];
        load8h(rr + j8 * 8, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[j8 * 8 + e] += f[e];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) v[j] += __half2float(rr[j]);
    }
  }
  if (p.relu && !relu_in_pack) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
}

// Direct outputs of 32 columns (row m < M, nb < N): FP32 logits, the packed argmax, or
// the FP16 row segment (paths without the TMA-store epilogue).
__device__ __forceinline__ void epi_out(const Params& p, int m, int nb, const float* v,
                                        unsigned long long& best) {
  const int nv = min(32, p.N - nb);
  const bool full = nv == 32;
  if (p.logits) {
    float* lr = p.logits + (size_t)m * p.N + nb;
    if (full && ((p.N & 3) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(lr + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) lr[j] = v[j];
    }
  }
  if (p.argmax) {  // ascending scan, strict '>' keeps the lowest id among equal maxima
    float bv = v[0];
    int bj = 0;
#pragma unroll
    for (int j = 1; j < 32; ++j)
      if (j < nv && v[j] > bv) {
        bv = v[j];
        bj = j;
      }
    const unsigned long long k = pack_argmax(bv, nb + bj);
    best = k > best ? k : best;
    return;
  }
  if (!p.C) return;  // logits-only (beam search) epilogue
  __half* cr = p.C + (size_t)m * p.ldc + nb;
  if (full && ((reinterpret_cast<uintptr_t>(cr) & 15) == 0)) {
#pragma unroll
    for (int j8 = 0; j8 < 4; ++j8) {
      uint4 pk;
      pk.x = pack_half2_sat(v[j8 * 8 + 0], v[j8 * 8 + 1]);
      pk.y = pack_half2_sat(v[j8 * 8 + 2], v[j8 * 8 + 3]);
      pk.z = pack_half2_sat(v[j8 * 8 + 4], v[j8 * 8 + 5]);
      pk.w = pack_half2_sat(v[j8 * 8 + 6], v[j8 * 8 + 7]);
      reinterpret_cast<uint4*>(cr)[j8] = pk;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv) cr[j] = from_f<__half>(v[j]);
  }
}

// ---- TMA store of a 32 x 32 FP16 tile staged with the 64-B swizzle
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}


// ---- beam epilogue: online log-sum-exp and the top-8
// (value desc, id asc) of one row's segment of logits, kept in registers across chunks
constexpr int kBeamKB = 8;
constexpr int kBeamRec = 2 + 2 * kBeamKB;
struct BeamAcc {
  float mx, sum;
  float tv[kBeamKB];
  int ti[kBeamKB];
  __device__ __forceinline__ void init() {
    mx = -INFINITY;
    sum = 0.f;
#pragma unroll
    for (int k = 0; k < kBeamKB; ++k) { tv[k] = -INFINITY; ti[k] = 0x7fffffff; }
  }
  __device__ __forceinline__ static bool better(float a, int ia, float b, int ib) {
    return a > b || (a == b && ia < ib);
  }
  // 32 columns nb..nb+31 of the row, nv of them valid.  The chunk maximum decides whether
  // the chunk can enter the top-8 at all (after the first chunks it rarely can), so the
  // per-element work is one exp and one add.
  __device__ __forceinline__ void add(const float* v, int nb, int nv) {
    float cm = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv) cm = fmaxf(cm, v[j]);
    float cs = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv) cs += __expf(v[j] - cm);
    if (cm > mx) {
      sum = sum * __expf(mx - cm) + cs;
      mx = cm;
    } else {
      sum += cs * __expf(cm - mx);
    }
    if (!(cm >= tv[kBeamKB - 1])) return;   // nothing of this chunk enters the top-8
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv && better(v[j], nb + j, tv[kBeamKB - 1], ti[kBeamKB - 1])) insert(v[j], nb + j);
  }
  __device__ __forceinline__ void insert(float cv, int ci) {
#pragma unroll
    for (int k = 0; k < kBeamKB; ++k) {
      if (better(cv, ci, tv[k], ti[k])) {
        const float t1 = tv[k];
        const int t2 = ti[k];
        tv[k] = cv; ti[k] = ci; cv = t1; ci = t2;
      }
    }
  }
  __device__ __forceinline__ void store(float* rec) const {
    rec[0] = mx;
    rec[1] = sum;
#pragma unroll
    for (int k = 0; k < kBeamKB; ++k) {
      rec[2 + k] = tv[k];
      rec[2 + kBeamKB + k] = __int_as_float(ti[k]);
    }
  }
};

// Host: TMA descriptor (cached) of a row-major FP16 [rows][cols] matrix with leading dim ld:
// operand maps box {BK, box_rows}, 128-B swizzle; output maps (out) box {32, 32}, 64-B swizzle.
CUtensorMap make_map(const void* ptr, int rows, int cols, int ld, int box_rows, bool out = false);
int num_sms();

}  // namespace tc
}  // namespace nmt
