// decode_fused.cu — the FP16 decode step as ONE persistent kernel (per contiguous range of
// its phases): embedding + LN, and per decoder layer the QKV projection, cached RPR self-
// attention with the KV append, self-output projection, cross-query projection, cross-
// attention over the once-per-sentence encoder K/V, cross-output projection, FFN1, FFN2,
// then the final LayerNorm (the step the paper calls "the most time-
// consuming part").  Unfused, these are 11 dependent launches whose fixed costs
// (launch, setup, pipeline fill, teardown: 6-7 us each) dominate small-batch steps.
//
// Work is a list of ITEMS in phase order: GEMM tiles (128 rows x 64/128 columns, full K,
// tcgen05 MMA into TMEM, TMA-fed) and SIMT items (8 rows of embedding / LayerNorm, or 8
// (row, head) attention tasks), all row-block local: an item of row block rb depends only on
// the previous phase's items of rb, tracked by per-(phase, row block) completion counters in
// global memory.  CTAs take items from one global atomic counter, in order, so a CTA only
// ever waits for items taken earlier by running CTAs: no co-residency assumption, no grid
// barrier (safe next to the other workers' kernels).  Row blocks pipeline through the
// phases (rb 0 can be in FFN1 while rb 5 is in the QKV projection).
//
// Roles (384 threads): warp 0 = scheduler + TMA producer (weights requested before the
// activation dependency is satisfied), warp 1 = tcgen05 MMA issuer (one thread, double-
// buffered TMEM accumulators), warp 2 = TMEM allocator, warps 4-11 = math: GEMM epilogues
// and the SIMT items.  Arithmetic, tile shapes, split-K association and epilogue order are
// those of the unfused path (gemm_tc.cu decode_config, attention.cu, kernels.cu), so the
// fused step is bit-identical to it (tests/test_gpu_fused.py).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "rowops.cuh"
#include "tc_dev.cuh"
#include "warp_attn.cuh"
#include "decode_fused.h"

namespace nmt {
namespace dfz {

using namespace tc;

constexpr int NST = 6;            // stage ring (A 16 KB + B <= 16 KB per stage)
constexpr int STAGE = 32768;
constexpr int A_BYTES = BM * BK * 2;
constexpr int NMW = 8;            // math warps (4 TMEM lane quadrants x 2 column halves)
constexpr int MW0 = 4;            // first math warp
constexpr int kThreadsF = 32 * (MW0 + NMW);
constexpr int kRB = 128;          // rows per row block (= UMMA M)
constexpr int kMaxRB = 128;       // row blocks per launch (16384 rows)

enum Kind { K_EMB = 0, K_GEMM = 1, K_SELF = 2, K_CROSS = 3, K_LN = 4 };

__device__ __forceinline__ int phase_kind(int p, int nph) {
  if (p == 0) return K_EMB;
  if (p == nph - 1) return K_LN;
  const int r = (p - 1) & 7;
  return r == 1 ? K_SELF : r == 4 ? K_CROSS : K_GEMM;
}
__device__ __forceinline__ int phase_layer(int p) { return (p - 1) >> 3; }
// GEMM slot within a layer: 0 QKV, 1 self-out, 2 cross-q, 3 cross-out, 4 FFN1, 5 FFN2
__device__ __forceinline__ int gemm_slot(int p) {
  const int r = (p - 1) & 7;
  return r == 0 ? 0 : r == 2 ? 1 : r == 3 ? 2 : r == 5 ? 3 : r == 6 ? 4 : 5;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bounded spin on a completion counter (a scheduling bug traps instead of hanging the GPU):
// tight polling first (the producer is usually a few hundred ns away), then backing off.
__device__ __forceinline__ void wait_count(const int* c, int target) {
  if (ld_acquire(c) >= target) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (i > 256) __nanosleep(64);
    if (ld_acquire(c) >= target) return;
    if ((i & 255) == 0 && clock64() - t0 > 20000000000ll)
      NMT_TRAP("wait_count", ld_acquire(c), target);
  }
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float2 ld_cg_f2x2(const float2* p, float2& b) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  b = make_float2(v.z, v.w);
  return make_float2(v.x, v.y);
}
// merge_stats_n (tc_dev.cuh) with L2-only loads (the statistics are written in this launch)
template <int NCH>
__device__ __forceinline__ float2 merge_stats_cg(const float2* st, float eps) {
  float4 q[NCH / 2];
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) {
    float2 b;
    const float2 a = ld_cg_f2x2(st + 2 * i, b);
    q[i] = make_float4(a.x, a.y, b.x, b.y);
  }
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
template <int E>
__device__ __forceinline__ void ldrow_cg(const __half* p, float* v) {
#pragma unroll
  for (int i = 0; i < E; i += 8) {
    const uint4 u = ld_cg16(p + i);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __half22float2(h[e]);
      v[i + 2 * e] = x.x;
      v[i + 2 * e + 1] = x.y;
    }
  }
}

struct Smem {
  uint64_t full[NST], empty[NST], tfull[2], tempty[2], rfull[2], rempty[2];
  int ring[2];
  uint32_t tmem;
  int R, t, S, total, nb;
  int rel_layer;
  int pstart[kMaxPhases + 1];
  float relk[16][64], relv[16][64];
  float x[NMW][16];
};

// Items of phase p for R live rows (row-block local; the last row block may be partial).
__device__ __forceinline__ int rows_per_item(int kind, int H) {
  return (kind == K_SELF || kind == K_CROSS) ? NMW / H : NMW;
}

template <int E, int DH>
__global__ void __launch_bounds__(kThreadsF, 1) k_decode_fused(const __grid_constant__ FusedParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* stages = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // shared address space kept
  Smem& S = *reinterpret_cast<Smem*>(stages + NST * STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nph = 2 + 8 * P.Ld;
  constexpr int d = 32 * E;
  const int H = d / DH;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&S.tfull[a], 1);
      mbar_init(&S.tempty[a], NMW);
      mbar_init(&S.rfull[a], 1);
      mbar_init(&S.rempty[a], 1 + NMW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // live rows, step and source length of this step (written by the previous launches)
    const int R = P.st->n_live;
    S.R = R;
    S.t = P.st->t;
    S.S = P.st->S;
    S.rel_layer = -1;
    const int nb = (R + kRB - 1) / kRB;
    S.nb = nb;
    const int last = R - (nb - 1) * kRB;
    int acc = 0;
    for (int p = 0; p < nph; ++p) {
      S.pstart[p] = acc;
      if (p < P.pbeg || p >= P.pend || R <= 0) continue;
      const int kind = phase_kind(p, nph);
      if (kind == K_GEMM) {
        acc += nb * P.L[phase_layer(p)].g[gemm_slot(p)].nt;
      } else {
        const int rpi = rows_per_item(kind, H);
        acc += (nb - 1) * (kRB / rpi) + (last + rpi - 1) / rpi;
      }
    }
    S.pstart[nph] = acc;
    S.total = acc;
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem;
  const int R = S.R, total = S.total;
  if (P.trace && threadIdx.x == 0) P.trace[4 * 65536 + blockIdx.x] = gtimer();
  int* done = P.ctr + 2;   // [phase][row block] completion counters

  // item -> (phase, row block, index within the row block)
  auto decode = [&](int item, int& p, int& rb, int& j) {
    p = P.pbeg;
    while (p + 1 < nph && S.pstart[p + 1] <= item) ++p;
    const int sub = item - S.pstart[p];
    const int kind = phase_kind(p, nph);
    const int per = kind == K_GEMM ? P.L[phase_layer(p)].g[gemm_slot(p)].nt
                                   : kRB / rows_per_item(kind, H);
    rb = sub / per;
    j = sub - rb * per;
  };
  // completion count of phase p at row block rb
  auto expected = [&](int p, int rb) {
    const int kind = phase_kind(p, nph);
    if (kind == K_GEMM) return P.L[phase_layer(p)].g[gemm_slot(p)].nt;
    const int rpi = rows_per_item(kind, H);
    const int rows = min(kRB, R - rb * kRB);
    return (rows + rpi - 1) / rpi;
  };

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ scheduler + TMA producer
      uint32_t it = 0;
      for (int k = 0;; ++k) {
        int item = atomicAdd(P.ctr, 1);
        if (item >= total) item = -1;
        const int slot = k & 1;
        mbar_wait(&S.rempty[slot], ((k >> 1) & 1) ^ 1);
        S.ring[slot] = item;
        mbar_arrive(&S.rfull[slot]);
        if (item < 0) break;
        int p, rb, j;
        decode(item, p, rb, j);
        if (phase_kind(p, nph) != K_GEMM) continue;
        const GemmPhase& G = P.L[phase_layer(p)].g[gemm_slot(p)];
        const int n0 = j * G.bn, m0 = rb * kRB;
        // a row block with few live rows loads 32-row A boxes (rows beyond are never stored)
        const bool small = R - m0 <= 32;
        const CUtensorMap* ma = small ? &P.L[phase_layer(p)].ma32[gemm_slot(p)]
                                      : &P.L[phase_layer(p)].ma[gemm_slot(p)];
        const CUtensorMap* mb = &P.L[phase_layer(p)].mb[gemm_slot(p)];
        const int kbt = G.K / BK;
        const uint32_t bbytes = (uint32_t)G.bn * BK * 2;
        const uint32_t abytes = small ? 32 * BK * 2 : A_BYTES;
        const int npre = min(kbt, NST);
        // weights first: they never depend on this launch's work
        for (int kb = 0; kb < npre; ++kb) {
          const uint32_t q = it + kb, st = q % NST;
          mbar_wait(&S.empty[st], ((q / NST) & 1) ^ 1);
          mbar_expect_tx(&S.full[st], abytes + bbytes);
          tma_load_2d(stages + st * STAGE + A_BYTES, mb, &S.full[st], kb * BK, n0);
        }
        if (p > P.pbeg) {   // the activation rows of rb are ready (previous phase complete)
          wait_count(done + (p - 1) * kMaxRB + rb, expected(p - 1, rb));
          fence_proxy_async_global();
        }
        for (int kb = 0; kb < kbt; ++kb) {
          const uint32_t q = it + kb, st = q % NST;
          if (kb >= npre) {
            mbar_wait(&S.empty[st], ((q / NST) & 1) ^ 1);
            mbar_expect_tx(&S.full[st], abytes + bbytes);
            tma_load_2d(stages + st * STAGE + A_BYTES, mb, &S.full[st], kb * BK, n0);
          }
          tma_load_2d(stages + st * STAGE, ma, &S.full[st], kb * BK, m0);
        }
        it += kbt;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      uint32_t it = 0, ng = 0;
      for (int k = 0;; ++k) {
        const int slot = k & 1;
        mbar_wait(&S.rfull[slot], (k >> 1) & 1);
        const int item = S.ring[slot];
        mbar_arrive(&S.rempty[slot]);
        if (item < 0) break;
        int p, rb, j;
        decode(item, p, rb, j);
        if (phase_kind(p, nph) != K_GEMM) continue;
        const GemmPhase& G = P.L[phase_layer(p)].g[gemm_slot(p)];
        const int kbt = G.K / BK;
        const uint32_t idesc = (1u << 4) | ((uint32_t)(G.bn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        const uint32_t acc = ng & 1, aph = (ng >> 1) & 1;
        ++ng;
        mbar_wait(&S.tempty[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < kbt; ++kb, ++it) {
          const uint32_t st = it % NST;
          mbar_wait(&S.full[st], (it / NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // split = 2: the K halves accumulate separately (the unfused cluster split-K)
          const bool second = G.split && kb >= kbt / 2;
          const uint32_t dcol = tmem + acc * 128 + (second ? 64u : 0u);
          const bool first = kb == 0 || (G.split && kb == kbt / 2);
          const uint64_t da = make_desc_sw128(stages + st * STAGE);
          const uint64_t db = make_desc_sw128(stages + st * STAGE + A_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk)
            mma_f16(dcol, da + 2 * kk, db + 2 * kk, idesc, (first && kk == 0) ? 0u : 1u);
          mma_commit(&S.empty[st]);
        }
        mma_commit(&S.tfull[acc]);
      }
    }
  } else if (warp >= MW0) {  // ------------------------------------------ math warps
    const int w = warp - MW0;
    const int mt = threadIdx.x - 32 * MW0;   // 0..255
    uint32_t ng = 0;
    unsigned long long t_recv = 0, t_ready = 0;
    int cur_item = 0;
    auto signal = [&](int p, int rb) {      // this item's outputs are visible gpu-wide
      fence_proxy_async_global();           // generic-proxy stores -> later TMA (async) reads
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NMW) : "memory");
      if (mt == 0) {
        // the CTA barrier orders every math thread's stores before this release (the
        // CUTLASS generic-barrier pattern: __syncthreads, then one red.release.gpu)
        red_release_add(done + p * kMaxRB + rb, 1);
        if (P.trace) {   // debug timeline: (phase, rb, cta), received, inputs ready, done
          unsigned long long* tr = P.trace + 4 * (size_t)cur_item;
          tr[0] = ((unsigned long long)p << 40) | ((unsigned long long)rb << 20) | blockIdx.x;
          tr[1] = t_recv;
          tr[2] = t_ready;
          tr[3] = gtimer();
        }
      }
    };
    for (int k = 0;; ++k) {
      const int slot = k & 1;
      mbar_wait(&S.rfull[slot], (k >> 1) & 1);
      const int item = S.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.rempty[slot]);
      if (item < 0) break;
      if (P.trace) t_recv = gtimer();
      cur_item = item;
      int p, rb, j;
      decode(item, p, rb, j);
      const int kind = phase_kind(p, nph);
      const int l = kind == K_EMB ? 0 : kind == K_LN ? P.Ld - 1 : phase_layer(p);
      const FusedLayer& Lw = P.L[l];
      if (kind == K_GEMM) {
        const GemmPhase& G = Lw.g[gemm_slot(p)];
        const uint32_t acc = ng & 1, aph = (ng >> 1) & 1;
        ++ng;
        const int q = w & 3, hf = w >> 2;
        const int m = rb * kRB + q * 32 + lane;
        const bool row_ok = m < R;
        const int wcols = G.bn / 2;                 // columns of this warp: 32 or 64
        const int cb = hf * wcols;
        // the accumulator is ready only after the producer saw this row block's inputs
        // complete: everything this launch wrote (statistics, residual) is read after it
        mbar_wait(&S.tfull[acc], aph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (P.trace) t_ready = gtimer();
        float2 ln = make_float2(0.f, 0.f);
        if (G.ln_st && row_ok) ln = merge_stats_cg<E>(G.ln_st + (size_t)m * (G.K / 32), P.eps);
        const uint32_t tb = tmem + acc * 128 + ((uint32_t)(q * 32) << 16);
        for (int c0 = cb; c0 < cb + wcols; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tb + c0, v);
          if (G.split) {
            float v2[32];
            tmem_ld32(tb + 64 + c0, v2);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (0.f + v[i]) + v2[i];
          }
          if (c0 + 32 >= cb + wcols) {  // this warp's columns read: release the accumulator
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.tempty[acc]);
          }
          const int n0 = j * G.bn + c0;
          if (!row_ok) continue;
          // epilogue in the order of tc::epi_math: folded LN, bias, residual, ReLU
          if (G.ln_st) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 c = *reinterpret_cast<const float4*>(G.ln_c + n0 + i);
              v[i] = ln.y * fmaf(-ln.x, c.x, v[i]);
              v[i + 1] = ln.y * fmaf(-ln.x, c.y, v[i + 1]);
              v[i + 2] = ln.y * fmaf(-ln.x, c.z, v[i + 2]);
              v[i + 3] = ln.y * fmaf(-ln.x, c.w, v[i + 3]);
            }
          }
          if (G.bias) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              const uint4 u = *reinterpret_cast<const uint4*>(G.bias + n0 + i);
              const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __half22float2(h[e]);
                v[i + 2 * e] += f.x;
                v[i + 2 * e + 1] += f.y;
              }
            }
          }
          if (G.R) {
            const __half* rr = G.R + (size_t)m * d + n0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 u = ld_cg16(rr + 8 * i);
              add_h2(u.x, v[8 * i + 0], v[8 * i + 1]);
              add_h2(u.y, v[8 * i + 2], v[8 * i + 3]);
              add_h2(u.z, v[8 * i + 4], v[8 * i + 5]);
              add_h2(u.w, v[8 * i + 6], v[8 * i + 7]);
            }
          }
          if (G.st_out) G.st_out[(size_t)m * (G.N / 32) + n0 / 32] = chunk_stats(v);
          uint32_t hh[16];
          if (G.relu) {
#pragma unroll
            for (int i = 0; i < 16; ++i) hh[i] = pack_half2_sat_relu(v[2 * i], v[2 * i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) hh[i] = pack_half2_sat(v[2 * i], v[2 * i + 1]);
          }
          uint4* cr = reinterpret_cast<uint4*>(G.C + (size_t)m * G.ldc + n0);
#pragma unroll
          for (int i = 0; i < 4; ++i) cr[i] = make_uint4(hh[4 * i], hh[4 * i + 1], hh[4 * i + 2], hh[4 * i + 3]);
        }
        signal(p, rb);
        continue;
      }
      // ---------------- SIMT items: wait for the previous phase at this row block
      if (p > P.pbeg) {
        if (lane == 0) wait_count(done + (p - 1) * kMaxRB + rb, expected(p - 1, rb));
        __syncwarp();
      }
      if (P.trace) t_ready = gtimer();
      const int t = S.t;
      if (kind == K_EMB || kind == K_LN) {
        // one warp per row (kernels.cu k_embed_dec_ln_vec / k_layernorm_vec)
        const int row = rb * kRB + j * NMW + w;
        if (row < R) {
          float v[E];
          if (kind == K_EMB) {
            ldrow<__half, E>(P.emb + (size_t)P.ids[row] * d + lane * E, v);
            const float* pp = P.pe + (size_t)t * d + lane * E;
#pragma unroll
            for (int i = 0; i < E; i += 4) {
              const float4 qv = *reinterpret_cast<const float4*>(pp + i);
              v[i] = to_f(from_f<__half>(v[i] * P.scale + qv.x));
              v[i + 1] = to_f(from_f<__half>(v[i + 1] * P.scale + qv.y));
              v[i + 2] = to_f(from_f<__half>(v[i + 2] * P.scale + qv.z));
              v[i + 3] = to_f(from_f<__half>(v[i + 3] * P.scale + qv.w));
            }
            strow<__half, E>(P.g + (size_t)row * d + lane * E, v);
            ln_contig<__half, E>(v, d, P.ln0_g, P.ln0_b, P.eps, lane);
          } else {
            ldrow_cg<E>(P.g + (size_t)row * d + lane * E, v);
            ln_contig<__half, E>(v, d, P.lnf_g, P.lnf_b, P.eps, lane);
          }
          strow<__half, E>(P.u + (size_t)row * d + lane * E, v);
        }
        signal(p, rb);
        continue;
      }
      // attention: task w = (row, head)
      using WA = WarpAttn<__half, DH, true>;
      const int rpi = NMW / H;
      const int row = rb * kRB + j * rpi + w / H, h = w % H;
      if (kind == K_SELF) {
        if (P.use_rpr && S.rel_layer != l) {   // A^K / A^V[0..k] of this layer, once per CTA
          for (int i = mt; i < (P.kclip + 1) * DH; i += 32 * NMW) {
            S.relv[i / DH][i % DH] = to_f(Lw.relv[i]);
            S.relk[i / DH][i % DH] = to_f(Lw.relk[i]);
          }
          asm volatile("bar.sync 2, %0;" ::"r"(32 * NMW) : "memory");
          if (mt == 0) S.rel_layer = l;
        }
        if (row < R) {   // kernels: attention.cu k_attn_dec_self
          const int slot = P.row_slot[row];
          const __half* src = P.qkv + (size_t)row * 3 * d + h * DH;
          WA wa;
          wa.init(lane, src, rsqrtf((float)DH));
          Raw8<__half> kt, vt;
          if (wa.kq == 0) {
            kt.load_cg(src + d + wa.sub * 8);
            vt.load_cg(src + 2 * d + wa.sub * 8);
            kt.store(Lw.kc + ((size_t)slot * P.Tmax + t) * d + h * DH + wa.sub * 8);
            vt.store(Lw.vc + ((size_t)slot * P.Tmax + t) * d + h * DH + wa.sub * 8);
          }
          float* x = S.x[w];
          if (P.use_rpr) {
            for (int b0 = 0; b0 <= P.kclip; b0 += WA::KP) {
              const int b = b0 + wa.kq;
              float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
              if (b <= P.kclip) {
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = S.relk[b][wa.sub * 8 + e];
              }
              const float e = wa.group_dot(f);
              if (b <= P.kclip && wa.sub == 0) x[b] = e;
            }
            __syncwarp();
          }
          const int* anc_row = P.anc ? P.anc + (size_t)slot * P.Tmax : nullptr;
          const size_t hoff = (size_t)h * DH;
          auto addr = [&](int jj, const __half*& kp, const __half*& vp) {
            if (jj == t) {
              kp = src + d;
              vp = src + 2 * d;
            } else {
              const int sl = anc_row ? anc_row[jj] : slot;
              const size_t o = ((size_t)sl * P.Tmax + jj) * d + hoff;
              kp = Lw.kc + o;
              vp = Lw.vc + o;
            }
          };
          const int n = t + 1;
          const int kc = P.kclip;
          if (P.use_rpr) {
            auto bias = [&](int jj) { return x[max(jj - t, -kc) + kc]; };
            auto vadd = [&](int jj, float* f) {
              const float* rv = S.relv[max(jj - t, -kc) + kc] + wa.sub * 8;
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] += rv[e];
            };
            for (int j0 = 0; j0 < n; j0 += WA::CH) wa.chunk(j0, n, n, addr, bias, vadd);
          } else {
            auto bias = [](int) { return 0.f; };
            auto vadd = [](int, float*) {};
            for (int j0 = 0; j0 < n; j0 += WA::CH) wa.chunk(j0, n, n, addr, bias, vadd);
          }
          float o[8];
          wa.finish(o);
          if (wa.kq == 0) store8(P.attn_out + (size_t)row * d + hoff + wa.sub * 8, o);
        }
      } else if (row < R) {   // cross-attention (attention.cu k_attn_cross)
        const int Sl = S.S;
        const int slot = P.row_slot[row] / P.beam;
        WA wa;
        wa.init(lane, P.q + (size_t)row * d + h * DH, rsqrtf((float)DH));
        const int n = P.src_len[slot];
        const __half* base = P.ckv + (size_t)slot * Sl * P.ldkv + h * DH;
        const int koff = Lw.koff, voff = Lw.voff;
        auto addr = [&](int jj, const __half*& kp, const __half*& vp) {
          kp = base + (size_t)jj * P.ldkv + koff;
          vp = base + (size_t)jj * P.ldkv + voff;
        };
        auto bias = [](int) { return 0.f; };
        auto vadd = [](int, float*) {};
        wa.chunk(0, n, Sl, addr, bias, vadd);
        for (int j0 = WA::CH; j0 < n; j0 += WA::CH) wa.chunk(j0, n, n, addr, bias, vadd);
        float o[8];
        wa.finish(o);
        if (wa.kq == 0) store8(P.attn_out + (size_t)row * d + h * DH + wa.sub * 8, o);
      }
      signal(p, rb);
    }
  }
  // ---------------- teardown: TMEM, then the last CTA out resets the counters
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(P.ctr + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {   // every CTA has finished every item: zero the counters for the next launch
    __threadfence();
    const int n = 2 + nph * kMaxRB;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i != 1) P.ctr[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      P.ctr[1] = 0;
    }
  }
}

size_t smem_bytes() { return NST * STAGE + sizeof(Smem) + 1024; }

}  // namespace dfz

size_t fused_counter_ints() { return 2 + (size_t)dfz::kMaxPhases * dfz::kMaxRB; }

bool fused_supported(int d, int H, int F, int Ld) {
  const int dh = d / H;
  return (d == 512 || d == 256) && dh == 64 && (8 % H == 0) && Ld >= 1 && Ld <= kMaxFusedLayers &&
         F % 128 == 0 && (3 * d) % 128 == 0;
}

void decode_fused(const FusedParams& p, int E, cudaStream_t s) {
  using namespace dfz;
  static_assert(sizeof(FusedParams) <= 32000, "kernel parameter block too large");
  const int grid = tc::num_sms();
  const size_t smem = smem_bytes();
#define NMT_DF(EE)                                                                          \
  do {                                                                                      \
    static const bool attr = [&] {                                                          \
      NMT_CUDA(cudaFuncSetAttribute(k_decode_fused<EE, 64>,                                  \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      return true;                                                                          \
    }();                                                                                    \
    (void)attr;                                                                             \
    k_decode_fused<EE, 64><<<grid, kThreadsF, smem, s>>>(p);                                 \
  } while (0)
  if (E == 16) NMT_DF(16);
  else if (E == 8) NMT_DF(8);
  else throw CudaError("decode_fused: d must be 256 or 512");
#undef NMT_DF
  NMT_LAUNCH_CHECK();
}

}  // namespace nmt
