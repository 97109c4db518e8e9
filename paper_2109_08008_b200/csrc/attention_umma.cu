// attention_umma.cu — encoder RPR self-attention (Shaw et al. keys AND values, clip 8;
// PAPER.md:23, :34; reading R7) on the 5th-generation tensor cores, FP16 in / FP32 out:
//   S  = Q K^T            tcgen05 M=128 (queries) x N=128 (keys) x K=64, accumulator in TMEM
//   QA = Q A^K^T          N=32 (17 relative buckets, zero-padded)
//   one thread per query row (tcgen05.ld of its TMEM row): e_ij = (S_ij + QA_i[r(i,j)]) /
//   sqrt(dh), masked j >= len, exp2 softmax in FP32 (two passes: max, then exp / sum),
//   P_ij = exp(e_ij - max) and the bucket sums B_i[r] = sum_{j: r(i,j) = r} P_ij written to
//   shared memory as FP16 MMA operands (R19)
//   O  = P V + B A^V      N=64, V and A^V as MN-major (value-row) operands, then O / sum_j P_ij
// with r(i,j) = clip(j - i, -k, k) + k.  A tile is 128 query rows: 128 / SPP items
// ((sentence, head) pairs) of SPP = 32 / 64 / 128 padded rows each side by side (block-
// diagonal: a row only attends its own item's keys), so short sentences do not waste the
// tile.  Persistent CTAs walk the tiles; warp 0 streams each tile's Q / K / V head slices
// with TMA into a 2-slot ring, warp 1 issues the MMAs (QK^T of tile k+1 before P V of tile
// k), two groups of 4 warps run the softmax / epilogue of alternate tiles against double-
// buffered TMEM accumulators (512 columns).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_dev.cuh"

namespace nmt {
namespace ua {

using namespace tc;

constexpr int TILE = 128 * 128;          // one 128-row x 64-column FP16 operand tile (SW128)
constexpr int SLOT = 3 * TILE;           // Q, K, V
constexpr int PT = 2 * TILE;             // P [128 rows][128 keys] = two SW128 atoms columns
constexpr int BT = TILE;                 // bucket sums [128][64] (32 used)
constexpr int kThreadsU = 384;           // warps: 0 TMA, 1 MMA, 2 TMEM, 3 idle, 4-11 softmax
constexpr uint32_t kTmemCols = 512;      // three buffers x (S / O 128 + QA 32) = 480
constexpr int NTB = 3;                   // TMEM buffers: tiles in flight between QK^T and the epilogue
constexpr uint32_t TBC = 160;            // columns per TMEM buffer: S [0,128), O aliases S [64,128), QA [128,160)

struct USmem {
  // Q / K and V of a slot are loaded and released separately: Q / K are consumed by the
  // QK^T MMA (released early, so the next tile's loads overlap this tile's softmax), V by
  // P V
  uint64_t full[2], empty[2], vfull[2], vempty[2], pfull[2], sfull[NTB], ofull[NTB], tfree[NTB];
  uint32_t tmem;
  float qa[2][128][17];                  // per group: q . A^K rows (FP32, bucket-indexed)
};

// debug timeline of CTA 0 (nmt_debug_attn_trace): per local tile k < 64, 8 globaltimer
// stamps {Q/K TMA issued, V TMA issued, QK^T issued, S seen by softmax, P ready,
// P V issued, O seen by epilogue, TMEM freed}
__device__ unsigned long long g_ua_trace[64 * 16];
__device__ __forceinline__ unsigned long long ua_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define UA_TR(k, e) \
  do { if (trace && blockIdx.x == 0 && (k) < 64) g_ua_trace[(k) * 16 + (e)] = ua_now(); } while (0)

__device__ __forceinline__ uint32_t swz(int r, int chunk) {   // SW128 byte offset of (row, 16-B chunk)
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((chunk ^ (r & 7)) << 4));
}

// idesc: D F32, A/B F16, a K-major, b K-major (b_mn = 0) or MN-major (b_mn = 1), N, M = 128
__host__ __device__ constexpr uint32_t idesc(int n, int b_mn) {
  return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int SPP>
__global__ void __launch_bounds__(kThreadsU, 1) k_attn_enc_umma(
    const __grid_constant__ CUtensorMap mqkv, const int* __restrict__ len,
    const __half* __restrict__ relk, const __half* __restrict__ relv, __half* __restrict__ out,
    int B, int S, int d, int H, int kclip, int trace) {
  constexpr int IPT = 128 / SPP;         // items per tile
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);   // keeps the shared address space
  uint8_t* slots = sm;                             // [2][Q | K | V]
  uint8_t* sP = slots + 2 * SLOT;                  // [2][P]
  uint8_t* sB = sP + 2 * PT;                       // [2][B]
  uint8_t* sAK = sB + 2 * BT;                      // A^K [32 buckets][64] K-major (B of QA)
  uint8_t* sAV = sAK + 32 * 128;                   // A^V [32 buckets][64] MN-major (B of B A^V)
  USmem& U = *reinterpret_cast<USmem*>(sAV + 32 * 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = B * H, tiles = (items + IPT - 1) / IPT;
  const int G = gridDim.x, c = blockIdx.x;
  const int nloc = c < tiles ? (tiles - 1 - c) / G + 1 : 0;
  const int R = 2 * kclip + 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&U.full[i], 1);
      mbar_init(&U.empty[i], 1);
      mbar_init(&U.vfull[i], 1);
      mbar_init(&U.vempty[i], 1);
      mbar_init(&U.pfull[i], 4);
    }
    for (int i = 0; i < NTB; ++i) {
      mbar_init(&U.sfull[i], 1);
      mbar_init(&U.ofull[i], 1);
      mbar_init(&U.tfree[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mqkv)) : "memory");
  }
  // relative tables once per CTA (rows >= R zero), both in the SW128 operand layout
  for (int idx = threadIdx.x; idx < 32 * 8; idx += blockDim.x) {
    const int r = idx >> 3, ch = idx & 7;
    uint4 k4 = make_uint4(0u, 0u, 0u, 0u), v4 = k4;
    if (r < R) {
      k4 = *reinterpret_cast<const uint4*>(relk + r * 64 + ch * 8);
      v4 = *reinterpret_cast<const uint4*>(relv + r * 64 + ch * 8);
    }
    *reinterpret_cast<uint4*>(sAK + swz(r, ch)) = k4;
    *reinterpret_cast<uint4*>(sAV + swz(r, ch)) = v4;
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&U.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();   // thread-written operand tiles -> the MMA (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = U.tmem;

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer
      // two streams (Q / K of tile kq, V of tile kv), issued as their slots free up
      auto src_row = [&](int t, int a, int& h) {
        const int it = t * IPT + a;
        // a missing item (last tile) loads rows past the tensor: zero-filled by TMA
        h = it < items ? it % H : 0;
        return it < items ? (it / H) * S : B * S + 256;
      };
      int kq = 0, kv = 0;
      while (kv < nloc) {
        bool did = false;
        if (kq < nloc && mbar_test(&U.empty[kq & 1], ((kq >> 1) & 1) ^ 1)) {
          const int sl = kq & 1, t = c + kq * G;
          UA_TR(kq, 0);
          mbar_expect_tx(&U.full[sl], IPT * 2 * SPP * 128);
          uint8_t* dst = slots + sl * SLOT;
#pragma unroll 1
          for (int a = 0; a < IPT; ++a) {
            int h;
            const int y = src_row(t, a, h);
            tma_load_2d(dst + a * SPP * 128, &mqkv, &U.full[sl], h * 64, y);
            tma_load_2d(dst + TILE + a * SPP * 128, &mqkv, &U.full[sl], d + h * 64, y);
          }
          ++kq;
          did = true;
        }
        if (kv < kq && mbar_test(&U.vempty[kv & 1], ((kv >> 1) & 1) ^ 1)) {
          const int sl = kv & 1, t = c + kv * G;
          UA_TR(kv, 1);
          mbar_expect_tx(&U.vfull[sl], IPT * SPP * 128);
          uint8_t* dst = slots + sl * SLOT + 2 * TILE;
#pragma unroll 1
          for (int a = 0; a < IPT; ++a) {
            int h;
            const int y = src_row(t, a, h);
            tma_load_2d(dst + a * SPP * 128, &mqkv, &U.vfull[sl], 2 * d + h * 64, y);
          }
          ++kv;
          did = true;
        }
        if (!did) __nanosleep(20);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      // Two independent streams: QK^T of tile kq (needs its Q / K / V slot loaded and its
      // TMEM buffer drained) and P V of tile kp (needs its softmax done).  A blocking wait
      // on one would stall the other (P V of tile k behind the TMA latency of tile k + 2),
      // so the issuer polls both and issues whichever is ready.
      int kq = 0, kp = 0;
      while (kp < nloc) {
        bool did = false;
        if (kq < nloc && kq < kp + NTB) {
          const int sl = kq & 1, tb = kq % NTB;
          if (mbar_test(&U.full[sl], (kq >> 1) & 1) && mbar_test(&U.tfree[tb], ((kq / NTB) & 1) ^ 1)) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint8_t* base = slots + sl * SLOT;
            const uint32_t tS = tmem + tb * TBC, tQA = tS + 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t dq = make_desc_sw128(base) + 2 * kk;
              mma_f16(tS, dq, make_desc_sw128(base + TILE) + 2 * kk, idesc(128, 0), kk > 0);
              mma_f16(tQA, dq, make_desc_sw128(sAK) + 2 * kk, idesc(32, 0), kk > 0);
            }
            mma_commit(&U.sfull[tb]);
            UA_TR(kq, 2);
            mma_commit(&U.empty[sl]);   // Q / K consumed: the next tile's Q / K may load
            ++kq;
            did = true;
          }
        }
        if (kp < kq && mbar_test(&U.pfull[kp & 1], (kp >> 1) & 1) &&
            mbar_test(&U.vfull[kp & 1], (kp >> 1) & 1)) {
          const int sl = kp & 1, bf = kp & 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t tO = tmem + (kp % NTB) * TBC + 64;   // aliases S: read before pfull
          const uint8_t* vb = slots + sl * SLOT + 2 * TILE;
          // O = P V: K = 128 keys; P K-major (two 64-key atom columns), V MN-major (8-key
          // groups 1024 B apart: +2048 B per 16 keys)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_f16(tO, make_desc_sw128(sP + bf * PT + (kk >> 2) * TILE) + 2 * (kk & 3),
                    make_desc_sw128(vb + kk * 2048), idesc(64, 1), kk > 0);
          // O += B A^V: K = 32 buckets
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            mma_f16(tO, make_desc_sw128(sB + bf * BT) + 2 * kk, make_desc_sw128(sAV + kk * 2048),
                    idesc(64, 1), 1u);
          mma_commit(&U.ofull[kp % NTB]);
          UA_TR(kp, 5);
          mma_commit(&U.vempty[sl]);   // V of this slot consumed
          ++kp;
          did = true;
        }
        if (!did) __nanosleep(20);
      }
    }
  } else if (warp >= 4) {   // ------------------------------------------------ softmax + epilogue
    const int grp = (warp - 4) >> 2, q = warp & 3, r = q * 32 + lane;   // tile row r
    const int a = r / SPP, i = r - a * SPP;                              // item, query row in item
    const float sl2 = 1.4426950408889634f * rsqrtf(64.f);
    for (int k = grp; k < nloc; k += 2) {
      const int bf = k & 1, t = c + k * G;
      const int it = t * IPT + a;
      const bool item_ok = it < items;
      const int b = item_ok ? it / H : 0, h = item_ok ? it % H : 0;
      const int n = item_ok ? len[b] : 0;
      const bool row_ok = i < n;
      const int tb = k % NTB;
      mbar_wait(&U.sfull[tb], (k / NTB) & 1);
      if (r == 0) UA_TR(k, 3);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t trow = tmem + tb * TBC + ((uint32_t)(q * 32) << 16);
      float* qa = U.qa[grp][r];
      {
        float v[32];
        tmem_ld32(trow + 128, v);
#pragma unroll
        for (int e = 0; e < 17; ++e) qa[e] = v[e];
      }
      if (r == 0) UA_TR(k, 8);
      // pass 1: row maximum of the scaled scores over this item's keys j < n
      float mx = -INFINITY;
#pragma unroll 1
      for (int c0 = 0; c0 < SPP; c0 += 32) {
        float v[32];
        tmem_ld32(trow + ((a * SPP + c0) & ~31), v);   // SPP < 32: the item's keys within
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int j = c0 + jj - ((a * SPP) & 31);   // key index within the item
          const float s = (v[jj] + qa[min(max(j - i, -kclip), kclip) + kclip]) * sl2;
          if (j >= 0 && j < n) mx = fmaxf(mx, s);
        }
      }
      if (!row_ok) mx = 0.f;
      if (r == 0) UA_TR(k, 9);
      // pass 2: P = exp2(s - max) (0 for masked keys / rows), sums, bucket sums, FP16 P row
      uint8_t* prow = sP + bf * PT;
      float sum = 0.f, lo = 0.f, hi = 0.f;
      uint8_t* brow = sB + bf * BT;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)   // zero this row's bucket sums
        *reinterpret_cast<uint4*>(brow + swz(r, ch)) = make_uint4(0u, 0u, 0u, 0u);
      // other items' key columns of this row are zero
#pragma unroll
      for (int kc = 0; kc < 16; ++kc) {
        const int key0 = kc * 8;
        if (key0 < a * SPP || key0 >= (a + 1) * SPP)
          *reinterpret_cast<uint4*>(prow + (kc >> 3) * TILE + swz(r, kc & 7)) = make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll 1
      for (int c0 = 0; c0 < (SPP < 32 ? 32 : SPP); c0 += 32) {
        float v[32];
        const int cb = (a * SPP + c0) & ~31;           // first tile column of this window
        tmem_ld32(trow + cb, v);
        uint32_t hp[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          float p2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = c0 + jj + e - ((a * SPP) & 31), dj = j - i;
            const float s = (v[jj + e] + qa[min(max(dj, -kclip), kclip) + kclip]) * sl2;
            const float p = (row_ok && j >= 0 && j < n) ? exp2f(s - mx) : 0.f;
            p2[e] = p;
            sum += p;
            lo += dj <= -kclip ? p : 0.f;
            hi += dj >= kclip ? p : 0.f;
          }
          hp[jj / 2] = pack_half2_sat(p2[0], p2[1]);
        }
        // FP16 P into the K-major SW128 tile: tile key = cb + 8*u + e
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kc = cb / 8 + u;
          *reinterpret_cast<uint4*>(prow + (kc >> 3) * TILE + swz(r, kc & 7)) =
              make_uint4(hp[4 * u], hp[4 * u + 1], hp[4 * u + 2], hp[4 * u + 3]);
        }
      }
      if (r == 0) UA_TR(k, 10);
      // band buckets: one key each (j = i + r - k for |r - k| < k), ends: the clipped sums
      if (row_ok) {
        __half* bh = nullptr;
        for (int dd = -kclip + 1; dd < kclip; ++dd) {
          const int j = i + dd;
          if (j < 0 || j >= n) continue;
          // P_ij again from the stored FP16 tile (the value the P V product uses)
          const int key = a * SPP + j;
          const __half pv = *reinterpret_cast<const __half*>(prow + (key >> 6) * TILE +
                                                              swz(r, (key >> 3) & 7) + (key & 7) * 2);
          const int bk = dd + kclip;
          bh = reinterpret_cast<__half*>(brow + swz(r, bk >> 3) + (bk & 7) * 2);
          *bh = pv;
        }
        *reinterpret_cast<__half*>(brow + swz(r, 0)) = __float2half(lo);
        *reinterpret_cast<__half*>(brow + swz(r, (2 * kclip) >> 3) + ((2 * kclip) & 7) * 2) =
            __float2half(hi);
      }
      if (r == 0) UA_TR(k, 11);
      fence_async_smem();   // P / B tiles (generic stores) -> the MMA (async proxy)
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (r == 0) UA_TR(k, 12);
      __syncwarp();
      if (lane == 0) mbar_arrive(&U.pfull[bf]);
      if (r == 0) UA_TR(k, 4);
      // epilogue: O / sum -> FP16 (query rows in [n, S) written as 0; rows >= S belong to
      // the next sentence)
      mbar_wait(&U.ofull[tb], (k / NTB) & 1);
      if (r == 0) UA_TR(k, 6);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float o[64];
      tmem_ld32(trow + 64, o);
      tmem_ld32(trow + 96, o + 32);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&U.tfree[tb]);
      if (r == 0) UA_TR(k, 7);
      if (item_ok && i < S) {
        const float inv = row_ok && sum > 0.f ? 1.f / sum : 0.f;
        uint4* orow = reinterpret_cast<uint4*>(out + ((size_t)b * S + i) * d + h * 64);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          orow[u] = make_uint4(pack_half2_sat(o[8 * u] * inv, o[8 * u + 1] * inv),
                               pack_half2_sat(o[8 * u + 2] * inv, o[8 * u + 3] * inv),
                               pack_half2_sat(o[8 * u + 4] * inv, o[8 * u + 5] * inv),
                               pack_half2_sat(o[8 * u + 6] * inv, o[8 * u + 7] * inv));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

constexpr size_t smem_bytes() { return 2 * SLOT + 2 * PT + 2 * BT + 2 * 32 * 128 + sizeof(USmem) + 1024; }

template <int SPP>
void launch(const __half* qkv, const int* len, const __half* relk, const __half* relv, __half* out,
            int B, int S, int d, int H, int kclip, cudaStream_t s) {
  static const bool attr = [] {
    NMT_CUDA(cudaFuncSetAttribute(k_attn_enc_umma<SPP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem_bytes()));
    return true;
  }();
  (void)attr;
  const CUtensorMap map = make_map(qkv, B * S, 3 * d, 3 * d, SPP);
  const int tiles = (B * H + (128 / SPP) - 1) / (128 / SPP);
  const int grid = std::min(tiles, num_sms());
  static const int trace = getenv("NMT_ATTN_TRACE") ? 1 : 0;   // debug timeline (CTA 0)
  launch_k(k_attn_enc_umma<SPP>, dim3(grid), dim3(kThreadsU), smem_bytes(), s, map, len, relk, relv,
           out, B, S, d, H, kclip, trace);
}

}  // namespace ua

void attn_umma_trace(unsigned long long* h_out, int cap) {
  NMT_CUDA(cudaDeviceSynchronize());
  NMT_CUDA(cudaMemcpyFromSymbol(h_out, ua::g_ua_trace, sizeof(unsigned long long) * std::min(cap, 64 * 16)));
}

// FP16, dh = 64, S <= 128, RPR on (the tables are required: zero tables give vanilla attention).
void attn_encoder_umma(const __half* qkv, const int* len, const __half* relk, const __half* relv,
                       __half* out, int B, int S, int d, int H, int kclip, cudaStream_t s) {
  if (d / H != 64 || S > 128 || kclip > 8 || kclip < 1 || !relk || !relv)
    throw CudaError("attn_encoder_umma: needs dh = 64, S <= 128, 1 <= k <= 8 and RPR tables");
  if (S <= 8) ua::launch<8>(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
  else if (S <= 16) ua::launch<16>(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
  else if (S <= 32) ua::launch<32>(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
  else if (S <= 64) ua::launch<64>(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
  else ua::launch<128>(qkv, len, relk, relv, out, B, S, d, H, kclip, s);
  NMT_LAUNCH_CHECK();
}

}  // namespace nmt
