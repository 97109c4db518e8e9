// gemm_tc.cu — FP16 tensor-core GEMM for sm_100a: tcgen05.mma (kind::f16, FP32 accumulator
// in TMEM), operands staged by TMA (cp.async.bulk.tensor, 128B swizzle) through an
// mbarrier ring.  Persistent and warp-specialised:
//   warp 0     TMA producer (one elected thread)
//   warp 1     MMA issuer (one thread), double-buffered TMEM accumulators so the
//              epilogue of unit i overlaps the main loop of unit i+1
//   warp 2     TMEM allocator
//   warps 4..7 epilogue: TMEM -> registers (tcgen05.ld) -> fused bias / residual / ReLU /
//              FP16 store, or the vocab argmax (packed atomicMax; logits never stored,
//              PAPER.md:143)
// C[M][N] = A[M][K] . B[N][K]^T.  Every projection of the path is one of these (QKV / out /
// FFN / cross-K/V / decoder / tied vocab projection).
// Optional deterministic split-K (decode GEMMs have few rows and few output tiles): every
// split writes an FP32 partial; the last split to arrive for a tile (atomic counter) sums
// the partials in split order 0..S-1 and runs the epilogue, so results do not depend on
// which CTA finishes last nor on the number of rows (batch invariance).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"
#include "tc_dev.cuh"

namespace nmt {
namespace tc {

// Debug timeline (NMT_GEMM_TRACE set at the launch; single-CTA units only): CTA c, local unit
// k < 32, 8 globaltimer stamps at g_gemm_trace[(c * 32 + k) * 8 + e]: 0 producer: first load
// of the unit issued, 1 producer: last load issued, 2 MMA: accumulator free (tempty), 3 MMA:
// last commit (tfull), 4 epilogue warp 4: starts waiting for tfull, 5 warp 4: tfull seen,
// 6 warp 4: accumulator released, 7 warp 4: last store of the unit issued.
__device__ unsigned long long g_gemm_trace[148 * 32 * 8];
__device__ __forceinline__ unsigned long long gt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GT(k, e)                                                                        \
  do {                                                                                  \
    if (p.trace && blockIdx.x < 148 && (k) < 32)                                        \
      g_gemm_trace[((size_t)blockIdx.x * 32 + (k)) * 8 + (e)] = gt_now();               \
  } while (0)

// PAIR = true: a CTA pair (cluster of 2 on one TPC) computes 256 x BN output units with
// tcgen05.mma.cta_group::2 (M = 256).  Each CTA stages its own 128 rows of A and BN/2 rows
// of B per k-block, so every SM moves (128 + BN/2) * BK * 2 bytes per 2*128*BN*BK FLOP —
// 1.5x the FLOP per staged byte of the single-CTA 128 x BN tile at BN = 256 (the encoder
// GEMMs at K = 512 are bound by L2 -> SM operand traffic).  The leader (rank 0) waits for
// both halves on its own `full` barrier (each CTA's TMA completes on it), issues the MMAs
// and multicasts its commits to both CTAs' `empty` / `tfull` barriers; both CTAs drain
// their own TMEM rows and release the accumulator on the leader's `tempty`.
// KS = 2: the split-K arithmetic of the cluster kernel below inside one persistent unit (two
// TMEM accumulators per unit over the two K halves, reduced (0 + p0) + p1 in FP32 before the
// epilogue): the large-row decode FFN2 keeps the association its small-row launches use.
// AM: the vocab argmax epilogue by chunk maxima (its own instantiation: the extra arrays
// would push the shared encoder-GEMM instantiation into spills).
// PL: plain FP16 epilogue (bias, ReLU, TMA stores; no residual / LN statistics / argmax),
// TMEM loads double-buffered: the next chunk's tcgen05.ld is in flight during this chunk's
// math and staging (the epilogue is a latency chain of ~4 dependent steps per chunk).
template <int BN, int STAGES, bool PAIR = false, int EW = 8, int NSTG = 1, bool BEAM = false,
          int KS = 1, bool AM = false, bool PL = false>
__global__ void __launch_bounds__(128 + 32 * EW, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapR,
              Params p) {
  using SM = Smem<BN, STAGES, PAIR, EW, NSTG>;
  constexpr int UM = PAIR ? 2 * BM : BM;             // output rows per unit
  constexpr uint32_t ACC_COLS = KS * BN;            // one accumulator = KS x BN FP32 columns
  // BN <= 256: two accumulators (the epilogue of unit i overlaps the MMAs of unit i+1);
  // BN = 512 fills TMEM with one (full-row tiles for the N = 512 projections: half the
  // units of BN = 256, so M = 16K..32K rows fit one or two waves of 148 SMs)
  constexpr int NACC = 2 * KS * BN <= 512 ? 2 : 1;
  constexpr int TC = NACC * KS * BN;
  constexpr uint32_t TMEM_COLS = TC <= 32 ? 32 : TC <= 64 ? 64 : TC <= 128 ? 128 : TC <= 256 ? 256 : 512;
  static_assert(KS == 1 || (!PAIR && !BEAM && KS == 2 && KS * BN <= 512), "KS = 2: single-CTA units");
  constexpr int BBOX = BN > 256 ? 256 : BN;         // TMA box rows of B (<= 256)
  static_assert(!(PAIR && BN > 256), "pair units use BN <= 256");
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on the __shared__ array: an integer round trip
  // would hide the address space (generic LD/ST instead of LDS/STS in the epilogue)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi = smem + STAGES * SM::STAGE;   // 1024-B aligned (STAGE is a multiple of 1024)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + SM::EPI);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained
  constexpr int NRB = NSTG > 2 ? NSTG : 2;
  uint64_t* rbar = tempty + 2;        // [EW][NRB] residual tile loaded (NSTG >= 2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + NRB * EW);

  const int kb_total = (p.K + BK - 1) / BK;
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  const int cid = PAIR ? (int)blockIdx.x >> 1 : (int)blockIdx.x;   // unit-stream index
  const int ncl = PAIR ? (int)gridDim.x >> 1 : (int)gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 * EW : EW);  // one arrive per epilogue warp (both CTAs)
    }
    for (int i = 0; i < NRB * EW; ++i) mbar_init(&rbar[i], 1);

    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync_all();  // peer barriers initialised before any remote use
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // dependents may launch once every CTA holds its TMEM (a dependent GEMM CTA allocating
  // on the same SM then waits for this one's dealloc, never the reverse)
  pdl_trigger();
  // Weight prefetch (B operand = weights, never written by the preceding kernels): with the
  // n-fastest unit order the first unit's column block (cid % num_n) does not depend on the
  // live-row count, so its first STAGES k-blocks of B are requested before the PDL wait
  // (expect_tx only; the producer's arrive.expect_tx for A completes the phase later).
  const int num_n = (p.N + BN - 1) / BN;
  int npre = 0;
  if constexpr (!PAIR) {
    if (warp == 0 && lane == 0 && p.nfast && p.bpre && !(p.dbg & 32)) {
      npre = kb_total < STAGES ? kb_total : STAGES;
      const int n0 = (cid % num_n) * BN;
      for (int st = 0; st < npre; ++st) {
        uint8_t* sb = smem + st * SM::STAGE + SM::A_BYTES;
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                         smem_u32(&full[st])),
                     "r"((uint32_t)SM::B_BYTES)
                     : "memory");
#pragma unroll
        for (int bo = 0; bo < BN; bo += BBOX)
          tma_load_2d(sb + bo * BK * 2, &mapB, &full[st], st * BK, n0 + bo);
      }
    }
  }
  // PDL: the setup above (barriers, tensor-map prefetch, TMEM allocation, weight prefetch)
  // overlaps the preceding kernel; its outputs (A, the live-row count) are read from here
  pdl_wait();
  const int M = p.dM ? min(p.M, *p.dM) : p.M;
  const int num_m = (M + UM - 1) / UM;
  const int units = num_m * num_n;   // CTAs with cid >= units skip to the teardown

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs of a pair)
      if (npre && cid >= units) {   // no work: let the prefetched weight tiles land, then exit
        for (int st = 0; st < npre; ++st) {
          mbar_arrive(&full[st]);
          mbar_wait(&full[st], 0);
        }
      }
      int it = 0, lu = 0;
      for (int u = cid; u < units; u += ncl, ++lu) {
        const int mi = p.nfast ? u / num_n : u % num_m, ni = p.nfast ? u % num_n : u / num_m;
        const int m0 = mi * UM + rank * BM, n0 = ni * BN + rank * (SM::BROWS);
        for (int kb = 0; kb < kb_total; ++kb, ++it) {
          if (kb == 1) GT(lu, 0);
          if (kb == kb_total - 1) GT(lu, 1);
          const int st = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* sa = smem + st * SM::STAGE;
          if constexpr (PAIR) {
            const uint32_t fb = mapa_u32(&full[st], 0);
            if (rank == 0) mbar_expect_tx(&full[st], 2 * SM::STAGE);
            tma_load_2d_pair(sa, &mapA, fb, kb * BK, m0);
            tma_load_2d_pair(sa + SM::A_BYTES, &mapB, fb, kb * BK, n0);
          } else {
            if ((p.dbg & 32) && it >= STAGES) {   // tuning: MMAs on stale tiles, no TMA
              mbar_arrive(&full[st]);
              continue;
            }
            if (it < npre) {   // B already requested before the PDL wait
              mbar_expect_tx(&full[st], SM::A_BYTES);
              tma_load_2d(sa, &mapA, &full[st], kb * BK, m0);
              continue;
            }
            mbar_expect_tx(&full[st], SM::STAGE);
            tma_load_2d(sa, &mapA, &full[st], kb * BK, m0);
#pragma unroll
            for (int bo = 0; bo < BN; bo += BBOX)
              tma_load_2d(sa + SM::A_BYTES + bo * BK * 2, &mapB, &full[st], kb * BK, n0 + bo);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (one thread; pair leader)
      constexpr uint32_t idesc = (1u << 4)                        // D = F32
                                 | (0u << 7) | (0u << 10)          // A, B = F16
                                 | ((uint32_t)(BBOX >> 3) << 17)   // N (per instruction)
                                 | ((uint32_t)(UM >> 4) << 24);    // M
      int it = 0, local = 0;
      for (int u = cid; u < units; u += ncl, ++local) {
        const int acc = NACC == 2 ? (local & 1) : 0;
        const uint32_t aph = NACC == 2 ? (local >> 1) & 1 : local & 1;
        mbar_wait(&tempty[acc], aph ^ 1);   // epilogue(s) drained this accumulator
        GT(local, 2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d0 = tmem + acc * ACC_COLS;
        const int kps = kb_total / KS;   // KS = 2: k-blocks [0, kps) -> d0, [kps, 2 kps) -> d0 + BN
        for (int kb = 0, first = 1; kb < kb_total; ++kb, ++it, first = 0) {
          if (KS == 2 && kb == kps) first = 1;
          const uint32_t d = d0 + (KS == 2 && kb >= kps ? BN : 0);
          const int st = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = make_desc_sw128(smem + st * SM::STAGE);
          const uint64_t db = make_desc_sw128(smem + st * SM::STAGE + SM::A_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {  // +32 B along K inside the swizzle atom
            const uint32_t accum = (first == 0 || kk > 0) ? 1u : 0u;
            if constexpr (PAIR) {
              mma_f16_pair(d, da + 2 * kk, db + 2 * kk, idesc, accum);
            } else {
#pragma unroll
              for (int bo = 0; bo < BN; bo += BBOX)   // N > 256: one MMA per 256-column half
                mma_f16(d + bo, da + 2 * kk, db + ((bo * BK * 2) >> 4) + 2 * kk, idesc, accum);
            }
          }
          if constexpr (PAIR) mma_commit_pair(&empty[st]);  // frees the stage in both CTAs
          else mma_commit(&empty[st]);
        }
        if constexpr (PAIR) mma_commit_pair(&tfull[acc]);
        else mma_commit(&tfull[acc]);
        GT(local, 3);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    // FP16 outputs leave through TMA stores: each warp converts 32 rows x 32 columns into
    // its 64-B-swizzled staging tile (conflict-free 16-B writes) and one lane issues the
    // bulk store (full-line writes instead of 32 scattered row segments per instruction).
    // EW warps = 4 TMEM lane quadrants x EW/4 column parts of HALF columns each
    const int e = warp - 4, q = warp & 3, half = e >> 2;
    constexpr int HALF = BN / (EW / 4), NPF = HALF <= 128 ? HALF / 8 : 1;
    uint8_t* stg0 = epi + e * NSTG * SM::STG;
    float* sbias = reinterpret_cast<float*>(epi + EW * NSTG * SM::STG);    // [kBiasMax]
    float* sb = sbias + kBiasMax + e * HALF;
    float* sc = sbias + kBiasMax + EW * HALF + e * HALF;
    // the whole bias vector once per CTA (read per unit otherwise: a global round trip)
    const bool bias_all = p.bias && p.N <= kBiasMax;
    if (bias_all) {
      for (int j = threadIdx.x - 128; j < p.N; j += 32 * EW) sbias[j] = __half2float(p.bias[j]);
      asm volatile("bar.sync 1, %0;" ::"r"(32 * EW) : "memory");
    }
    // residual through TMA (NSTG = 2, FP16 TMA-store outputs): the 32 x 32 residual block of
    // a chunk lands in the staging tile that then carries the chunk's output (in place)
    // NSTG = 4 (= the warp's chunks per unit): every residual block of the unit is requested
    // when the unit starts, so the loads overlap its main loop instead of one chunk each
    const bool rt = NSTG >= 2 && p.rtma;
    constexpr bool RALL = NSTG >= 4;
    static_assert(!RALL || BN / (EW / 4) / 32 <= NSTG, "one staging tile per chunk of the unit");
    uint32_t rph = 0;      // RALL: phase bit of each rbar of this warp
    uint32_t kchunk = 0;   // this warp's chunk counter (staging tile kchunk & 1)
    auto r_issue = [&](uint32_t k, int x, int y) {   // lane 0: TMA of a residual block
      if (lane == 0) {
        // tile k & 1 last carried chunk k - 2, whose store is the older of (at most) two
        // outstanding bulk groups
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        uint64_t* b = &rbar[2 * e + (k & 1)];
        mbar_expect_tx(b, SM::STG);
        tma_load_2d(stg0 + (k & 1) * SM::STG, &mapR, b, x, y);
      }
    };
    const uint32_t te0 = PAIR ? mapa_u32(&tempty[0], 0) : 0u, te1 = PAIR ? mapa_u32(&tempty[1], 0) : 0u;
    int local = 0;
    for (int u = cid; u < units; u += ncl, ++local) {
      const int mi = p.nfast ? u / num_n : u % num_m, ni = p.nfast ? u % num_n : u / num_m;
      const int m0 = mi * UM + rank * BM, n0 = ni * BN;
      const int acc = NACC == 2 ? (local & 1) : 0;
      const uint32_t aph = NACC == 2 ? (local >> 1) & 1 : local & 1;
      const int r = q * 32 + lane;
      const int m = m0 + r;
      const bool row_ok = m < M;
      const int cb = half * HALF;
      // residual rows and the bias slice fetched while the MMAs of this unit still run
      uint4 res[NPF];
      if constexpr (RALL) {
        if (rt && lane == 0) {
          bulk_wait_read0();   // the previous unit's stores have read every staging tile
          for (int j = 0; j * 32 < HALF && n0 + cb + j * 32 < p.N; ++j) {
            uint64_t* b = &rbar[NSTG * e + j];
            mbar_expect_tx(b, SM::STG);
            tma_load_2d(stg0 + j * SM::STG, &mapR, b, n0 + cb + j * 32, m0 + q * 32);
          }
        }
      } else if (rt && n0 + cb < p.N) {
        r_issue(kchunk, n0 + cb, m0 + q * 32);
      }
      const bool pf = !rt && HALF <= 128 && p.R && row_ok && n0 + cb + HALF <= p.N &&
                      ((reinterpret_cast<uintptr_t>(p.R + (size_t)m * p.ldr + n0 + cb) & 15) == 0);
      if (pf) {
        const uint4* rp = reinterpret_cast<const uint4*>(p.R + (size_t)m * p.ldr + n0 + cb);
#pragma unroll
        for (int i = 0; i < NPF; ++i) res[i] = rp[i];
      }
      __syncwarp();
      if (p.bias && !bias_all)
        for (int j = lane; j < HALF; j += 32) {
          const int n = n0 + cb + j;
          sb[j] = n < p.N ? __half2float(p.bias[n]) : 0.f;
        }
      float2 ln = make_float2(0.f, 0.f);
      if (p.ln_st) {
        for (int j = lane; j < HALF; j += 32) {
          const int n = n0 + cb + j;
          sc[j] = n < p.N ? p.ln_c[n] : 0.f;
        }
        if (row_ok) ln = merge_stats(p.ln_st + (size_t)m * (p.K / 32), p.K / 32, p.ln_eps);
      }
      __syncwarp();
      if (warp == 4 && lane == 0) GT(local, 4);
      mbar_wait(&tfull[acc], aph);
      if (warp == 4 && lane == 0) GT(local, 5);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + acc * ACC_COLS + ((uint32_t)(q * 32) << 16);
      unsigned long long best = 0ull;
      if constexpr (AM) {
        // vocab argmax: per 32-column chunk only its maximum (independent max ops), the
        // earliest chunk holding the row's maximum kept; then that chunk is read again from
        // TMEM for the lowest column equal to the maximum — the same (value, lowest id) as a
        // scan of every column, at about a third of the epilogue instructions
        float bestv = 0.f;
        int bestc = -1;
#pragma unroll
        for (int c0 = cb; c0 < cb + HALF; c0 += 32) {
          if (n0 + c0 >= p.N) break;   // warp-uniform
          float v[32];
          __syncwarp();
          tmem_ld32(tbase + c0, v);
          const int nv = min(32, p.N - (n0 + c0));
          float mx = v[0];
          if (nv == 32) {
            float m4[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) m4[j] = fmaxf(fmaxf(v[4 * j], v[4 * j + 1]), fmaxf(v[4 * j + 2], v[4 * j + 3]));
            mx = fmaxf(fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])),
                       fmaxf(fmaxf(m4[4], m4[5]), fmaxf(m4[6], m4[7])));
          } else {
#pragma unroll
            for (int j = 1; j < 32; ++j)
              if (j < nv) mx = fmaxf(mx, v[j]);
          }
          if (bestc < 0 || mx > bestv) {
            bestv = mx;
            bestc = c0;
          }
        }
        if (bestc >= 0) {   // warp-uniform (bestc >= 0 iff the warp's first chunk is inside N)
          // tcgen05.ld addresses are per warp: re-read every chunk some lane of this warp won
          // (usually one or two) and search it in the lanes that won it
          int bj = 0;
#pragma unroll 1
          for (int c0 = cb; c0 < cb + HALF; c0 += 32) {
            if (n0 + c0 >= p.N) break;
            if (!__ballot_sync(0xffffffffu, bestc == c0)) continue;
            float w[32];
            __syncwarp();
            tmem_ld32(tbase + c0, w);
            if (bestc == c0) {
              bj = 31;
#pragma unroll
              for (int j = 31; j >= 0; --j)
                if (w[j] == bestv) bj = j;
            }
          }
          best = pack_argmax(bestv, n0 + bestc + bj);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(acc ? te1 : te0);
          else mbar_arrive(&tempty[acc]);
        }
        if (row_ok && best) atomicMax(p.argmax + m, best);
        continue;
      }
      if constexpr (PL) {
        constexpr int NCH = HALF / 32;
        uint32_t rr[2][32];
        __syncwarp();
        tmem_ld32_nw(tbase + cb, rr[0]);
#pragma unroll
        for (int ci = 0; ci < NCH; ++ci) {
          const int c0 = cb + ci * 32;
          tmem_wait_ld(rr[ci & 1]);
          if (ci + 1 < NCH) {
            __syncwarp();
            tmem_ld32_nw(tbase + c0 + 32, rr[(ci + 1) & 1]);
          } else {   // every TMEM load of this warp has completed: release the accumulator
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              if constexpr (PAIR) mbar_arrive_cluster(acc ? te1 : te0);
              else mbar_arrive(&tempty[acc]);
              if (warp == 4) GT(local, 6);
            }
          }
          if (n0 + c0 >= p.N) continue;   // warp-uniform
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[ci & 1][j]);
          if (p.bias) {
            const float* bp = bias_all ? sbias + n0 + c0 : sb + (c0 - cb);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b = *reinterpret_cast<const float4*>(bp + j);
              v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
            }
          }
          uint32_t h[16];
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 16; ++i) h[i] = pack_half2_sat_relu(v[2 * i], v[2 * i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) h[i] = pack_half2_sat(v[2 * i], v[2 * i + 1]);
          }
          uint8_t* stg = stg0 + (NSTG == 2 ? (kchunk & 1) * SM::STG : 0);
          const int sw = (lane >> 1) & 3;
          if (lane == 0) {
            if constexpr (NSTG == 1) bulk_wait_read0();
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          }
          ++kchunk;
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((c ^ sw) << 4)) =
                make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&mapC, stg, n0 + c0, m0 + q * 32);
            bulk_commit();
          }
        }
        if (warp == 4 && lane == 0) GT(local, 7);
        continue;
      }
      BeamAcc bacc;
      if constexpr (BEAM) bacc.init();
#pragma unroll
      for (int c0 = cb; c0 < cb + HALF; c0 += 32) {
        float v[32];
        __syncwarp();
        tmem_ld32(tbase + c0, v);
        if constexpr (KS == 2) {   // the cluster kernel's reduction order: (0 + p0) + p1
          float v2[32];
          tmem_ld32(tbase + BN + c0, v2);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = 0.f + v[j];
            v[j] += v2[j];
          }
        }
        if (c0 + 32 >= cb + HALF) {  // this warp's columns read: release the accumulator
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_cluster(acc ? te1 : te0);
            else mbar_arrive(&tempty[acc]);
            if (warp == 4) GT(local, 6);
          }
        }
        if (p.dbg & 1) {
          if (v[0] == 1234.5f) p.C[0] = __float2half(v[1]);
        } else if (p.tstore) {
          if (n0 + c0 < p.N) {  // warp-uniform
            const bool rp = p.relu && !p.st_out;   // ReLU inside the pack instruction
            const int jc = (c0 - cb) >> 5;      // chunk of this warp's columns
            uint8_t* stg = stg0 + (RALL ? jc * SM::STG : NSTG == 2 ? (kchunk & 1) * SM::STG : 0);
            const int sw = (lane >> 1) & 3;     // 64-B swizzle: 16-B chunk c at c ^ ((row >> 1) & 3)
            if (!(p.dbg & 8))
              epi_math(p, m, n0 + c0, v, bias_all ? sbias + n0 + c0 : sb + (c0 - cb),
                       pf ? res + (c0 - cb) / 8 : nullptr, row_ok && !rt, sc + (c0 - cb), ln, rp);
            if (rt) {   // + residual (same order as the register path: after bias)
              if constexpr (RALL) {
                mbar_wait(&rbar[NSTG * e + jc], (rph >> jc) & 1);
                rph ^= 1u << jc;
              } else {
                mbar_wait(&rbar[2 * e + (kchunk & 1)], (kchunk >> 1) & 1);
              }
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const uint4 w4 = *reinterpret_cast<const uint4*>(stg + lane * 64 + ((c ^ sw) << 4));
                add_h2(w4.x, v[8 * c + 0], v[8 * c + 1]);
                add_h2(w4.y, v[8 * c + 2], v[8 * c + 3]);
                add_h2(w4.z, v[8 * c + 4], v[8 * c + 5]);
                add_h2(w4.w, v[8 * c + 6], v[8 * c + 7]);
              }
            }
            if (p.st_out && row_ok) p.st_out[(size_t)m * (p.N / 32) + (n0 + c0) / 32] = chunk_stats(v);
            uint32_t h[16];
            if (rp) {
#pragma unroll
              for (int i = 0; i < 16; ++i) h[i] = pack_half2_sat_relu(v[2 * i], v[2 * i + 1]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) h[i] = pack_half2_sat(v[2 * i], v[2 * i + 1]);
            }
            if (p.dbg & 4) {  // tuning: no staging / store
              uint32_t x = 0;
#pragma unroll
              for (int i = 0; i < 16; ++i) x ^= h[i];
              if (x == 0x12345678u) p.C[0] = __float2half(1.f);
              continue;
            }
            if (lane == 0) {   // the store that last used this staging tile has read it
              if constexpr (NSTG == 1) {
                bulk_wait_read0();
              } else if constexpr (RALL) {   // tile jc: last written NSTG chunks (groups) ago
                if (!rt) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NSTG - 1) : "memory");
              } else if (!rt) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              }
            }
            ++kchunk;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 4; ++c)
              *reinterpret_cast<uint4*>(stg + lane * 64 + ((c ^ sw) << 4)) =
                  make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
            fence_async_smem();
            __syncwarp();
            if (lane == 0 && !(p.dbg & 2)) {  // rows >= M / columns >= N clipped by the map
              tma_store_2d(&mapC, stg, n0 + c0, m0 + q * 32);
              bulk_commit();
            }
            if (!RALL && rt && c0 + 32 < cb + HALF && n0 + c0 + 32 < p.N)   // next chunk's residual
              r_issue(kchunk, n0 + c0 + 32, m0 + q * 32);         // (kchunk already advanced)
          }
        } else if (row_ok && n0 + c0 < p.N) {
          epi_math(p, m, n0 + c0, v, bias_all ? sbias + n0 + c0 : sb + (c0 - cb),
                   pf ? res + (c0 - cb) / 8 : nullptr, true, sc + (c0 - cb), ln);
          if (p.st_out) p.st_out[(size_t)m * (p.N / 32) + (n0 + c0) / 32] = chunk_stats(v);
          if constexpr (BEAM) bacc.add(v, n0 + c0, min(32, p.N - (n0 + c0)));
          else epi_out(p, m, n0 + c0, v, best);
        }
      }
      // RALL: a unit that stored fewer than NSTG chunks (N edge) drains its stores, so every
      // staging tile is again last written NSTG groups back
      if (RALL && p.tstore && !rt && lane == 0 && n0 + cb + HALF > p.N) bulk_wait_read0();
      if (warp == 4 && lane == 0) GT(local, 7);
      if (p.argmax && row_ok && best) atomicMax(p.argmax + m, best);
      if (BEAM && row_ok && n0 + cb < p.N) {   // this thread's segment of the row
        const int nseg = (p.N + HALF - 1) / HALF;
        bacc.store(p.bpart + ((size_t)m * nseg + (n0 + cb) / HALF) * kBeamRec);
      }
    }
    // the staging tiles must outlive the bulk stores' shared-memory reads; the global
    // writes complete with the grid (kernel boundary / PDL wait of the dependent)
    if (p.tstore && lane == 0) bulk_wait_read0();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync_all();  // the peer's MMAs / remote arrives are done
  else __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ cluster split-K
// Decode-size GEMMs (rows = live batch rows <= a few hundred): one 128 x 64 output tile is
// computed by a thread-block CLUSTER of S CTAs, CTA s accumulating k-blocks
// [s*kps, (s+1)*kps) in its own TMEM.  Partials are exchanged through distributed shared
// memory (no global round trip, no atomics): after a cluster barrier, CTA c reduces rows
// [c*128/S, (c+1)*128/S) by reading the S partials in split order 0..S-1 (deterministic,
// independent of the row count) and applies the fused epilogue.
__device__ __forceinline__ float4 ld_dsmem_f4(const float* local_addr, uint32_t rank) {
  uint32_t a = smem_u32(local_addr), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(ra)
               : "memory");
  return v;
}

// Epilogue for 16 consecutive columns (n0 % 16 == 0 assumed for the vector paths).
__device__ __forceinline__ void epilogue16(const Params& p, int m, int nb, float* v) {
  const int nv = min(16, p.N - nb);
  const bool full = nv == 16;
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nv) v[j] += __half2float(p.bias[nb + j]);
  }
  if (p.R) {
    const __half* rr = p.R + (size_t)m * p.ldr + nb;
    if (full && ((reinterpret_cast<uintptr_t>(rr) & 15) == 0)) {
      float f[8];
      load8h(rr, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += f[e];
      load8h(rr + 8, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[8 + e] += f[e];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nv) v[j] += __half2float(rr[j]);
    }
  }
  if (p.relu) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  __half* cr = p.C + (size_t)m * p.ldc + nb;
  if (full && ((reinterpret_cast<uintptr_t>(cr) & 15) == 0)) {
#pragma unroll
    for (int j8 = 0; j8 < 2; ++j8) {
      uint4 pk;
      __half2* h2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        h2[e] = __halves2half2(from_f<__half>(v[j8 * 8 + 2 * e]), from_f<__half>(v[j8 * 8 + 2 * e + 1]));
      reinterpret_cast<uint4*>(cr)[j8] = pk;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nv) cr[j] = from_f<__half>(v[j]);
  }
}

// 256 threads (warps 0-2 as in k_gemm_tc, warps 4-7 drain TMEM), a few stages, and the
// FP32 partial aliased onto the drained stage buffers: small enough for several CTAs per SM,
// so a decode GEMM's clusters run in one wave next to the other workers' kernels.
constexpr int kCThreads = 256;
template <int STAGES>
__global__ void __launch_bounds__(kCThreads, 3)
    k_gemm_tc_cluster(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB, Params p) {
  constexpr int BN = 64;
  using SM = Smem<BN, STAGES>;
  constexpr int LDP = BN + 4;  // padded FP32 partial row (conflict-light float4 stores)
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on the __shared__ array: an integer round trip
  // would hide the address space (generic LD/ST instead of LDS/STS in the epilogue)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // [BM][LDP] FP32 partial, written after the last MMA has drained every stage buffer
  float* part = reinterpret_cast<float*>(smem);
  static_assert(BM * LDP * 4 <= STAGES * SM::STAGE, "partial must fit in the stage buffers");
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SM::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int S = p.splits;
  const int s = (int)cluster_ctarank();          // split index == rank in the cluster
  const int tile = blockIdx.x / S;
  const int num_m = (p.M + BM - 1) / BM;         // grid sized by the host upper bound
  const int m0 = (tile % num_m) * BM, n0 = (tile / num_m) * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Barriers and the TMEM allocation come BEFORE the PDL trigger, in every CTA: a dependent
  // launched after the trigger may allocate all 512 columns on this SM and then block in its
  // griddepcontrol.wait for this grid, so allocating after the trigger can deadlock.
  if (warp == 0 && lane == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  pdl_trigger();
  pdl_wait();
  const int Meff = p.dM ? min(p.M, *p.dM) : p.M;
  const bool live = m0 < Meff;                   // uniform across the cluster
  const int kb_total = (p.K + BK - 1) / BK;
  const int kps = kb_total / S;

  if (live) {
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
      if (lane == 0) {
        for (int i = 0; i < kps; ++i) {
          const int kb = s * kps + i, st = i % STAGES;
          const uint32_t ph = (i / STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* sa = smem + st * SM::STAGE;
          mbar_expect_tx(&full[st], SM::STAGE);
          tma_load_2d(sa, &mapA, &full[st], kb * BK, m0);
          tma_load_2d(sa + SM::A_BYTES, &mapB, &full[st], kb * BK, n0);
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
        for (int i = 0; i < kps; ++i) {
          const int st = i % STAGES;
          const uint32_t ph = (i / STAGES) & 1;
          mbar_wait(&full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = make_desc_sw128(smem + st * SM::STAGE);
          const uint64_t db = make_desc_sw128(smem + st * SM::STAGE + SM::A_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk)
            mma_f16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[st]);
        }
        mma_commit(tfull);
      }
    } else if (warp >= 4 && warp < 8) {  // TMEM -> FP32 partial in this CTA's shared memory
      mbar_wait(tfull, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int q = warp & 3, r = q * 32 + lane;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(part + r * LDP + c0 + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  cluster_sync_all();  // every split's partial is in its shared memory
  if (live) {
    // CTA s reduces rows [s*BM/S, (s+1)*BM/S) of the tile: (row, 16-column group) per item
    const int rows = BM / S;
    for (int it = threadIdx.x; it < rows * (BN / 16); it += kCThreads) {
      const int rr = s * rows + it / (BN / 16), cg = (it % (BN / 16)) * 16;
      const int m = m0 + rr, nb = n0 + cg;
      if (m >= Meff || nb >= p.N) continue;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
      for (int sp = 0; sp < S; ++sp) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 f = ld_dsmem_f4(part + rr * LDP + cg + j, (uint32_t)sp);
          v[j] += f.x; v[j + 1] += f.y; v[j + 2] += f.z; v[j + 3] += f.w;
        }
      }
      epilogue16(p, m, nb, v);
    }
  }
  cluster_sync_all();  // keep shared memory alive until every CTA has read it
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot),
                 "r"(64));
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    NMT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

struct MapKey {
  const void* p;
  int rows, cols, ld, box;
  bool out;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box &&
           out == o.out;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.p);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull + ((size_t)k.cols << 20) + ((size_t)k.ld << 40) +
         (size_t)k.box + (k.out ? 0x5bd1e995ull : 0ull);
    return h;
  }
};

// Operand maps: box {BK, box_rows}, 128-B swizzle (UMMA K-major layout).  Output maps
// (out = true): box {32, 32}, 64-B swizzle (the epilogue's staging tile).
CUtensorMap encode_map(const void* ptr, int rows, int cols, int ld, int box_rows, bool out) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)(out ? 32 : BK), (cuuint32_t)(out ? 32 : box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            out ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// Tensor maps are pure functions of (pointer, shape, box): cache them (the arena and the
// weights never move), so a steady-state launch does no host-side encoding.
CUtensorMap make_map(const void* ptr, int rows, int cols, int ld, int box_rows, bool out) {
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  static std::mutex mu;
  MapKey k{ptr, rows, cols, ld, box_rows, out};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(k);
  if (it != cache.end()) return it->second;
  if (cache.size() > 65536) cache.clear();
  CUtensorMap m = encode_map(ptr, rows, cols, ld, box_rows, out);
  cache.emplace(k, m);
  return m;
}

// The TMA-store epilogue serves plain FP16 outputs (else mapC is unused).  With a device
// row count dM it also writes the rows of the last live tile beyond dM (up to the host
// bound M): those rows are dead (compacted away by pruning) and never read as live data.
CUtensorMap out_map(const GemmArgs& a, Params& p) {
  p.tstore = getenv("NMT_NO_TSTORE") == nullptr && a.C && !a.argmax && !a.logits &&
             (a.ldc % 8) == 0 && (a.N % 8) == 0 && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
  if (!p.tstore) return CUtensorMap{};
  return make_map(a.C, a.M, a.N, a.ldc, 32, true);
}

int num_sms() {
  static const int n = [] {
    int dev = 0, c = 0;
    NMT_CUDA(cudaGetDevice(&dev));
    NMT_CUDA(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev));
    return c;
  }();
  return n;
}

template <int BN, int STAGES, int EW = 8, int NSTG = 1, bool BEAM = false, int KS = 1, bool AM = false,
          bool PL = false>
void launch(const GemmArgs& a, cudaStream_t s) {
  using SM = Smem<BN, STAGES, false, EW, NSTG>;
  static_assert(SM::BYTES <= 227 * 1024, "shared memory over the sm_100 per-CTA limit");
  // thread-safe one-time attribute setup (C++11 static initialisation)
  static const bool attr = [&] {
    NMT_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, STAGES, false, EW, NSTG, BEAM, KS, AM, PL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES));
    return true;
  }();
  (void)attr;
  if (a.splits != KS) throw CudaError("gemm_tc: split count / kernel mismatch");
  if (KS > 1 && ((a.K + BK - 1) / BK) % KS) throw CudaError("gemm_tc: k-blocks not divisible by the splits");
  CUtensorMap ma = make_map(a.A, a.M, a.K, a.lda, BM);
  CUtensorMap mb = make_map(a.B, a.N, a.K, a.ldb, BN > 256 ? 256 : BN);
  Params p{};
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.bias = static_cast<const __half*>(a.bias);
  p.R = static_cast<const __half*>(a.R);
  p.ldr = a.ldr;
  p.C = static_cast<__half*>(a.C);
  p.ldc = a.ldc;
  p.relu = a.relu;
  p.dM = a.dM;
  p.argmax = a.argmax;
  p.logits = a.logits;
  p.bpart = a.beam_part;
  p.splits = 1;
  p.st_out = a.st_out;
  p.ln_st = a.ln_st;
  p.ln_c = a.ln_c;
  p.ln_eps = a.ln_eps;
  p.dbg = getenv("NMT_GEMM_DBG") ? atoi(getenv("NMT_GEMM_DBG")) : 0;
  static const bool trace = getenv("NMT_GEMM_TRACE") != nullptr;   // debug timeline only
  p.trace = trace && !BEAM;
  static const bool morder = getenv("NMT_GEMM_ORDER") && getenv("NMT_GEMM_ORDER")[0] == 'm';  // A/B only
  p.nfast = !morder;
  static const bool no_bpre = getenv("NMT_NO_BPRE") != nullptr;   // A/B only
  p.bpre = !no_bpre;
  const int units = ceil_div(a.M, BM) * ceil_div(a.N, BN);
  static const int cap = getenv("NMT_GEMM_GRID_CAP") ? atoi(getenv("NMT_GEMM_GRID_CAP")) : 0;  // tuning
  const int grid = std::min(units, cap > 0 && !a.dM ? cap : num_sms());  // persistent: one CTA per SM
  const CUtensorMap mc = out_map(a, p);
  static const bool no_rtma = getenv("NMT_NO_RTMA") != nullptr;   // A/B only
  p.rtma = NSTG >= 2 && p.tstore && a.R && !a.ln_st && !a.relu && (a.ldr % 8) == 0 &&
           (reinterpret_cast<uintptr_t>(a.R) & 15) == 0 && !no_rtma;
  const CUtensorMap mr = p.rtma ? make_map(a.R, a.M, a.N, a.ldr, 32, true) : CUtensorMap{};
  if (PL && (a.R || a.ln_st || a.st_out || !p.tstore)) throw CudaError("gemm_tc: plain epilogue misuse");
  launch_k(k_gemm_tc<BN, STAGES, false, EW, NSTG, BEAM, KS, AM, PL>, grid, 128 + 32 * EW, SM::BYTES, s, ma, mb, mc, mr, p);
  NMT_LAUNCH_CHECK();
}

// CTA-pair launch: clusters of 2 (one TPC), persistent over 256 x BN units.
template <int BN, int STAGES, int EW = 8, bool PL = false, bool AM = false>
void launch_pair(const GemmArgs& a, cudaStream_t s) {
  using SM = Smem<BN, STAGES, true, EW>;
  static_assert(SM::BYTES <= 227 * 1024, "shared memory over the sm_100 per-CTA limit");
  // thread-safe one-time attribute setup (C++11 static initialisation)
  static const bool attr = [&] {
    NMT_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, STAGES, true, EW, 1, false, 1, AM, PL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES));
    return true;
  }();
  (void)attr;
  CUtensorMap ma = make_map(a.A, a.M, a.K, a.lda, BM);
  CUtensorMap mb = make_map(a.B, a.N, a.K, a.ldb, BN / 2);
  Params p{};
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.bias = static_cast<const __half*>(a.bias);
  p.R = static_cast<const __half*>(a.R);
  p.ldr = a.ldr;
  p.C = static_cast<__half*>(a.C);
  p.ldc = a.ldc;
  p.relu = a.relu;
  p.dM = a.dM;
  p.argmax = a.argmax;
  p.logits = a.logits;
  p.bpart = a.beam_part;
  p.splits = 1;
  p.st_out = a.st_out;
  p.ln_st = a.ln_st;
  p.ln_c = a.ln_c;
  p.ln_eps = a.ln_eps;
  p.dbg = getenv("NMT_GEMM_DBG") ? atoi(getenv("NMT_GEMM_DBG")) : 0;
  static const bool trace = getenv("NMT_GEMM_TRACE") != nullptr;   // debug timeline only
  p.trace = trace;
  p.nfast = 1;
  const int units = ceil_div(a.M, 2 * BM) * ceil_div(a.N, BN);
  const int pairs = std::min(units, num_sms() / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(128 + 32 * EW);
  cfg.dynamicSmemBytes = SM::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  const CUtensorMap mc = out_map(a, p);
  if (PL && (a.R || a.ln_st || a.st_out || !p.tstore)) throw CudaError("gemm_tc: plain epilogue misuse");
  NMT_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_tc<BN, STAGES, true, EW, 1, false, 1, AM, PL>, ma, mb, mc,
                              CUtensorMap{}, p));
  NMT_LAUNCH_CHECK();
}

void launch_cluster(const GemmArgs& a, cudaStream_t s) {
  constexpr int STAGES = 3;
  using SM = Smem<64, STAGES>;
  const int bytes = SM::BYTES;
  // thread-safe one-time attribute setup (C++11 static initialisation)
  static const bool attr = [&] {
    NMT_CUDA(cudaFuncSetAttribute(k_gemm_tc_cluster<STAGES>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    NMT_CUDA(cudaFuncSetAttribute(k_gemm_tc_cluster<STAGES>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return true;
  }();
  (void)attr;
  const int S = a.splits;
  if (((a.K + BK - 1) / BK) % S || BM % S) throw CudaError("gemm_tc: bad cluster split");
  CUtensorMap ma = make_map(a.A, a.M, a.K, a.lda, BM);
  CUtensorMap mb = make_map(a.B, a.N, a.K, a.ldb, 64);
  Params p{};
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.bias = static_cast<const __half*>(a.bias);
  p.R = static_cast<const __half*>(a.R);
  p.ldr = a.ldr;
  p.C = static_cast<__half*>(a.C);
  p.ldc = a.ldc;
  p.relu = a.relu;
  p.dM = a.dM;
  p.splits = S;
  const int tiles = ceil_div(a.M, BM) * ceil_div(a.N, 64);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles * S);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  NMT_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_tc_cluster<STAGES>, ma, mb, p));
  NMT_LAUNCH_CHECK();
}

void gemm_trace(unsigned long long* h_out, int cap) {
  NMT_CUDA(cudaDeviceSynchronize());
  NMT_CUDA(cudaMemcpyFromSymbol(h_out, g_gemm_trace,
                                sizeof(unsigned long long) * std::min(cap, 148 * 32 * 8)));
}

}  // namespace tc

int decode_splits(int N, int K) {
  const int kb = (K + tc::BK - 1) / tc::BK, n_tiles = (N + 63) / 64;
  int sp = 1;
  while (sp * 2 <= 8 && kb % (sp * 2) == 0 && kb / (sp * 2) >= 2 && n_tiles * sp < 64) sp *= 2;
  return sp;
}

// Decode GEMMs (rows = live batch rows): the configuration depends on the weight shape
// only, never on the row count, so every output row is computed the same way whatever the
// batch (batch invariance).  Measured in captured graphs (tools/dec_gemm_sweep.py, 35-1
// shapes at 32 / 256 / 1024 rows, us per GEMM):
//   N = K = 512 (self-out, cross-q, cross-out): 128x128 7.0-7.4, 64-wide tiles 5.9-6.3
//   K = 2048 (FFN2): 128x128 14.1-14.7, cluster split-K 2 9.2-11.1, split 4 7.6-14.5
//   N = 1536 / 2048, K = 512 (QKV, FFN1): 128x128 6.9-8.0, 64-wide 6.0-9.4 (worse at 1024)
// so: 64-wide tiles for the square projections, split-K 2 through a thread-block cluster for
// K >= 2048 (no LN-statistics output there), 128x128 otherwise.  The per-GEMM floor of
// ~6 us is the dependent TMA round trips of the K loop plus launch and epilogue.
// Above 2048 rows (the host bound of the launch: the graph bucket) the tiles widen
// (graph-timed at 4096 / 8192 rows: QKV 13.9 -> 13.2 / 22.2 -> 17.4, FFN1 17.0 -> 13.6 /
// 26.2 -> 20.5, square 9.9 -> 8.0 (128) / 15.7 -> 10.4 (256), FFN2 25.4 / 49.0 in the
// cluster kernel): the output tile shape does not change any result (each output element
// is the same K-ordered MMA accumulation in every tile; tools/tile_identity.py checks it
// bit for bit), and FFN2 keeps its split-K association in the persistent kernel's KS = 2
// units, so batch invariance holds across the switch.
// NMT_DEC_TILE / NMT_DEC_SPLITS / NMT_DEC_POLICY=old override for tuning experiments.
void decode_config(GemmArgs& a) {
  static const int env_tile = getenv("NMT_DEC_TILE") ? atoi(getenv("NMT_DEC_TILE")) : 0;
  static const int env_splits = getenv("NMT_DEC_SPLITS") ? atoi(getenv("NMT_DEC_SPLITS")) : 0;
  static const bool old = getenv("NMT_DEC_POLICY") && std::string(getenv("NMT_DEC_POLICY")) == "old";
  a.splits = 1;
  if (env_splits > 1) {
    a.tile_n = 64;
    a.splits = env_splits;
  } else if (env_tile || old) {
    a.tile_n = env_tile ? env_tile : 128;
  } else if (a.K >= 2048 && !a.st_out && !a.ln_st && ((a.K + 63) / 64) % 2 == 0) {
    a.tile_n = a.M > 2048 ? 256 : 64;
    a.splits = 2;
  } else if (a.N <= 512 && a.K <= 512) {
    a.tile_n = a.M > 4096 ? 256 : a.M > 2048 ? 128 : 64;
  } else {
    a.tile_n = a.M >= 2048 ? 256 : 128;
  }
}

void gemm_tc(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.beam_part) {   // beam epilogue: 128 x 256 units, one 256-column segment per row
    if (a.logits || a.argmax || a.C || a.bias || a.R) throw CudaError("gemm_tc: beam epilogue is exclusive");
    // 4 epilogue warps: 256-column segments per thread, and the registers of a 256-thread
    // CTA keep the running top-8 without spills
    tc::launch<256, 4, 4, 1, true>(a, s);
    return;
  }
  if ((a.K % 8) || (a.lda % 8) || (a.ldb % 8) ||
      (reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(a.B) & 15))
    throw CudaError("gemm_tc: K / leading dims must be multiples of 8 and 16-B aligned");
  if ((a.st_out && a.N % 32) || (a.ln_st && (a.K % 32 || !a.ln_c)) ||
      ((a.st_out || a.ln_st) && a.splits > 1))
    throw CudaError("gemm_tc: LN folding needs N, K % 32 == 0 and the persistent kernel");
  if (a.tile_n == 256 && a.splits == 2) {
    tc::launch<256, 4, 8, 1, false, 2>(a, s);   // split-K association in persistent units
  } else if (a.splits > 1 && a.tile_n != 64) {
    throw CudaError("gemm_tc: split-K needs 64-wide cluster tiles or 256-wide KS = 2 units");
  } else if (a.tile_n == 64 && a.splits > 1) {
    tc::launch_cluster(a, s);   // split-K reduced through distributed shared memory
  } else if (a.tile_n == 64) {
    tc::launch<64, 4>(a, s);
  } else if (a.tile_n == 128) {
    tc::launch<128, 4, 8, 2>(a, s);
  } else if (const char* e = getenv("NMT_GEMM_CFG")) {  // tuning experiments only
    const std::string c(e);
    if (c == "128x4") tc::launch<128, 4>(a, s);
    else if (c == "256x3") tc::launch<256, 3>(a, s);
    else if (c == "256x3w16") tc::launch<256, 3, 16>(a, s);
    else if (c == "128x4w16") tc::launch<128, 4, 16>(a, s);
    else if (c == "pair256x4") tc::launch_pair<256, 4>(a, s);
    else if (c == "pair256x5") tc::launch_pair<256, 5>(a, s);
    else if (c == "pair256x6") tc::launch_pair<256, 6>(a, s);
    else if (c == "pair256x5w16") tc::launch_pair<256, 5, 16>(a, s);
    else if (c.rfind("pl", 0) == 0 && (a.R || a.ln_st || a.st_out || a.argmax || a.logits || !a.C))
      tc::launch<256, 4>(a, s);   // plain-epilogue configs apply to plain GEMMs only
    else if (c == "pl256x4") tc::launch<256, 4, 8, 1, false, 1, false, true>(a, s);
    else if (c == "plpair256x5") tc::launch_pair<256, 5, 8, true>(a, s);
    else if (c == "plpair256x6") tc::launch_pair<256, 6, 8, true>(a, s);
    else if (c == "pair256x4w16") tc::launch_pair<256, 4, 16>(a, s);
    else if (c == "512x2") tc::launch<512, 2>(a, s);
    else if (c == "256x3d") tc::launch<256, 3, 8, 2>(a, s);
    else if (c == "256x3q") tc::launch<256, 3, 8, 4>(a, s);
    else if (c == "256x2q") tc::launch<256, 2, 8, 4>(a, s);
    else tc::launch<256, 4>(a, s);
  } else if (a.R && a.K >= 2048 && !a.ln_st && !a.st_out && !a.relu && !a.dM &&
             !getenv("NMT_NO_PAIR_FFN2")) {
    // encoder FFN2 (K = 2048, residual): 256 x 256 units over a CTA pair (cta_group::2, each
    // CTA stages half of the B tile), 5 stages: 129 -> 121 us at M = 65520
    // (tools/gemm_bench.py); chosen from the weight shape only (batch invariance)
    tc::launch_pair<256, 5>(a, s);
  } else if (!a.R && !a.ln_st && !a.st_out && !a.argmax && !a.logits && !a.dM && a.C &&
             (a.ldc % 8) == 0 && (a.N % 8) == 0 && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 &&
             !getenv("NMT_NO_PLAIN_PAIR")) {
    // encoder QKV / FFN1 / cross K/V (bias, ReLU, FP16 out): 256 x 256 CTA-pair units with the
    // plain double-buffered-TMEM epilogue (tools/gemm_trace.py: the GEMMs are bound by shared-
    // memory traffic; a pair stages half the B tile per CTA): QKV 103.7 -> 99.6, FFN1 135.2 ->
    // 127.7, cross K/V 71.6 -> 69.5 us at M = 65520; chosen from the shape only
    tc::launch_pair<256, 5, 8, true>(a, s);
  } else if (a.R && a.K <= 512 && !a.ln_st && !a.relu) {
    // residual GEMM with a short main loop (attention output projection): 3 stages and two
    // staging tiles per epilogue warp, the residual blocks TMA-loaded ahead of their chunk
    // (measured 36.1 -> 30.9 us at 32768 rows; the 4-stage kernel wins everywhere else);
    // four staging tiles per warp: all four residual blocks of a unit requested at its start
    static const bool r2 = getenv("NMT_OUT_NSTG2") != nullptr;   // A/B only
    if (r2) tc::launch<256, 3, 8, 2>(a, s);
    else tc::launch<256, 3, 8, 4>(a, s);
  } else if (a.argmax && !a.logits && !a.C && !a.bias && !a.R && !a.ln_st &&
             !getenv("NMT_ARGMAX_SCAN")) {
    // vocab projection + argmax: the chunk-maximum epilogue (NMT_ARGMAX_SCAN: per-column
    // scan, A/B only).  CTA-pair units measured 7-8 % faster (NMT_PAIR_VOCAB=1, A/B only) but
    // stay opt-in: a full bench run with them in the PDL-chained decode graphs hung once
    static const bool pair = getenv("NMT_PAIR_VOCAB") != nullptr;
    if (pair) tc::launch_pair<256, 5, 8, false, true>(a, s);
    else tc::launch<256, 4, 8, 1, false, 1, true>(a, s);
  } else {
    // 128 x 256 tiles: 85 FLOP per staged byte at K = 512 (64 for 128 x 128)
    tc::launch<256, 4>(a, s);
  }
}

}  // namespace nmt
