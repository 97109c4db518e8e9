// beam.cu — batched beam search on the device ("the search ends when any
// candidate predicts the EOS symbol, and there are no candidates with higher scores";
// reading R15/R16: fairseq-style 2K candidates, unnormalised sum of log-probabilities).
//
// Layout: the live rows of a batch are grouped per sentence, K consecutive rows each
// (row r -> sentence group r / K).  Row r owns a physical cache slot row_slot[r]
// (= sentence_slot*K + k, fixed); beam re-ordering never copies K/V: each slot keeps an
// ancestry table anc[slot][j] = physical slot holding position j of its hypothesis, and a
// token history htok[slot][j] (j = 0 is BOS).  The self-attention kernel reads position j
// < t through anc (CopyBlocks-free beam reorder).
//
// Step t: vocab GEMM -> FP32 logits [rows][V];  k_beam_row_topk: per row LSE and the top-2K
// log-probs (value desc, id asc);  k_beam_select: per sentence the top-2K of the K x 2K
// candidates ordered by (score desc, slot*V + v asc), EOS candidates ranked < K finalise
// (best kept, ties -> earliest), the first K non-EOS become the new rows, actives are
// finalised at the cap, early stop when best finished >= best active.
#include "common.cuh"
#include "kernels.h"

namespace nmt {

constexpr int kKB = 8;  // candidates kept per row (= 2 * max beam 4)

// ------------------------------------------------------------------ per-row top-K + LSE
__device__ __forceinline__ bool cand_better(float a, int ia, float b, int ib) {
  return a > b || (a == b && ia < ib);
}

// Two passes over the row (L2-resident after the first): pass 1 keeps per thread only the
// running (max, sum exp) and its maximum's id — no per-element insertion, no divergence; the
// KB-th largest of the 256 thread maxima is a lower bound tau on the row's KB-th largest
// value, so pass 2 appends the few elements >= tau to shared memory and warp 0 selects the
// top-KB (value desc, id asc) from them.  Rows with more than kCandCap elements >= tau
// (massive ties) fall back to a block-wide selection over the whole row.
constexpr int kCandCap = 1024;
__global__ void __launch_bounds__(256) k_beam_row_topk(const float* __restrict__ logits, int V,
                                                       int KB, const int* __restrict__ dR,
                                                       float* __restrict__ cand_v,
                                                       int* __restrict__ cand_i) {
  const int row = blockIdx.x;
  if (row >= *dR) return;
  const float* x = logits + (size_t)row * V;
  float m = -INFINITY, s = 0.f;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float f = x[v];
    if (f > m) { s = s * __expf(m - f) + 1.f; m = f; }
    else s += __expf(f - m);
  }
  __shared__ float sm_m[8], sm_s[8], s_tmax[256];
  __shared__ float s_cv[kCandCap];
  __shared__ int s_ci[kCandCap];
  __shared__ int s_n;
  __shared__ float s_tau, s_lse;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  s_tmax[threadIdx.x] = m;
  if (threadIdx.x == 0) s_n = 0;
  {
    float mm = m;
    for (int o = 16; o; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
    float ss = (m == -INFINITY) ? 0.f : s * __expf(m - mm);
    ss = warp_sum(ss);
    if (lane == 0) { sm_m[warp] = mm; sm_s[warp] = ss; }
  }
  __syncthreads();
  if (warp == 0) {
    float mm = lane < 8 ? sm_m[lane] : -INFINITY;
    float M = mm;
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float ss = (lane < 8 && mm > -INFINITY) ? sm_s[lane] * __expf(mm - M) : 0.f;
    ss = warp_sum(ss);
    // tau = KB-th largest thread maximum: KB rounds of warp max over 8 maxima per lane
    float t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = s_tmax[lane * 8 + q];
    float tau = -INFINITY;
    for (int k = 0; k < KB; ++k) {
      float bv = -INFINITY;
      int bq = -1;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (t[q] > bv) { bv = t[q]; bq = q; }
      float wv = bv;
      for (int o = 16; o; o >>= 1) wv = fmaxf(wv, __shfl_xor_sync(0xffffffffu, wv, o));
      // remove one instance of the maximum (lowest lane holding it)
      const unsigned own = __ballot_sync(0xffffffffu, bq >= 0 && bv == wv);
      if (own && lane == __ffs(own) - 1) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q == bq) t[q] = -INFINITY;
      }
      tau = wv;
    }
    if (lane == 0) { s_tau = tau; s_lse = M + __logf(ss); }
  }
  __syncthreads();
  const float tau = s_tau;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float f = x[v];
    if (f >= tau) {
      const int at = atomicAdd(&s_n, 1);
      if (at < kCandCap) { s_cv[at] = f; s_ci[at] = v; }
    }
  }
  __syncthreads();
  const int n = s_n;
  const float lse = s_lse;
  if (n <= kCandCap) {
    if (warp == 0) {   // KB rounds of warp argmax (value desc, id asc) over the candidates
      for (int k = 0; k < KB; ++k) {
        float bv = -INFINITY;
        int bi = 0x7fffffff, bj = -1;
        for (int j = lane; j < n; j += 32)
          if (cand_better(s_cv[j], s_ci[j], bv, bi)) { bv = s_cv[j]; bi = s_ci[j]; bj = j; }
        float wv = bv;
        int wi = bi;
        for (int o = 16; o; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
          if (cand_better(ov, oi, wv, wi)) { wv = ov; wi = oi; }
        }
        if (bj >= 0 && bi == wi && bv == wv) s_cv[bj] = -INFINITY, s_ci[bj] = 0x7fffffff;
        __syncwarp();
        if (lane == 0) {
          cand_v[(size_t)row * KB + k] = wv - lse;        // log_softmax value
          cand_i[(size_t)row * KB + k] = wi;
        }
      }
    }
    return;
  }
  // fallback (more than kCandCap elements >= tau): KB rounds of block argmax over the row
  __shared__ float s_wv[8];
  __shared__ int s_wi[8];
  float last_v = INFINITY;
  int last_i = -1;
  for (int k = 0; k < KB; ++k) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      const float f = x[v];
      // strictly after (last_v, last_i) in (value desc, id asc) order
      const bool after = f < last_v || (f == last_v && v > last_i);
      if (after && cand_better(f, v, bv, bi)) { bv = f; bi = v; }
    }
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (cand_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { s_wv[warp] = bv; s_wi[warp] = bi; }
    __syncthreads();
    float wv = s_wv[0];
    int wi = s_wi[0];
    for (int w = 1; w < 8; ++w)
      if (cand_better(s_wv[w], s_wi[w], wv, wi)) { wv = s_wv[w]; wi = s_wi[w]; }
    __syncthreads();
    if (threadIdx.x == 0) {
      cand_v[(size_t)row * KB + k] = wv - lse;
      cand_i[(size_t)row * KB + k] = wi;
    }
    last_v = wv;
    last_i = wi;
  }
}

// ------------------------------------------------------------------ beam epilogue merge
// One warp per live row over the nseg partial records of the vocab GEMM's beam epilogue
// (tc_dev.cuh BeamAcc): LSE from the segment (max, sum) pairs, then KB rounds of warp
// argmax over the segments' sorted top-8 lists (each lane owns every 32nd segment).
__global__ void __launch_bounds__(128) k_beam_merge(const float* __restrict__ part, int nseg, int KB,
                                                    const int* __restrict__ dR,
                                                    float* __restrict__ cand_v,
                                                    int* __restrict__ cand_i) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= *dR) return;
  const float* pr = part + (size_t)row * nseg * (2 + 2 * kKB);
  float mm = -INFINITY;
  for (int g = lane; g < nseg; g += 32) mm = fmaxf(mm, pr[(size_t)g * (2 + 2 * kKB)]);
  float M = mm;
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float ss = 0.f;
  for (int g = lane; g < nseg; g += 32) {
    const float* r = pr + (size_t)g * (2 + 2 * kKB);
    if (r[0] > -INFINITY) ss += r[1] * __expf(r[0] - M);
  }
  ss = warp_sum(ss);
  const float lse = M + __logf(ss);
  constexpr int kMaxSeg = 16;   // segments per lane (nseg <= 512: V <= 65536)
  int ptr[kMaxSeg];
#pragma unroll
  for (int q = 0; q < kMaxSeg; ++q) ptr[q] = 0;
  for (int k = 0; k < KB; ++k) {
    float bv = -INFINITY;
    int bi = 0x7fffffff, bq = -1;
#pragma unroll
    for (int q = 0; q < kMaxSeg; ++q) {
      const int g = lane + 32 * q;
      if (g < nseg && ptr[q] < kKB) {
        const float* r = pr + (size_t)g * (2 + 2 * kKB);
        const float v = r[2 + ptr[q]];
        const int id = __float_as_int(r[2 + kKB + ptr[q]]);
        if (cand_better(v, id, bv, bi)) { bv = v; bi = id; bq = q; }
      }
    }
    float wv = bv;
    int wi = bi;
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
      if (cand_better(ov, oi, wv, wi)) { wv = ov; wi = oi; }
    }
    if (bq >= 0 && bi == wi && bv == wv) ptr[bq]++;
    if (lane == 0) {
      cand_v[(size_t)row * KB + k] = wv - lse;
      cand_i[(size_t)row * KB + k] = wi;
    }
  }
}

void beam_merge(const float* part, int nseg, int KB, const int* dR, int rows_upper, float* cand_v,
                int* cand_i, cudaStream_t s) {
  if (rows_upper <= 0) return;
  if (KB > kKB || nseg > 32 * 16) throw CudaError("beam_merge: 2K > 8 or V > 65536");
  k_beam_merge<<<ceil_div(rows_upper, 4), 128, 0, s>>>(part, nseg, KB, dR, cand_v, cand_i);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ teacher ensemble
// "a simple ensemble strategy", reading R26: per row the members' next-token
// distributions are averaged, ens[v] = logsumexp_m(x_m[v] - LSE_m) - log M (FP32).  One
// block per live row; pass 1: each member's LSE (online max / sum, block reduce); pass 2:
// the ensemble log-probabilities.  The per-row top-2K then runs on `ens` as for one model.
struct EnsLogits { const float* x[8]; };

__device__ __forceinline__ float block_lse(float m, float s) {
  __shared__ float bm[8], bs[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float mm = m;
  for (int o = 16; o; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  float ss = (m == -INFINITY) ? 0.f : s * __expf(m - mm);
  ss = warp_sum(ss);
  __syncthreads();
  if (lane == 0) { bm[warp] = mm; bs[warp] = ss; }
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) M = fmaxf(M, bm[w]);
  float S = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
    if (bm[w] > -INFINITY) S += bs[w] * __expf(bm[w] - M);
  return M + __logf(S);
}

__global__ void __launch_bounds__(256) k_ens_combine(EnsLogits L, int nm, int V,
                                                     const int* __restrict__ dR,
                                                     float* __restrict__ ens) {
  const int row = blockIdx.x;
  if (row >= *dR) return;
  float lse[8];
  for (int k = 0; k < nm; ++k) {
    const float* x = L.x[k] + (size_t)row * V;
    float m = -INFINITY, s = 0.f;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      const float f = x[v];
      if (f > m) { s = s * __expf(m - f) + 1.f; m = f; }
      else s += __expf(f - m);
    }
    lse[k] = block_lse(m, s);
  }
  const float logm = __logf((float)nm);
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    float a[8], mx = -INFINITY;
    for (int k = 0; k < nm; ++k) {
      a[k] = L.x[k][(size_t)row * V + v] - lse[k];
      mx = fmaxf(mx, a[k]);
    }
    float sum = 0.f;
    for (int k = 0; k < nm; ++k) sum += __expf(a[k] - mx);
    ens[(size_t)row * V + v] = mx + __logf(sum) - logm;
  }
}

void ens_combine(const float* const* logits, int nm, int V, const int* dR, int rows_upper,
                 float* ens, cudaStream_t s) {
  if (rows_upper <= 0) return;
  if (nm < 1 || nm > 8) throw CudaError("ens_combine: 1..8 members");
  EnsLogits L{};
  for (int k = 0; k < nm; ++k) L.x[k] = logits[k];
  k_ens_combine<<<rows_upper, 256, 0, s>>>(L, nm, V, dR, ens);
  NMT_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ per-sentence select
// One warp per live sentence group.  Shared staging per warp: the K parents' ancestry and
// token histories (t+1 ints each), so the in-place rewrite of the group's slots is safe.
struct SelCand { float v; int k; int tok; };

template <int K>
__global__ void __launch_bounds__(128) k_beam_select(
    const float* __restrict__ cand_v, const int* __restrict__ cand_i, float* __restrict__ score,
    int* __restrict__ prev_tok, uint8_t* __restrict__ done, const int* __restrict__ row_slot,
    const int* __restrict__ cap, int* __restrict__ anc, int* __restrict__ htok, int Tmax,
    float* __restrict__ best_score, int* __restrict__ out_tok, int* __restrict__ gen_len,
    DevState* st, int V, int eos, int NB, float* __restrict__ nb_score,
    int* __restrict__ nb_len, int* __restrict__ nb_tok, int* __restrict__ nb_cnt,
    int* __restrict__ parent_out) {
  extern __shared__ int sm_i[];
  constexpr int KB = 2 * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int grp = blockIdx.x * nw + warp;
  const int n_live = st->n_live;
  if (grp * K >= n_live) return;
  const int r0 = grp * K;
  if (done[r0]) {  // finished sentence waiting to be pruned
    if (parent_out && lane < K) parent_out[r0 + lane] = -1;
    return;
  }
  const int t = st->t;
  const int sent = row_slot[r0] / K;
  int* s_anc = sm_i + warp * 2 * K * (Tmax + 1);
  int* s_tok = s_anc + K * (Tmax + 1);
  __shared__ SelCand s_sel[4][2 * K];
  __shared__ int s_cnt[4];
  // candidate per lane: row k = lane / KB, rank q = lane % KB
  float cv = -INFINITY;
  int ck = 0x7fffffff, ctok = 0, ckey = 0x7fffffff;
  if (lane < K * KB) {
    const int k = lane / KB, q = lane % KB;
    const float sc = score[r0 + k];
    if (sc > -INFINITY) {
      cv = sc + cand_v[(size_t)(r0 + k) * KB + q];
      ctok = cand_i[(size_t)(r0 + k) * KB + q];
      ck = k;
      ckey = k * V + ctok;
    }
  }
  // 2K rounds of warp argmax by (score desc, slot*V + v asc)
  for (int rank = 0; rank < 2 * K; ++rank) {
    float wv = cv; int wk = ckey;
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
      const int okey = __shfl_xor_sync(0xffffffffu, wk, o);
      if (cand_better(ov, okey, wv, wk)) { wv = ov; wk = okey; }
    }
    if (ckey == wk && cv == wv && wv > -INFINITY) {
      s_sel[warp][rank] = {cv, ck, ctok};
      cv = -INFINITY; ckey = 0x7fffffff;
    } else if (lane == 0 && !(wv > -INFINITY)) {
      s_sel[warp][rank] = {-INFINITY, -1, 0};
    }
    __syncwarp();
  }
  // sequential bookkeeping by lane 0 (K tiny).  The finished list keeps the NB best
  // (score desc, ties -> earlier finalised; NB = 1: the best only, reading R27).
  __shared__ int s_done[4], s_nops[4], s_op_pos[4][3 * K], s_op_k[4][3 * K], s_op_tok[4][3 * K];
  __shared__ SelCand s_new[4][K];
  if (lane == 0) {
    float lst[4];
    int cnt = NB == 1 ? (best_score[sent] > -INFINITY ? 1 : 0) : nb_cnt[sent];
    if (NB == 1) lst[0] = best_score[sent];
    else
      for (int i = 0; i < cnt; ++i) lst[i] = nb_score[(size_t)sent * NB + i];
    int nops = 0;
    auto try_insert = [&](const SelCand& c) {
      if (cnt == NB && !(c.v > lst[NB - 1])) return;
      int pos = 0;
      while (pos < cnt && lst[pos] >= c.v) ++pos;
      for (int i = min(cnt, NB - 1); i > pos; --i) lst[i] = lst[i - 1];
      lst[pos] = c.v;
      cnt = min(cnt + 1, NB);
      s_op_pos[warp][nops] = pos;
      s_op_k[warp][nops] = c.k;
      s_op_tok[warp][nops] = c.tok;
      ++nops;
    };
    int n_new = 0;
    for (int rank = 0; rank < 2 * K; ++rank) {
      const SelCand c = s_sel[warp][rank];
      if (!(c.v > -INFINITY)) break;
      if (c.tok == eos) {
        if (rank < K) try_insert(c);
      } else if (n_new < K) {
        s_new[warp][n_new++] = c;
      }
    }
    const bool at_cap = t + 1 >= cap[sent];
    if (at_cap)
      for (int i = 0; i < n_new; ++i) try_insert(s_new[warp][i]);
    float best_act = -INFINITY;
    for (int i = 0; i < n_new; ++i) best_act = fmaxf(best_act, s_new[warp][i].v);
    const bool early = cnt >= NB && lst[NB - 1] >= best_act;
    s_done[warp] = at_cap || n_new == 0 || early;
    s_cnt[warp] = n_new;
    s_nops[warp] = nops;
    if (NB == 1) {
      if (cnt) best_score[sent] = lst[0];
    } else {
      for (int i = 0; i < cnt; ++i) nb_score[(size_t)sent * NB + i] = lst[i];
      nb_cnt[sent] = cnt;
      best_score[sent] = cnt ? lst[0] : -INFINITY;
    }
  }
  __syncwarp();
  const int n_new = s_cnt[warp], nops = s_nops[warp];
  const bool sdone = s_done[warp];
  // apply the insertions in order: shift the list rows below `pos`, then write the new
  // hypothesis = htok[parent][1..t] + token.  Position 0 is mirrored to out_tok.
  for (int o = 0; o < nops; ++o) {
    const int pos = s_op_pos[warp][o];
    const int ps = row_slot[r0 + s_op_k[warp][o]];
    if (NB > 1) {
      int* base = nb_tok + (size_t)sent * NB * Tmax;
      for (int i = NB - 1; i > pos; --i) {
        const int len = nb_len[(size_t)sent * NB + i - 1];
        for (int j = lane; j < len; j += 32) base[(size_t)i * Tmax + j] = base[(size_t)(i - 1) * Tmax + j];
        __syncwarp();
        if (lane == 0) nb_len[(size_t)sent * NB + i] = len;
      }
      for (int j = lane; j < t; j += 32) base[(size_t)pos * Tmax + j] = htok[(size_t)ps * Tmax + j + 1];
      if (lane == 0) {
        base[(size_t)pos * Tmax + t] = s_op_tok[warp][o];
        nb_len[(size_t)sent * NB + pos] = t + 1;
      }
    }
    if (pos == 0) {
      for (int j = lane; j < t; j += 32) out_tok[(size_t)sent * Tmax + j] = htok[(size_t)ps * Tmax + j + 1];
      if (lane == 0) {
        out_tok[(size_t)sent * Tmax + t] = s_op_tok[warp][o];
        gen_len[sent] = t + 1;
      }
    }
    __syncwarp();
  }
  if (sdone) {
    if (parent_out && lane < K) parent_out[r0 + lane] = -1;
    if (lane < K) done[r0 + lane] = 1;
    if (lane == 0) atomicAdd(&st->n_done, K);
    return;
  }
  // stage parents' ancestry / history, then rewrite this group's slots in place
  for (int i = 0; i < n_new; ++i) {
    const int ps = row_slot[r0 + s_new[warp][i].k];
    for (int j = lane; j <= t; j += 32) {
      s_anc[i * (Tmax + 1) + j] = j < t ? anc[(size_t)ps * Tmax + j] : ps;
      s_tok[i * (Tmax + 1) + j] = htok[(size_t)ps * Tmax + j];
    }
  }
  __syncwarp();
  for (int i = 0; i < K; ++i) {
    const int r = r0 + i, slot = row_slot[r];
    if (i < n_new) {
      for (int j = lane; j <= t; j += 32) {
        anc[(size_t)slot * Tmax + j] = s_anc[i * (Tmax + 1) + j];
        htok[(size_t)slot * Tmax + j] = s_tok[i * (Tmax + 1) + j];
      }
      if (lane == 0) {
        if (t + 1 < Tmax) htok[(size_t)slot * Tmax + t + 1] = s_new[warp][i].tok;
        prev_tok[r] = s_new[warp][i].tok;
        score[r] = s_new[warp][i].v;
        if (parent_out) parent_out[r] = r0 + s_new[warp][i].k;
      }
    } else if (lane == 0) {
      score[r] = -INFINITY;  // fewer than K continuations (tiny vocabularies)
      prev_tok[r] = eos;
      if (parent_out) parent_out[r] = -1;
    }
  }
}

void beam_row_topk(const float* logits, int V, int KB, const int* dR, int rows_upper,
                   float* cand_v, int* cand_i, cudaStream_t s) {
  if (rows_upper <= 0) return;
  if (KB > kKB) throw CudaError("beam_row_topk: 2K > 8");
  k_beam_row_topk<<<rows_upper, 256, 0, s>>>(logits, V, KB, dR, cand_v, cand_i);
  NMT_LAUNCH_CHECK();
}

void beam_select(int K, const float* cand_v, const int* cand_i, float* score, int* prev_tok,
                 uint8_t* done, const int* row_slot, const int* cap, int* anc, int* htok,
                 int Tmax, float* best_score, int* out_tok, int* gen_len, DevState* st, int V,
                 int eos, int rows_upper, cudaStream_t s, int NB, float* nb_score, int* nb_len,
                 int* nb_tok, int* nb_cnt, int* parent_out) {
  if (rows_upper <= 0) return;
  if (NB < 1 || NB > K) throw CudaError("beam_select: nbest must be in [1, beam]");
  const int groups = (rows_upper + K - 1) / K, nw = 4;
  const size_t smem = (size_t)nw * 2 * K * (Tmax + 1) * sizeof(int);
#define NMT_BS(KK)                                                                            \
  k_beam_select<KK><<<ceil_div(groups, nw), nw * 32, smem, s>>>(                              \
      cand_v, cand_i, score, prev_tok, done, row_slot, cap, anc, htok, Tmax, best_score,       \
      out_tok, gen_len, st, V, eos, NB, nb_score, nb_len, nb_tok, nb_cnt, parent_out)
  switch (K) {
    case 1: NMT_BS(1); break;
    case 2: NMT_BS(2); break;
    case 3: NMT_BS(3); break;
    case 4: NMT_BS(4); break;
    default: throw CudaError("beam_select: beam must be 1..4");
  }
#undef NMT_BS
  NMT_LAUNCH_CHECK();
}

__global__ void k_beam_init(int* row_slot, int* prev_tok, uint8_t* done, float* score, int* htok,
                            int Tmax, float* best_score, int* gen_len, DevState* st, int B, int K,
                            int S, int bos, int* nb_cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < B * K) {
    row_slot[r] = r;
    prev_tok[r] = bos;
    done[r] = 0;
    score[r] = (r % K == 0) ? 0.f : -INFINITY;  // t = 0: only the BOS hypothesis is active
    htok[(size_t)r * Tmax] = bos;
  }
  if (r < B) {
    best_score[r] = -INFINITY;
    gen_len[r] = 0;
    if (nb_cnt) nb_cnt[r] = 0;
  }
  if (r == 0) {
    st->t = 0;
    st->n_live = B * K;
    st->n_done = 0;
    st->prunes = 0;
    st->S = S;
  }
}

void beam_init(int* row_slot, int* prev_tok, uint8_t* done, float* score, int* htok, int Tmax,
               float* best_score, int* gen_len, DevState* st, int B, int K, int S, int bos,
               cudaStream_t s, int* nb_cnt) {
  const int n = B * K;
  k_beam_init<<<ceil_div(n > 0 ? n : 1, 128), 128, 0, s>>>(row_slot, prev_tok, done, score, htok,
                                                           Tmax, best_score, gen_len, st, B, K, S,
                                                           bos, nb_cnt);
  NMT_LAUNCH_CHECK();
}

}  // namespace nmt
