// decode_fused.h — parameters of the fused FP16 decode-step kernel (decode_fused.cu).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace nmt {

constexpr int kMaxFusedLayers = 6;
namespace dfz {
constexpr int kMaxPhases = 2 + 8 * kMaxFusedLayers;
}

// One projection of a decoder layer: C[m][n] = epilogue(A[m] . B[n]), A and B through the
// tensor maps ma / mb of FusedLayer.  Shape policy = gemm_tc.cu decode_config (weight shape
// only): bn 64 / 128 output columns per tile, split = 1 keeps the two K halves in separate
// accumulators summed in the epilogue (the unfused cluster split-K association).
struct GemmPhase {
  int N, K, bn, nt, split, relu, ldc;
  const __half* bias;      // [N] or null
  const __half* R;         // residual [rows][d] (the stream g) or null
  __half* C;
  float2* st_out;          // LN-folding producer: per-row (mean, M2) of 32-column chunks
  const float2* ln_st;     // LN-folding consumer: statistics of A's rows, and c[n]
  const float* ln_c;
};

struct FusedLayer {
  CUtensorMap ma[6], mb[6];   // QKV, self-out, cross-q, cross-out, FFN1, FFN2
  CUtensorMap ma32[6];        // A with 32-row boxes: a row block with <= 32 live rows
  GemmPhase g[6];
  const __half *relk, *relv;
  __half *kc, *vc;            // this layer's self-attention cache [slot][Tmax][d]
  int koff, voff;             // cross K / V column offsets in the cross cache
};

struct FusedParams {
  FusedLayer L[kMaxFusedLayers];
  int Ld, Tmax, kclip, use_rpr, beam, ldkv;
  int pbeg, pend;             // phase range of this launch: 0 = embed, 1 + 8l + {0..7}, 1 + 8Ld = LN
  float eps, scale;
  const int* ids;             // tokens w_t per live row (prev_tok or teacher forcing)
  const __half *emb, *ln0_g, *ln0_b, *lnf_g, *lnf_b;
  const float* pe;
  __half *g, *u, *qkv, *attn_out, *q;
  const int *row_slot, *anc, *src_len;
  const __half* ckv;
  DevState* st;
  int* ctr;                   // [0] next item, [1] CTAs done, [2..] (phase, row block) counters
  unsigned long long* trace;  // optional timeline (nmt_debug_fused_trace): per item 4 x u64
};

size_t fused_counter_ints();
bool fused_supported(int d, int H, int F, int Ld);
void decode_fused(const FusedParams& p, int E, cudaStream_t s);

}  // namespace nmt
