// gemm_simt.cu — CUDA-core GEMM, C = A . B^T with fused epilogues.
// Used for the FP32 parity mode (true FP32: TF32 cannot meet 1e-4) and as
// the reference the tcgen05 kernel is unit-tested against.  64x64 tile, BK = 16,
// 256 threads x (4x4) outputs, FP32 accumulation.
#include "common.cuh"
#include "kernels.h"

namespace nmt {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;

template <class T>
__global__ void __launch_bounds__(256) k_gemm_simt(GemmArgs a) {
  __shared__ float As[BK][BM + PAD];
  __shared__ float Bs[BK][BN + PAD];
  const int M = a.dM ? min(a.M, *a.dM) : a.M;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  const T* A = static_cast<const T*>(a.A);
  const T* B = static_cast<const T*>(a.B);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += BK) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int idx = threadIdx.x + 256 * e;
      int r = idx >> 4, k = idx & 15;
      int gm = m0 + r, gn = n0 + r, gk = k0 + k;
      As[k][r] = (gm < M && gk < a.K) ? to_f(A[(size_t)gm * a.lda + gk]) : 0.f;
      Bs[k][r] = (gn < a.N && gk < a.K) ? to_f(B[(size_t)gn * a.ldb + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float4 av = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      float4 bv = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }
  const T* bias = static_cast<const T*>(a.bias);
  const T* R = static_cast<const T*>(a.R);
  T* C = static_cast<T*>(a.C);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    unsigned long long best = 0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= a.N) continue;
      float v = acc[i][j];
      if (bias) v += to_f(bias[n]);
      if (R) v += to_f(R[(size_t)m * a.ldr + n]);
      if (a.relu) v = fmaxf(v, 0.f);
      if (a.logits) a.logits[(size_t)m * a.N + n] = v;
      if (a.argmax) {
        unsigned long long k = pack_argmax(v, n);
        best = k > best ? k : best;
      } else {
        if (C) C[(size_t)m * a.ldc + n] = from_f<T>(v);  // C == null: logits only (beam)
      }
    }
    if (a.argmax && best) atomicMax(a.argmax + m, best);
  }
}
}  // namespace

template <class T> void gemm_simt(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.st_out || a.ln_st) throw CudaError("gemm_simt: LN folding is an FP16 tcgen05 feature");
  dim3 grid(ceil_div(a.N, BN), ceil_div(a.M, BM));
  k_gemm_simt<T><<<grid, 256, 0, s>>>(a);
  NMT_LAUNCH_CHECK();
}

template void gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void gemm_simt<__half>(const GemmArgs&, cudaStream_t);

template <> void gemm<float>(const GemmArgs& a, cudaStream_t s) { gemm_simt<float>(a, s); }
template <> void gemm<__half>(const GemmArgs& a, cudaStream_t s) { gemm_tc(a, s); }

}  // namespace nmt
