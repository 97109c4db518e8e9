// common.cuh — shared device helpers for the sm_100a kernels (no method arithmetic
// beyond FP16<->FP32 conversion and warp reductions).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace nmt {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define NMT_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::nmt::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + \
                             __FILE__ + ":" + std::to_string(__LINE__));                \
  } while (0)

// Every kernel launch of the library goes through NMT_LAUNCH_CHECK, which also counts
// it (nmt_stats.launches / bench "gpu_launches").
extern std::atomic<unsigned long long> g_launches;
#define NMT_LAUNCH_CHECK()    \
  do {                        \
    ++::nmt::g_launches;      \
    NMT_CUDA(cudaGetLastError()); \
  } while (0)

// ---- element conversion --------------------------------------------------------------
template <class T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }

// FP32 -> storage type.  FP16: round-to-nearest-even, saturating at +-65504 (reading R19).
template <class T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __half from_f<__half>(float v) {
  v = fminf(fmaxf(v, -65504.f), 65504.f);
  return __float2half_rn(v);
}
// (lo, hi) -> saturating round-to-nearest half2 in one instruction (same values as from_f)
__device__ __forceinline__ uint32_t pack_half2_sat(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Ordered-float key: larger float -> larger unsigned key (finite inputs).
__device__ __forceinline__ uint32_t ordered_key(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
// Packed (value, id) key for argmax with ties -> lowest id: max over keys.
__device__ __forceinline__ unsigned long long pack_argmax(float v, int id) {
  return ((unsigned long long)ordered_key(v) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)id);
}
__device__ __forceinline__ int unpack_argmax_id(unsigned long long k) {
  return (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ---- bounded-wait timeout -------------------------------------------------------------
// A pipeline or scheduling bug traps (a clean launch failure) instead of hanging the GPU.
// Built with -DNMT_TRAP_DIAG (NMT_EXTRA_NVCC), the trapping thread first prints where it
// was waiting (the printf buffer is flushed when the launch failure is reported).
#ifdef NMT_TRAP_DIAG
#define NMT_TRAP(tag, a, b)                                                                  \
  do {                                                                                       \
    unsigned smid_;                                                                          \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                       \
    printf("NMT_TRAP %s:%d %s block (%d,%d) of (%d,%d) thread %d of %d sm %u a=%u b=%u\n",  \
           __FILE__, __LINE__, tag, (int)blockIdx.x, (int)blockIdx.y, (int)gridDim.x,        \
           (int)gridDim.y, (int)threadIdx.x, (int)blockDim.x, smid_, (unsigned)(a),          \
           (unsigned)(b));                                                                   \
    __trap();                                                                                \
  } while (0)
#else
#define NMT_TRAP(tag, a, b) __trap()
#endif

// ---- programmatic dependent launch (PDL) -----------------------------------------------
// Decode-step kernels are launched with programmatic stream serialisation while a step is
// captured into a CUDA graph: the next kernel's CTAs are scheduled while the previous
// kernel drains, and block in pdl_wait() until it has completed (memory visible).
extern thread_local bool g_pdl;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  NMT_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

}  // namespace nmt
