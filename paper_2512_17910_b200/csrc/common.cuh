// Shared helpers for the sm_100a kernels of libalora_sm100a.so.
#pragma once

#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#include "../../include/alora_sm100a.h"

#define ALORA_CUDA_CHECK(expr)                  \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return ALORA_ECUDA;  \
  } while (0)

#define ALORA_LAUNCH_CHECK()                          \
  do {                                                \
    cudaError_t _e = cudaGetLastError();              \
    if (_e != cudaSuccess) return ALORA_ECUDA;        \
  } while (0)

namespace alora {

// Every kernel asks for the max-shared-memory carveout so the SMs never switch the
// L1/smem split between the 200 KB tcgen05 GEMM and the small kernels around it
// (a carveout change drains the SM and costs microseconds per launch).
template <typename Kernel>
inline void prefer_max_smem(Kernel kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       static_cast<int>(cudaSharedmemCarveoutMaxShared));
}

constexpr int kNumSMs = 148;

// ---- programmatic dependent launch (PDL)
// Forward-path kernels are launched with programmatic stream serialization: kernel i+1 is scheduled while
// kernel i drains, runs its prologue (barrier init, TMEM alloc, tensor-map prefetch, weight TMA) and
// blocks in pdl_wait() until kernel i has completed and its writes are visible. Launched without the
// attribute, both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_on() {
  static const bool on = [] {
    const char* e = getenv("ALORA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Launch log (profiling only): while the executor profiles, every kernel launched through launch_pdl is
// recorded with its grid, so tests and the bench can tell which kernel variant served each step.
struct LaunchNote {
  const void* fn;
  unsigned grid;
};
inline thread_local std::vector<LaunchNote>* g_launch_log = nullptr;
inline void note_launch(const void* fn, dim3 grid) {
  if (g_launch_log) g_launch_log->push_back({fn, grid.x * grid.y * grid.z});
}

// cudaLaunchKernelEx with the PDL attribute (plus optional extra attributes).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              const cudaLaunchAttribute* extra, int n_extra, Args&&... args) {
  note_launch(reinterpret_cast<const void*>(kernel), grid);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[4];
  int n = 0;
  for (int i = 0; i < n_extra && n < 3; ++i) attr[n++] = extra[i];
  if (pdl_on()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
constexpr int kGluBlock = 64;  // gate|up interleave granularity of w_in_t (llama)

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions in a fixed order (deterministic): warp tree, then warp 0.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem /* >= 32 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = (lane < nw) ? smem[lane] : T(0);
  if (wid == 0) r = warp_sum(r);
  if (threadIdx.x == 0) smem[0] = r;
  __syncthreads();
  return smem[0];
}

template <typename T>
__device__ __forceinline__ T block_max(T v, T* smem, T lowest) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = (lane < nw) ? smem[lane] : lowest;
  if (wid == 0) r = warp_max(r);
  if (threadIdx.x == 0) smem[0] = r;
  __syncthreads();
  return smem[0];
}

// Sequence owning packed row m: cu_q is ascending with cu_q[0] = 0.
__device__ __forceinline__ int seq_of_row(const int32_t* cu_q, int n_seqs, int m) {
  int lo = 0, hi = n_seqs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cu_q[mid] <= m) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace alora
