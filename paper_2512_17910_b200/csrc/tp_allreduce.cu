// Tensor-parallel all-reduce fused with the residual add and the RMSNorm that follows it, over peer memory.
//
// The row-parallel O-projection and MLP-down of a TP rank (reference model.py:269-271 is
// the unsharded x += o / x += mlp) produce fp32 partial residual updates that must be summed over ranks
// before `x += delta; h = rmsnorm(x) * w`. Instead of an NCCL all-reduce followed by a separate norm kernel,
// every rank's GEMM writes its partial into its own slot of a symmetric buffer that all ranks have mapped
// (CUDA IPC over NVLink / NVSwitch, or plain device pointers when the ranks share one GPU), and ONE kernel
// per rank does the exchange and the norm:
//
//   one-shot (small M: decode, short suffix steps)  every rank reads all ranks' partial rows, sums them in
//                                                   rank order, adds the residual and normalises all rows;
//   two-shot (larger M)                             rank r reduces rows [r*M/N, (r+1)*M/N) (sum in rank
//                                                   order + residual + norm) into its reduced-x / reduced-h
//                                                   area; after a second barrier every rank gathers the
//                                                   other ranks' reduced rows (N-1)/N of x and h.
//
// Both sum the partials in rank order, so every rank ends with bitwise-identical x and h (the replicated
// residual stream stays replicated). Synchronisation is per CTA: block b of every rank signals block b of
// every peer (st.release.sys into the peer's flag slot [b][rank]) and waits for the peers' signals in its own
// slots (ld.acquire.sys); the value is a per-block epoch counter kept on the device (the same sequence of
// calls on every rank), so the kernel is CUDA-graph capturable. Partials alternate between two slots by call
// parity: a rank rewrites a slot only after the barrier of the next call, which every peer enters after it
// finished reading that slot. The two-shot reduced rows alternate the same way.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace alora {

namespace {

constexpr int kTpMaxRanks = 8;
constexpr int kTpMaxBlocks = 2 * kNumSMs;
constexpr int kTpThreads = 256;

inline int64_t tp_align(int64_t x) { return (x + 255) / 256 * 256; }

struct TpArgs {
  char* peer[kTpMaxRanks];  // base of each rank's symmetric buffer
  int rank, n, M, d;
  int one_shot;
  int64_t part_off;  // this call's partial slot
  int64_t redx_off, redh_off, flags_off, epoch_off;
  float* x;                // [M, d] this rank's residual stream (updated in place)
  const float* w;          // norm gain (nullptr: no gain)
  float eps;
  __nv_bfloat16* h;        // [M, d] normalised output; nullptr = residual update only
  int timeout_trap;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Block b of this rank meets block b of every peer: flag slot [b][src rank] of the destination rank.
__device__ __forceinline__ void peer_barrier(const TpArgs& a, int b, uint32_t v) {
  __syncthreads();  // the block's writes happen-before thread t's release
  if (threadIdx.x < a.n) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(a.peer[threadIdx.x] + a.flags_off) + b * kTpMaxRanks + a.rank;
    st_release_sys(dst, v);
    const uint32_t* mine =
        reinterpret_cast<const uint32_t*>(a.peer[a.rank] + a.flags_off) + b * kTpMaxRanks + threadIdx.x;
    unsigned spins = 0;
    while ((int)(ld_acquire_sys(mine) - v) < 0) {
      __nanosleep(64);
      if (a.timeout_trap && ++spins > (1u << 26)) {  // a peer never arrived: fail loudly, do not hang
        printf("alora tp all-reduce: rank %d block %d waited too long for rank %d (flag %u < %u)\n", a.rank, b,
               (int)threadIdx.x, ld_acquire_sys(mine), v);
        __trap();
      }
    }
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(kTpThreads) tp_ar_norm_kernel(const TpArgs a, int trigger) {
  pdl_wait();  // the GEMM that wrote this rank's partial has completed
  if (trigger) pdl_trigger();
  __shared__ float red[32];
  __shared__ uint32_t e_sh;
  const int b = blockIdx.x, tid = threadIdx.x;
  uint32_t* epoch = reinterpret_cast<uint32_t*>(a.peer[a.rank] + a.epoch_off) + b;
  if (tid == 0) e_sh = *epoch;
  __syncthreads();
  const uint32_t e = e_sh;
  peer_barrier(a, b, e + 1);
  const int n4 = a.d >> 2;
  const int per = a.one_shot ? a.M : (a.M + a.n - 1) / a.n;
  const int r0 = a.one_shot ? 0 : min(a.M, a.rank * per), r1 = min(a.M, r0 + per);
  float4* redx = reinterpret_cast<float4*>(a.peer[a.rank] + a.redx_off);
  uint2* redh = reinterpret_cast<uint2*>(a.peer[a.rank] + a.redh_off);
  for (int row = r0 + b; row < r1; row += gridDim.x) {
    float4 v[V];
    float ss = 0.f;
    float4* xr = reinterpret_cast<float4*>(a.x + (int64_t)row * a.d);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int i = tid + j * kTpThreads;
      if (i >= n4) { v[j] = make_float4(0.f, 0.f, 0.f, 0.f); continue; }
      float4 q[kTpMaxRanks];
#pragma unroll
      for (int p = 0; p < kTpMaxRanks; ++p)  // every peer's load in flight before the adds
        if (p < a.n)
          q[p] = __ldcg(reinterpret_cast<const float4*>(a.peer[p] + a.part_off) + (int64_t)row * n4 + i);
      float4 s = q[0];
#pragma unroll
      for (int p = 1; p < kTpMaxRanks; ++p)
        if (p < a.n) { s.x += q[p].x; s.y += q[p].y; s.z += q[p].z; s.w += q[p].w; }
      float4 x = xr[i];
      x.x += s.x; x.y += s.y; x.z += s.z; x.w += s.w;
      v[j] = x;
      xr[i] = x;
      if (!a.one_shot) __stcg(redx + (int64_t)row * n4 + i, x);
      ss = fmaf(x.x, x.x, ss); ss = fmaf(x.y, x.y, ss); ss = fmaf(x.z, x.z, ss); ss = fmaf(x.w, x.w, ss);
    }
    if (a.h == nullptr) continue;
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)a.d + a.eps);
    uint2* hr = reinterpret_cast<uint2*>(a.h + (int64_t)row * a.d);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int i = tid + j * kTpThreads;
      if (i >= n4) break;
      float4 y = make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
      if (a.w) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(a.w) + i);
        y.x *= g.x; y.y *= g.y; y.z *= g.z; y.w *= g.w;
      }
      __nv_bfloat162 lo = __floats2bfloat162_rn(y.x, y.y), hi = __floats2bfloat162_rn(y.z, y.w);
      const uint2 o = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      hr[i] = o;
      if (!a.one_shot) __stcg(redh + (int64_t)row * n4 + i, o);
    }
  }
  if (!a.one_shot) {
    peer_barrier(a, b, e + 2);  // every rank's reduced rows of this block index are published
    for (int p = 0; p < a.n; ++p) {
      if (p == a.rank) continue;
      const int q0 = min(a.M, p * per), q1 = min(a.M, q0 + per);
      const float4* px = reinterpret_cast<const float4*>(a.peer[p] + a.redx_off);
      const uint2* ph = reinterpret_cast<const uint2*>(a.peer[p] + a.redh_off);
      for (int row = q0 + b; row < q1; row += gridDim.x) {
        float4* xr = reinterpret_cast<float4*>(a.x + (int64_t)row * a.d);
        for (int i = tid; i < n4; i += kTpThreads) xr[i] = __ldcg(px + (int64_t)row * n4 + i);
        if (a.h) {
          uint2* hr = reinterpret_cast<uint2*>(a.h + (int64_t)row * a.d);
          for (int i = tid; i < n4; i += kTpThreads) hr[i] = __ldcg(ph + (int64_t)row * n4 + i);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) *epoch = e + 2;
}

struct TpLayout {
  int64_t part[2], redx[2], redh[2], flags, epoch, total;
};

TpLayout tp_layout(int64_t T, int64_t d) {
  TpLayout L{};
  int64_t off = 0;
  auto take = [&](int64_t bytes) { const int64_t o = off; off = tp_align(off + bytes); return o; };
  L.flags = take((int64_t)kTpMaxBlocks * kTpMaxRanks * 4);
  L.epoch = take((int64_t)kTpMaxBlocks * 4);
  L.part[0] = take(T * d * 4);
  L.part[1] = take(T * d * 4);
  L.redx[0] = take(T * d * 4);
  L.redh[0] = take(T * d * 2);
  L.redx[1] = take(T * d * 4);
  L.redh[1] = take(T * d * 2);
  L.total = off;
  return L;
}

}  // namespace

int64_t tp_buffer_bytes(int max_tokens, int d) { return tp_layout(max_tokens, d).total; }

float* tp_partial_slot(void* own, int max_tokens, int d, int slot) {
  return reinterpret_cast<float*>(static_cast<char*>(own) + tp_layout(max_tokens, d).part[slot & 1]);
}

int tp_allreduce_norm(void* const* peers, int n, int rank, int colocated, int max_tokens, int slot, int M, int d,
                      float* x, const float* w, float eps, __nv_bfloat16* h, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  if (n < 2 || n > kTpMaxRanks || rank < 0 || rank >= n || M > max_tokens || d % 4 || d > 4 * kTpThreads * 8)
    return ALORA_EINVAL;
  const TpLayout L = tp_layout(max_tokens, d);
  TpArgs a{};
  for (int p = 0; p < n; ++p) {
    if (!peers[p]) return ALORA_EINVAL;
    a.peer[p] = static_cast<char*>(peers[p]);
  }
  a.rank = rank; a.n = n; a.M = M; a.d = d;
  // one-shot while each rank's reads of all N partials stay small (latency-bound: one barrier); two-shot
  // above, where reading N full partials would cost N x the traffic of a reduce-scatter + all-gather
  a.one_shot = (int64_t)M * d * 4 * n <= (int64_t)4 << 20;
  a.part_off = L.part[slot & 1];
  // the reduced rows alternate by call parity too: block b of a rank rewrites them right after ITS barrier of
  // the next call, while a peer's block b' != b (the row -> block map changes with M) may still be gathering
  // this call's rows; two calls later every peer's kernel of this call has completed (stream order)
  a.redx_off = L.redx[slot & 1]; a.redh_off = L.redh[slot & 1]; a.flags_off = L.flags; a.epoch_off = L.epoch;
  a.x = x; a.w = w; a.eps = eps; a.h = h;
  a.timeout_trap = 1;
  const int rows = a.one_shot ? M : (M + n - 1) / n;
  // Ranks sharing one GPU (the single-device test harness): while some ranks spin here, the others' kernels
  // must still be able to launch -- including thread-block clusters (the segmented LoRA shrink: 8 CTAs of
  // ~200 KB in one GPC), which spinning CTAs spread over a GPC's SMs could block. So one CTA per rank, and
  // the next kernel is not released early (its CTAs could take the SMs a peer's kernel needs). The harness
  // also needs more hardware work queues than streams (tests/conftest.py: CUDA_DEVICE_MAX_CONNECTIONS),
  // or a rank's kernels can queue behind a peer's spinning kernel. One rank per GPU (the deployment) has no
  // such coupling: a full grid of CTAs.
  const int cap = colocated ? 1 : kTpMaxBlocks;
  const int grid = std::max(1, std::min(rows, cap));
  const int v = (d / 4 + kTpThreads - 1) / kTpThreads;
  const int trigger = colocated ? 0 : 1;
  cudaError_t err;
  if (v <= 1) err = launch_pdl(tp_ar_norm_kernel<1>, dim3(grid), dim3(kTpThreads), 0, st, nullptr, 0, a, trigger);
  else if (v <= 2) err = launch_pdl(tp_ar_norm_kernel<2>, dim3(grid), dim3(kTpThreads), 0, st, nullptr, 0, a, trigger);
  else if (v <= 4) err = launch_pdl(tp_ar_norm_kernel<4>, dim3(grid), dim3(kTpThreads), 0, st, nullptr, 0, a, trigger);
  else err = launch_pdl(tp_ar_norm_kernel<8>, dim3(grid), dim3(kTpThreads), 0, st, nullptr, 0, a, trigger);
  ALORA_CUDA_CHECK(err);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

void configure_tp() {
  prefer_max_smem(tp_ar_norm_kernel<1>);
  prefer_max_smem(tp_ar_norm_kernel<2>);
  prefer_max_smem(tp_ar_norm_kernel<4>);
  prefer_max_smem(tp_ar_norm_kernel<8>);
}

}  // namespace alora

extern "C" {

int64_t alora_tp_buffer_bytes(int32_t max_tokens, int32_t d_model) {
  if (max_tokens < 1 || d_model < 1) return ALORA_EINVAL;
  return alora::tp_buffer_bytes(max_tokens, d_model);
}

int64_t alora_tp_partial_offset(int32_t max_tokens, int32_t d_model, int32_t slot) {
  if (max_tokens < 1 || d_model < 1) return ALORA_EINVAL;
  return reinterpret_cast<int64_t>(alora::tp_partial_slot(nullptr, max_tokens, d_model, slot));
}

int alora_device_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 1) return ALORA_EINVAL;
  *out = nullptr;
  if (cudaMalloc(out, (size_t)bytes) != cudaSuccess) return ALORA_ECUDA;
  if (cudaMemset(*out, 0, (size_t)bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(*out);
    *out = nullptr;
    return ALORA_ECUDA;
  }
  return ALORA_OK;
}

int alora_device_free(void* p) { return cudaFree(p) == cudaSuccess ? ALORA_OK : ALORA_ECUDA; }

int alora_ipc_get_handle(void* dev_ptr, uint8_t* out64) {
  if (!dev_ptr || !out64) return ALORA_EINVAL;
  cudaIpcMemHandle_t hnd;
  if (cudaIpcGetMemHandle(&hnd, dev_ptr) != cudaSuccess) return ALORA_ECUDA;
  static_assert(sizeof(hnd) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out64, &hnd, 64);
  return ALORA_OK;
}

int alora_ipc_open(const uint8_t* handle64, void** out_ptr) {
  if (!handle64 || !out_ptr) return ALORA_EINVAL;
  cudaIpcMemHandle_t hnd;
  memcpy(&hnd, handle64, 64);
  *out_ptr = nullptr;
  return cudaIpcOpenMemHandle(out_ptr, hnd, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? ALORA_OK : ALORA_ECUDA;
}

int alora_ipc_close(void* ptr) { return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? ALORA_OK : ALORA_ECUDA; }

int alora_tp_allreduce_norm(void* const* peers, int32_t n_ranks, int32_t rank, int32_t colocated,
                            int32_t max_tokens, int32_t slot, int32_t M, int32_t d, float* x, const float* w,
                            float eps, void* h, void* stream) {
  if (!peers || !x) return ALORA_EINVAL;
  alora::configure_kernels();
  return alora::tp_allreduce_norm(peers, n_ranks, rank, colocated, max_tokens, slot, M, d, x, w, eps,
                                  static_cast<__nv_bfloat16*>(h), static_cast<cudaStream_t>(stream));
}

}  // extern "C"
