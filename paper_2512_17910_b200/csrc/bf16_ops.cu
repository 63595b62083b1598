// bf16-tier elementwise / row kernels around the tensor-core GEMM and attention:
// embedding gather, RMSNorm -> bf16 GEMM operand, RoPE, the segmented LoRA
// shrink and the per-tile adapter masks that let the GEMM skip absent adapters.

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace alora {

// ----------------------------------------------------------------- embed ---
// x (fp32 residual) = embed[tok] (+ sinusoidal pos for the ref arch, model.py:263)
// tokens[m] < 0 names the previous forward's greedy id of span -tokens[m]-1 (prev_ids: the next_ids buffer
// of the step, which still holds the previous launch's ids when this first kernel runs): decode steps can be
// launched before the host has read the previous step's output.
__global__ void embed_bf16_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                                  const __nv_bfloat16* __restrict__ embed, const float* __restrict__ pos_table, int d,
                                  float* __restrict__ x, const int32_t* __restrict__ prev_ids) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  int tok = tokens[m];
  if (tok < 0) tok = prev_ids[-tok - 1];
  const __nv_bfloat16* e = embed + (int64_t)tok * d;
  const float* p = pos_table ? pos_table + (int64_t)positions[m] * d : nullptr;
  float* xr = x + (int64_t)m * d;
  if (d % 8 == 0) {  // 16-byte embedding loads, two float4 stores
    for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(e + i);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
      float f[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
        f[2 * k] = t.x;
        f[2 * k + 1] = t.y;
      }
      if (p) {
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] += p[i + k];
      }
      *reinterpret_cast<float4*>(xr + i) = make_float4(f[0], f[1], f[2], f[3]);
      *reinterpret_cast<float4*>(xr + i + 4) = make_float4(f[4], f[5], f[6], f[7]);
    }
    return;
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = __bfloat162float(e[i]);
    xr[i] = p ? v + p[i] : v;
  }
}

int embed_bf16(const int32_t* tokens, const int32_t* positions, const __nv_bfloat16* embed, const float* pos_table,
               int M, int d, float* x, cudaStream_t st, const int32_t* prev_ids) {
  if (M == 0) return ALORA_OK;
  ALORA_CUDA_CHECK(launch_pdl(embed_bf16_kernel, dim3(M), dim3(256), 0, st, nullptr, 0, tokens, positions, embed, pos_table, d, x,
                              prev_ids));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// --------------------------------------------------------------- rmsnorm ---
// One CTA per row, fp32 sum of squares in a fixed tree order; output bf16.
// Row cached in registers (float4 per thread per 1024 columns): x is read once, h written with 8-byte stores.
template <int V>
__global__ void __launch_bounds__(256) rmsnorm_bf16_vec_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows,
                                                               int d, const float* __restrict__ w, float eps,
                                                               __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)src * d);
  const int n4 = d >> 2;
  float4 v[V];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * 256;
    v[j] = i < n4 ? __ldg(xr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss = fmaf(v[j].x, v[j].x, ss); ss = fmaf(v[j].y, v[j].y, ss);
    ss = fmaf(v[j].z, v[j].z, ss); ss = fmaf(v[j].w, v[j].w, ss);
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)r * d);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * 256;
    if (i >= n4) break;
    float4 y = make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
    if (w) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(w) + i);
      y.x *= g.x; y.y *= g.y; y.z *= g.z; y.w *= g.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(y.x, y.y), hi = __floats2bfloat162_rn(y.z, y.w);
    o[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

__global__ void rmsnorm_bf16_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows, int d,
                                    const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float* xr = x + (int64_t)src * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float y = xr[i] * inv;
    if (w) y *= w[i];
    out[(int64_t)r * d + i] = __float2bfloat16_rn(y);
  }
}

int rmsnorm_bf16(const float* x, const int32_t* rows, int n_rows, int d, const float* w, float eps,
                 __nv_bfloat16* out, cudaStream_t st) {
  if (n_rows == 0) return ALORA_OK;
  if (d % 4 == 0 && d <= 8192) {
    const int v = (d / 4 + 255) / 256;
    if (v <= 1) ALORA_CUDA_CHECK(launch_pdl(rmsnorm_bf16_vec_kernel<1>, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, rows, d, w, eps, out));
    else if (v <= 2) ALORA_CUDA_CHECK(launch_pdl(rmsnorm_bf16_vec_kernel<2>, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, rows, d, w, eps, out));
    else if (v <= 4) ALORA_CUDA_CHECK(launch_pdl(rmsnorm_bf16_vec_kernel<4>, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, rows, d, w, eps, out));
    else ALORA_CUDA_CHECK(launch_pdl(rmsnorm_bf16_vec_kernel<8>, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, rows, d, w, eps, out));
  } else {
    ALORA_CUDA_CHECK(launch_pdl(rmsnorm_bf16_kernel, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, rows, d, w, eps, out));
  }
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// Sum of exactly NP split-K partials (all loads issued before the adds; split order kept). A compile-time
// count keeps only NP float4 in flight per call: the runtime-count version held 8 (32 registers), which
// capped qkv_finalize at one 512-thread CTA per SM (two waves at M = 240).
template <int NP>
__device__ __forceinline__ float4 sum_parts_n(const float* __restrict__ base, int64_t pstride) {
  float4 t[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) t[p] = __ldcg(reinterpret_cast<const float4*>(base + p * pstride));
  float4 acc = t[0];
#pragma unroll
  for (int p = 1; p < NP; ++p) { acc.x += t[p].x; acc.y += t[p].y; acc.z += t[p].z; acc.w += t[p].w; }
  return acc;
}

// Dispatch a kernel template on the split count (1..8).
#define ALORA_NP_SWITCH(np, ...)                                          \
  switch (np) {                                                           \
    case 1: { constexpr int NP = 1; __VA_ARGS__; } break;                 \
    case 2: { constexpr int NP = 2; __VA_ARGS__; } break;                 \
    case 3: { constexpr int NP = 3; __VA_ARGS__; } break;                 \
    case 4: { constexpr int NP = 4; __VA_ARGS__; } break;                 \
    case 5: { constexpr int NP = 5; __VA_ARGS__; } break;                 \
    case 6: { constexpr int NP = 6; __VA_ARGS__; } break;                 \
    case 7: { constexpr int NP = 7; __VA_ARGS__; } break;                 \
    default: { constexpr int NP = 8; __VA_ARGS__; } break;                \
  }

// Sum of up to 8 split-K partials at float4 index i (all loads issued before the adds; split order kept).
__device__ __forceinline__ float4 sum_parts4(const float* __restrict__ base, int64_t pstride, int nparts) {
  float4 t[8];
#pragma unroll
  for (int p = 0; p < 8; ++p)
    if (p < nparts) t[p] = __ldcg(reinterpret_cast<const float4*>(base + p * pstride));
  float4 acc = t[0];
#pragma unroll
  for (int p = 1; p < 8; ++p)
    if (p < nparts) { acc.x += t[p].x; acc.y += t[p].y; acc.z += t[p].z; acc.w += t[p].w; }
  return acc;
}

// ------------------------------------------------- deferred split-K consumers ---
// x[src] (+)= sum_p partials[p][src] in split order (the o-proj / MLP-down epilogue the split-K GEMM
// deferred), then out[r] = bf16(rmsnorm(x[src]) * w).
template <int V, int NP>
__global__ void __launch_bounds__(256) residual_rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ part,
                                                               int64_t pstride,
                                                               const int32_t* __restrict__ rows, int d,
                                                               const float* __restrict__ w, float eps,
                                                               __nv_bfloat16* __restrict__ out,
                                                               unsigned long long* __restrict__ zero_rows) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  if (zero_rows && threadIdx.x == 0) zero_rows[r] = 0ull;  // the lm_head's fused argmax accumulates here
  float4* xr = reinterpret_cast<float4*>(x + (int64_t)src * d);
  const int n4 = d >> 2;
  float4 v[V];
  // Loads in flight before the first add: every chunk's at d <= 2048 (V * NP <= 16 float4); one chunk's
  // at a time above that (d = 4096 / 8192), where holding all of them spilled and capped occupancy.
  constexpr int kGroup = V * NP <= 16 ? V : 1;
  float ss = 0.f;
#pragma unroll
  for (int j0 = 0; j0 < V; j0 += kGroup) {
    float4 pp[kGroup][NP > 0 ? NP : 1];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int j = j0 + g, i = threadIdx.x + j * 256;
      v[j] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < NP; ++p)
        if (i < n4) pp[g][p] = __ldcg(reinterpret_cast<const float4*>(part + (int64_t)src * d + 4 * i + p * pstride));
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int j = j0 + g, i = threadIdx.x + j * 256;
      if (NP > 0 && i < n4) {
        float4 acc = pp[g][0];
#pragma unroll
        for (int p = 1; p < NP; ++p) { acc.x += pp[g][p].x; acc.y += pp[g][p].y; acc.z += pp[g][p].z; acc.w += pp[g][p].w; }
        v[j].x += acc.x; v[j].y += acc.y; v[j].z += acc.z; v[j].w += acc.w;
        xr[i] = v[j];
      }
      ss = fmaf(v[j].x, v[j].x, ss); ss = fmaf(v[j].y, v[j].y, ss);
      ss = fmaf(v[j].z, v[j].z, ss); ss = fmaf(v[j].w, v[j].w, ss);
    }
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)r * d);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * 256;
    if (i >= n4) break;
    float4 y = make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
    if (w) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(w) + i);
      y.x *= g.x; y.y *= g.y; y.z *= g.z; y.w *= g.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(y.x, y.y), hi = __floats2bfloat162_rn(y.z, y.w);
    o[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

int residual_rmsnorm_bf16(float* x, const float* partials, int nparts, int M, const int32_t* rows, int n_rows, int d,
                          const float* w, float eps, __nv_bfloat16* out, cudaStream_t st,
                          unsigned long long* zero_rows) {
  if (n_rows == 0) return ALORA_OK;
  if (partials == nullptr) nparts = 0;
  if (d % 4 != 0 || d > 8192) {
    if (nparts > 0 || zero_rows) return ALORA_EINVAL;
    return rmsnorm_bf16(x, rows, n_rows, d, w, eps, out, st);
  }
  if (nparts > 8) return ALORA_EINVAL;
  const int v = (d / 4 + 255) / 256;
  const int64_t ps = (int64_t)M * d;
  cudaError_t err = cudaSuccess;
#define ALORA_RMS_LAUNCH(VV, NPP)                                                                                  \
  err = launch_pdl(residual_rmsnorm_kernel<VV, NPP>, dim3(n_rows), dim3(256), 0, st, nullptr, 0, x, partials, ps, rows, \
                   d, w, eps, out, zero_rows)
#define ALORA_RMS_V(VV)                                          \
  if (nparts == 0) {                                             \
    ALORA_RMS_LAUNCH(VV, 0);                                     \
  } else {                                                       \
    ALORA_NP_SWITCH(nparts, ALORA_RMS_LAUNCH(VV, NP));           \
  }
  if (v <= 1) { ALORA_RMS_V(1) }
  else if (v <= 2) { ALORA_RMS_V(2) }
  else if (v <= 4) { ALORA_RMS_V(4) }
  else { ALORA_RMS_V(8) }
#undef ALORA_RMS_V
#undef ALORA_RMS_LAUNCH
  ALORA_CUDA_CHECK(err);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

__global__ void __launch_bounds__(256) sum_partials_kernel(const float* __restrict__ part, int nparts, int64_t n4,
                                                           float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<float4*>(out)[i] = sum_parts4(part + 4 * i, 4 * n4, nparts);
}

int sum_partials_f32(const float* partials, int nparts, int64_t n, float* out, cudaStream_t st) {
  if (n == 0) return ALORA_OK;
  if (nparts < 1 || nparts > 8 || n % 4) return ALORA_EINVAL;
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 4 * kNumSMs);
  ALORA_CUDA_CHECK(launch_pdl(sum_partials_kernel, dim3(grid), dim3(256), 0, st, nullptr, 0, partials, nparts, n4, out));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// Deferred epilogue of a split-K QKV projection: per row, sum the splits (in order), rotate-half RoPE in
// fp32 on the q and k heads (the kEpiRope math of the GEMM epilogue, one rounding), store q|k|v bf16 and
// scatter the k and v rows into the paged pool (model.py:217-222) -- the step's kv_write, fused.
template <int NP>
__global__ void __launch_bounds__(512, 2) qkv_finalize_kernel(const float* __restrict__ part, int64_t pstride,
                                                           int Nq, int Nkv, int D,
                                                           const int32_t* __restrict__ positions,
                                                           const float* __restrict__ cos_t,
                                                           const float* __restrict__ sin_t,
                                                           __nv_bfloat16* __restrict__ qkv, int ldq,
                                                           const int32_t* __restrict__ slot_mapping,
                                                           __nv_bfloat16* __restrict__ pool, int n_layers, int layer,
                                                           int B) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int N = Nq + 2 * Nkv;
  const int half = D / 2;
  const int pos = positions[m];
  const int slot = slot_mapping[m];
  __nv_bfloat16* krow = nullptr;
  __nv_bfloat16* vrow = nullptr;
  if (slot >= 0) {
    const int64_t blk = slot / B, r = slot % B;
    krow = pool + (((blk * n_layers + layer) * 2 + 0) * B + r) * Nkv;
    vrow = pool + (((blk * n_layers + layer) * 2 + 1) * B + r) * Nkv;
  }
  const float* row = part + (int64_t)m * N;
  auto sum4 = [&](int col) { return sum_parts_n<NP>(row + col, pstride); };
  auto pack4 = [](float a, float b, float c, float d) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
    return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  };
  const int rope_q4 = (Nq + Nkv) / 2 / 4;  // 4-wide groups of rotate pairs over the q and k heads
  const int v4 = Nkv / 4;
  for (int t = threadIdx.x; t < rope_q4 + v4; t += blockDim.x) {
    if (t < rope_q4) {
      const int i = t * 4;                    // pair index
      const int head = i / half, j = i % half;  // 4 pairs stay inside one head (half % 4 == 0)
      const int c1 = head * D + j, c2 = c1 + half;
      const float4 x1 = sum4(c1), x2 = sum4(c2);
      const float4 cs = __ldg(reinterpret_cast<const float4*>(cos_t + (int64_t)pos * half + j));
      const float4 sn = __ldg(reinterpret_cast<const float4*>(sin_t + (int64_t)pos * half + j));
      const uint2 r1 = pack4(x1.x * cs.x - x2.x * sn.x, x1.y * cs.y - x2.y * sn.y, x1.z * cs.z - x2.z * sn.z,
                             x1.w * cs.w - x2.w * sn.w);
      const uint2 r2 = pack4(x2.x * cs.x + x1.x * sn.x, x2.y * cs.y + x1.y * sn.y, x2.z * cs.z + x1.z * sn.z,
                             x2.w * cs.w + x1.w * sn.w);
      *reinterpret_cast<uint2*>(qkv + (int64_t)m * ldq + c1) = r1;
      *reinterpret_cast<uint2*>(qkv + (int64_t)m * ldq + c2) = r2;
      if (krow && c1 >= Nq) {
        *reinterpret_cast<uint2*>(krow + (c1 - Nq)) = r1;
        *reinterpret_cast<uint2*>(krow + (c2 - Nq)) = r2;
      }
    } else {
      const int c = Nq + Nkv + (t - rope_q4) * 4;
      const float4 x = sum4(c);
      const uint2 r = pack4(x.x, x.y, x.z, x.w);
      *reinterpret_cast<uint2*>(qkv + (int64_t)m * ldq + c) = r;
      if (vrow) *reinterpret_cast<uint2*>(vrow + (c - Nq - Nkv)) = r;
    }
  }
}

int qkv_finalize_bf16(const float* partials, int nparts, int M, int Nq, int Nkv, int D, const int32_t* positions,
                      const float* cos_t, const float* sin_t, __nv_bfloat16* qkv, int ldq, const int32_t* slot_mapping,
                      __nv_bfloat16* kv_pool, int n_layers, int layer, int B, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  if (nparts < 1 || nparts > 8 || !partials || !positions || !cos_t || !sin_t || D % 8 || Nq % D || Nkv % D || ldq % 4)
    return ALORA_EINVAL;
  const int64_t ps = (int64_t)M * (Nq + 2 * Nkv);
  cudaError_t err = cudaSuccess;
  ALORA_NP_SWITCH(nparts, err = launch_pdl(qkv_finalize_kernel<NP>, dim3(M), dim3(512), 0, st, nullptr, 0, partials, ps,
                                           Nq, Nkv, D, positions, cos_t, sin_t, qkv, ldq, slot_mapping, kv_pool,
                                           n_layers, layer, B));
  ALORA_CUDA_CHECK(err);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// Deferred epilogue of a split-K shrink: the kEpiLoraSelect row/slot/target select on the summed splits.
__global__ void __launch_bounds__(128) lora_select_finalize_kernel(const float* __restrict__ part, int nparts,
                                                                   int64_t pstride, int M, int SR, int rank,
                                                                   int P, int tbit0,
                                                                   const int32_t* __restrict__ row_slot,
                                                                   const uint8_t* __restrict__ row_apply,
                                                                   const uint8_t* __restrict__ targets,
                                                                   __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int slot = row_slot[m];
  const bool takes = slot >= 0 && row_apply[m];
  const uint32_t tbits = takes ? (uint32_t)targets[slot] >> tbit0 : 0u;
  const float* row = part + (int64_t)m * P * SR;
  for (int c = threadIdx.x * 4; c < P * SR; c += blockDim.x * 4) {
    const int t = c / SR, off = c % SR;  // SR % 4 == 0: a 4-column group stays in one plane
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((tbits >> t) & 1u) acc = sum_parts4(row + c, pstride, nparts);
    float e[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((off + k) / rank != slot) e[k] = 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(e[0], e[1]), hi = __floats2bfloat162_rn(e[2], e[3]);
    *reinterpret_cast<uint2*>(out + ((int64_t)t * M + m) * SR + off) =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

int lora_select_finalize_bf16(const float* partials, int nparts, int M, int SR, int rank, const int32_t* row_slot,
                              const uint8_t* row_apply, const uint8_t* slot_targets, __nv_bfloat16* s,
                              cudaStream_t st, int n_planes, int tbit0) {
  if (M == 0) return ALORA_OK;
  if (nparts < 1 || nparts > 8 || SR % 4 || rank < 1 || n_planes < 1 || tbit0 < 0 || tbit0 + n_planes > 8)
    return ALORA_EINVAL;
  ALORA_CUDA_CHECK(launch_pdl(lora_select_finalize_kernel, dim3(M), dim3(128), 0, st, nullptr, 0, partials, nparts,
                              (int64_t)M * n_planes * SR, M, SR, rank, n_planes, tbit0, row_slot, row_apply,
                              slot_targets, s));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------ rope ---
// Rotate-half RoPE, fp32 math on bf16 q/k (k heads follow the q heads in the row).
__global__ void rope_bf16_kernel(__nv_bfloat16* __restrict__ qkv, int ld, const int32_t* __restrict__ positions,
                                 int H, int Hkv, int D, const float* __restrict__ cos_t,
                                 const float* __restrict__ sin_t) {
  const int m = blockIdx.x;
  const int half = D / 2;
  const int pos = positions[m];
  for (int i = threadIdx.x; i < (H + Hkv) * half; i += blockDim.x) {
    const int head = i / half, j = i % half;
    __nv_bfloat16* b = qkv + (int64_t)m * ld + head * D;
    const float c = cos_t[(int64_t)pos * half + j], s = sin_t[(int64_t)pos * half + j];
    const float x1 = __bfloat162float(b[j]), x2 = __bfloat162float(b[j + half]);
    b[j] = __float2bfloat16_rn(x1 * c - x2 * s);
    b[j + half] = __float2bfloat16_rn(x2 * c + x1 * s);
  }
}

int rope_bf16(__nv_bfloat16* qkv, int ld, const int32_t* positions, int M, int H, int Hkv, int D,
              const float* cos_t, const float* sin_t, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  rope_bf16_kernel<<<M, 256, 0, st>>>(qkv, ld, positions, H, Hkv, D, cos_t, sin_t);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// -------------------------------------------------------------- lora shrink ---
// s[t][m][slot*R + j] = bf16( sum_k h[m,k] * down[t][slot][j][k] ) on the row's own slot when the row takes
// the delta and the adapter targets t; every other entry of the row is written 0 so that the GEMM's extra
// K range contributes exact zeros (rows before the invocation keep the base bits, model.py:145).
// Segmented: one CTA per row, 3*R warps-worth of dot products; down rows stream from L2.
constexpr int kShrinkThreads = 256;

__global__ void __launch_bounds__(kShrinkThreads) lora_shrink_bf16_kernel(
    const __nv_bfloat16* __restrict__ h, int M, int K, const int32_t* __restrict__ row_slot,
    const uint8_t* __restrict__ row_apply, const __nv_bfloat16* __restrict__ down, int n_slots, int R,
    const uint8_t* __restrict__ slot_targets, __nv_bfloat16* __restrict__ s, int P, int tbit0) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  pdl_wait();  // h comes from the RMSNorm before
  pdl_trigger();
  const int m = blockIdx.x;
  const int KS = n_slots * R;
  const int slot = row_slot[m];
  const bool take = slot >= 0 && row_apply[m];
  const uint32_t tb = take ? (uint32_t)slot_targets[slot] >> tbit0 : 0u;
  // zero the row's P * KS entries (other slots, untargeted projections)
  for (int i = threadIdx.x; i < P * KS; i += blockDim.x) {
    const int t = i / KS, c = i % KS;
    const bool mine = take && (c / R == slot) && ((tb >> t) & 1);
    if (!mine) s[((int64_t)t * M + m) * KS + c] = __float2bfloat16_rn(0.f);
  }
  if (!take) return;
  const __nv_bfloat16* xr = h + (int64_t)m * K;
  for (int i = threadIdx.x * 8; i < K; i += blockDim.x * 8) *reinterpret_cast<int4*>(xs + i) = *reinterpret_cast<const int4*>(xr + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int o = warp; o < P * R; o += nwarps) {
    const int t = o / R, j = o % R;
    if (!((tb >> t) & 1)) continue;
    const __nv_bfloat16* dn = down + (((int64_t)t * n_slots + slot) * R + j) * K;
    float acc = 0.f;
    for (int k = lane * 8; k < K; k += 256) {
      const int4 a = *reinterpret_cast<const int4*>(xs + k);
      const int4 b = __ldg(reinterpret_cast<const int4*>(dn + k));
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 fa = __bfloat1622float2(a2[e]), fb = __bfloat1622float2(b2[e]);
        acc = fmaf(fa.x, fb.x, acc);
        acc = fmaf(fa.y, fb.y, acc);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) s[((int64_t)t * M + m) * KS + slot * R + j] = __float2bfloat16_rn(acc);
  }
}

int lora_shrink_bf16(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                     const __nv_bfloat16* down, int n_slots, int R, const uint8_t* slot_targets, __nv_bfloat16* s,
                     cudaStream_t st, int n_planes, int tbit0) {
  if (M == 0 || n_slots == 0) return ALORA_OK;
  if (K % 8 != 0 || n_planes < 1 || tbit0 < 0 || tbit0 + n_planes > 8) return ALORA_EINVAL;
  if (K * 2 > 48 * 1024) {
    static bool configured = false;
    if (!configured) {
      if (cudaFuncSetAttribute(lora_shrink_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, K * 2) !=
          cudaSuccess)
        return ALORA_ECUDA;
      configured = true;
    }
  }
  ALORA_CUDA_CHECK(launch_pdl(lora_shrink_bf16_kernel, dim3(M), dim3(kShrinkThreads), (size_t)K * 2, st, nullptr, 0, h,
                              M, K, row_slot, row_apply, down, n_slots, R, slot_targets, s, n_planes, tbit0));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------------------------------------------------
// Segmented LoRA shrink (model.py:141, `x @ down_t` of the rows that take the delta): the aLoRA eval step has
// only the post-invocation rows of each request (and decode rows) on an adapter, a few dozen to a few hundred
// per adapter, so the work is each adapter's down matrices streamed once against its own rows -- bandwidth, not
// tensor throughput. Work item = (adapter slot, chunk of 64 of its active rows), one cluster of KS CTAs per item,
// CTA `rank` owning the K range [rank K/KS, (rank+1) K/KS):
//   before the dependency wait  the chunk's active rows (row_slot == slot and row_apply, in row order) are
//                               listed (step metadata, not written by the kernels before)
//   after it                    K sub-slices of 128 stream through a cp.async ring: the down rows of every
//                               targeted plane [P*R x 128] and the chunk's h rows [64 x 128]; warp w computes the
//                               [16-row tile w%4] x [half w/4 of the P*R columns] outputs with mma.sync m16n8k16,
//                               each warp over the whole K range in order (no intra-CTA reduction)
//   reduction                   the KS ranks' [64 x P*R] partials through DSMEM, summed in rank order (every rank
//                               reduces a slice of the outputs), written to s[t][row][slot*R + j] in bf16
//   zero fill                   chunk 0 of each slot writes 0 to every other row's entries of this slot in every
//                               plane (and to all rows of an untargeted plane), so the expand GEMM (extra K of the
//                               projection) adds exact zeros there (base rows stay bitwise, model.py:145)
// KS depends on K only and a row's sums never depend on its chunk or warp: the result is batch invariant.
constexpr int kSegThreads = 256;
constexpr int kSegRowChunk = 64;
constexpr int kSegKB = 128;  // K sub-slice per ring stage

__device__ __forceinline__ uint32_t smem_u32addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void seg_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32addr(dst)), "l"(src));
}
__device__ __forceinline__ void seg_ldsm4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32addr(p)));
}
__device__ __forceinline__ void seg_ldsm2(uint32_t (&r)[2], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(smem_u32addr(p)));
}
__device__ __forceinline__ void seg_mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// [rows][kSegKB] bf16 tile, 16-byte chunk c of row r at chunk (c ^ (r & 7))
__device__ __forceinline__ int seg_off(int row, int k) {
  const int c = (k >> 3) ^ (row & 7);
  return row * kSegKB + (c << 3) + (k & 7);
}

template <int R, int P>
struct SegCfg {
  static constexpr int kN = P * R;                      // output columns of an item (all planes)
  static constexpr int kNT = kN / 8;                    // n8 tiles
  static constexpr int kNTW = (kNT + 1) / 2;            // n8 tiles per warp (two column halves)
  static constexpr int kStage = (kN + kSegRowChunk) * kSegKB * 2;
  static constexpr int kRed = kSegRowChunk * kN * 4;
  static constexpr int kStages = (200 * 1024 - kRed) / kStage < 4 ? (200 * 1024 - kRed) / kStage : 4;
  static constexpr int kSmem = kStages * kStage + kRed;
  static_assert(kStages >= 2, "shrink ring");
};

template <int R, int P>
__global__ void __launch_bounds__(kSegThreads) lora_shrink_seg_kernel(
    const __nv_bfloat16* __restrict__ h, int M, int K, int KS, const int32_t* __restrict__ row_slot,
    const uint8_t* __restrict__ row_apply, const __nv_bfloat16* __restrict__ down, int n_slots,
    const uint8_t* __restrict__ slot_targets, __nv_bfloat16* __restrict__ s, int tbit0) {
  using C = SegCfg<R, P>;
  extern __shared__ __align__(128) uint8_t seg_smem[];
  float* red = reinterpret_cast<float*>(seg_smem + C::kStages * C::kStage);  // [64][kN] this rank's partial
  __shared__ int rows[kSegRowChunk];
  __shared__ int warp_cnt[kSegThreads / 32];
  const int slot = blockIdx.x % n_slots, chunk = blockIdx.x / n_slots;
  const int rank = blockIdx.y;  // == cluster rank (cluster dims (1, KS, 1))
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Kr = K / KS, k_base = rank * Kr, n_sub = Kr / kSegKB;
  const int ldS = n_slots * R;
  const int tmask = (slot_targets[slot] >> tbit0) & ((1 << P) - 1);
  // active rows of this chunk (ordinals [chunk*64, chunk*64 + 64) among the slot's rows, in row order)
  const int per_warp = (M + (kSegThreads / 32) - 1) / (kSegThreads / 32);
  const int r_lo = warp * per_warp, r_hi = min(M, r_lo + per_warp);
  int cnt = 0;
  for (int r = r_lo + lane; r - lane < r_hi; r += 32) {
    const bool act = r < r_hi && row_slot[r] == slot && row_apply[r];
    cnt += __popc(__ballot_sync(0xffffffffu, act));
  }
  if (lane == 0) warp_cnt[warp] = cnt;
  __syncthreads();
  int base = 0, n_act = 0;
  for (int w = 0; w < kSegThreads / 32; ++w) {
    if (w < warp) base += warp_cnt[w];
    n_act += warp_cnt[w];
  }
  const int c0 = chunk * kSegRowChunk, nc = max(0, min(kSegRowChunk, n_act - c0));
  {
    int ord = base;
    for (int r = r_lo + lane; r - lane < r_hi; r += 32) {
      const bool act = r < r_hi && row_slot[r] == slot && row_apply[r];
      const unsigned b = __ballot_sync(0xffffffffu, act);
      const int my = ord + __popc(b & ((1u << lane) - 1));
      if (act && my >= c0 && my < c0 + nc) rows[my - c0] = r;
      ord += __popc(b);
    }
  }
  __syncthreads();
  const bool work = nc > 0 && tmask != 0;  // uniform over the cluster (same slot and chunk)
  // down sub-slices do not depend on the previous kernel; h does
  auto load_down = [&](int sub) {
    __nv_bfloat16* sd = reinterpret_cast<__nv_bfloat16*>(seg_smem + (sub % C::kStages) * C::kStage);
    const int k0 = k_base + sub * kSegKB;
    for (int i = tid; i < C::kN * (kSegKB / 8); i += kSegThreads) {
      const int q = i / (kSegKB / 8), c = i % (kSegKB / 8);
      const int t = q / R, j = q % R;
      if ((tmask >> t) & 1)
        seg_cp16(sd + seg_off(q, c * 8), down + (((int64_t)t * n_slots + slot) * R + j) * K + k0 + c * 8);
    }
  };
  auto load_h = [&](int sub) {
    __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(seg_smem + (sub % C::kStages) * C::kStage) + C::kN * kSegKB;
    const int k0 = k_base + sub * kSegKB;
    for (int i = tid; i < kSegRowChunk * (kSegKB / 8); i += kSegThreads) {
      const int rr = i / (kSegKB / 8), c = i % (kSegKB / 8);
      if (rr < nc) seg_cp16(sh + seg_off(rr, c * 8), h + (int64_t)rows[rr] * K + k0 + c * 8);
      else *reinterpret_cast<int4*>(sh + seg_off(rr, c * 8)) = make_int4(0, 0, 0, 0);
    }
  };
  if (work)
    for (int sub = 0; sub < min(n_sub, C::kStages - 1); ++sub) load_down(sub);
  pdl_wait();
  pdl_trigger();
  if (chunk == 0) {  // zero every row of this slot that takes no delta, in every plane; ranks split the rows
    const int rows_per = (M + KS - 1) / KS;
    const int z0 = rank * rows_per, z1 = min(M, z0 + rows_per);
    for (int i = tid; i < (z1 - z0) * P * (R / 8); i += kSegThreads) {
      const int r = z0 + i / (P * (R / 8)), t = (i / (R / 8)) % P, c = (i % (R / 8)) * 8;
      if (((tmask >> t) & 1) && row_slot[r] == slot && row_apply[r]) continue;
      *reinterpret_cast<int4*>(s + ((int64_t)t * M + r) * ldS + slot * R + c) = make_int4(0, 0, 0, 0);
    }
  }
  if (!work) return;
  for (int sub = 0; sub < C::kStages - 1; ++sub) {  // exactly kStages - 1 groups, so the wait below is exact
    if (sub < n_sub) load_h(sub);
    asm volatile("cp.async.commit_group;");  // group `sub` = its h (+ every down issued so far)
  }
  const int rt = warp & 3, nh = warp >> 2;  // 16-row tile, column half
  const bool rows_live = rt * 16 < nc;
  float acc[C::kNTW][4];
#pragma unroll
  for (int f = 0; f < C::kNTW; ++f)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[f][e] = 0.f;
  for (int sub = 0; sub < n_sub; ++sub) {
    const int nxt = sub + C::kStages - 1;
    if (nxt < n_sub) {
      __syncthreads();  // stage nxt % kStages (last used by sub - 1) is no longer read
      load_down(nxt);
      load_h(nxt);
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(C::kStages - 1) : "memory");
    __syncthreads();
    const __nv_bfloat16* sd = reinterpret_cast<const __nv_bfloat16*>(seg_smem + (sub % C::kStages) * C::kStage);
    const __nv_bfloat16* sh = sd + C::kN * kSegKB;
    if (rows_live) {
#pragma unroll
      for (int ks = 0; ks < kSegKB; ks += 16) {
        uint32_t afr[4];
        seg_ldsm4(afr, sh + seg_off(rt * 16 + (lane & 15), ks + (lane >> 4) * 8));
#pragma unroll
        for (int f = 0; f < C::kNTW; ++f) {
          const int nt = nh * C::kNTW + f;
          if (nt >= C::kNT) break;
          uint32_t b2[2];
          seg_ldsm2(b2, sd + seg_off(nt * 8 + (lane & 7), ks + ((lane >> 3) & 1) * 8));
          seg_mma(acc[f], afr, b2[0], b2[1]);
        }
      }
    }
  }
  // this rank's partial -> smem (each warp its own outputs)
  if (rows_live) {
#pragma unroll
    for (int f = 0; f < C::kNTW; ++f) {
      const int nt = nh * C::kNTW + f;
      if (nt >= C::kNT) break;
      const int r0 = rt * 16 + (lane >> 2), c = nt * 8 + (lane & 3) * 2;
      *reinterpret_cast<float2*>(red + r0 * C::kN + c) = make_float2(acc[f][0], acc[f][1]);
      *reinterpret_cast<float2*>(red + (r0 + 8) * C::kN + c) = make_float2(acc[f][2], acc[f][3]);
    }
  }
  if (KS > 1) asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
  else __syncthreads();
  // rank q sums outputs [q n / KS, (q+1) n / KS) over the ranks in rank order
  const int n_out = nc * C::kN;
  const int o0 = rank * n_out / KS, o1 = (rank + 1) * n_out / KS;
  for (int i = o0 + tid; i < o1; i += kSegThreads) {
    const int rr = i / C::kN, q = i % C::kN, t = q / R, j = q % R;
    if (!((tmask >> t) & 1)) continue;
    float v = 0.f;
    for (int src = 0; src < KS; ++src) {
      float x;
      if (KS > 1) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32addr(red + i)), "r"(src));
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(ra) : "memory");
      } else {
        x = red[i];
      }
      v += x;
    }
    s[((int64_t)t * M + rows[rr]) * ldS + slot * R + j] = __float2bfloat16_rn(v);
  }
  if (KS > 1) asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// cluster size: 8 CTAs over K when every rank gets whole 128-wide sub-slices (fixed by K alone: batch invariant)
int seg_split(int K) {
  for (int ks : {8, 4, 2, 1})
    if (K % (ks * kSegKB) == 0) return ks;
  return -1;
}

bool lora_shrink_seg_fits(int K) { return seg_split(K) > 0; }

template <int R, int P>
int launch_shrink_seg(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                      const __nv_bfloat16* down, int n_slots, const uint8_t* slot_targets, __nv_bfloat16* s,
                      cudaStream_t st, int tbit0, int max_rows) {
  using C = SegCfg<R, P>;
  const int KS = seg_split(K);
  if (KS < 1) return ALORA_EINVAL;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(lora_shrink_seg_kernel<R, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  const int chunks = std::max(1, (std::min(max_rows, M) + kSegRowChunk - 1) / kSegRowChunk);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = KS;
  attr[0].val.clusterDim.z = 1;
  ALORA_CUDA_CHECK(launch_pdl(lora_shrink_seg_kernel<R, P>, dim3(n_slots * chunks, KS), dim3(kSegThreads), C::kSmem,
                              st, attr, KS > 1 ? 1 : 0, h, M, K, KS, row_slot, row_apply, down, n_slots, slot_targets,
                              s, tbit0));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

template <int R>
int launch_shrink_seg_p(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                        const __nv_bfloat16* down, int n_slots, const uint8_t* slot_targets, __nv_bfloat16* s,
                        cudaStream_t st, int P, int tbit0, int max_rows) {
  switch (P) {
    case 1: return launch_shrink_seg<R, 1>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, tbit0, max_rows);
    case 2: return launch_shrink_seg<R, 2>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, tbit0, max_rows);
    case 3: return launch_shrink_seg<R, 3>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, tbit0, max_rows);
    default: return ALORA_EINVAL;
  }
}

int lora_shrink_seg_bf16(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                         const __nv_bfloat16* down, int n_slots, int R, const uint8_t* slot_targets,
                         __nv_bfloat16* s, cudaStream_t st, int P, int tbit0, int max_rows) {
  if (M == 0 || n_slots == 0) return ALORA_OK;
  if (K % kSegKB != 0 || P < 1 || P > 3 || tbit0 < 0 || tbit0 + P > 8) return ALORA_EINVAL;
  switch (R) {
    case 8: return launch_shrink_seg_p<8>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, P, tbit0, max_rows);
    case 16: return launch_shrink_seg_p<16>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, P, tbit0, max_rows);
    case 32: return launch_shrink_seg_p<32>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, P, tbit0, max_rows);
    case 64: return launch_shrink_seg_p<64>(h, M, K, row_slot, row_apply, down, n_slots, slot_targets, s, st, P, tbit0, max_rows);
    default: return ALORA_EINVAL;
  }
}

// One 32-bit mask per 128-row GEMM tile: bit `slot` set when any row of the tile takes that adapter's delta.
__global__ void lora_tile_masks_kernel(const int32_t* __restrict__ row_slot, const uint8_t* __restrict__ row_apply,
                                       int M, uint32_t* __restrict__ masks) {
  pdl_wait();
  pdl_trigger();
  const int tile = blockIdx.x;
  const int m = tile * 128 + threadIdx.x;
  uint32_t bit = 0;
  if (m < M) {
    const int slot = row_slot[m];
    if (slot >= 0 && slot < 32 && row_apply[m]) bit = 1u << slot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bit |= __shfl_xor_sync(0xffffffffu, bit, o);
  __shared__ uint32_t part[4];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = bit;
  __syncthreads();
  if (threadIdx.x == 0) masks[tile] = part[0] | part[1] | part[2] | part[3];
}

void configure_bf16_ops() {
  prefer_max_smem(embed_bf16_kernel);
  prefer_max_smem(rmsnorm_bf16_kernel);
  prefer_max_smem(rope_bf16_kernel);
  prefer_max_smem(lora_shrink_bf16_kernel);
  prefer_max_smem(lora_tile_masks_kernel);
  prefer_max_smem(rmsnorm_bf16_vec_kernel<1>);
  prefer_max_smem(rmsnorm_bf16_vec_kernel<2>);
  prefer_max_smem(rmsnorm_bf16_vec_kernel<4>);
  prefer_max_smem(rmsnorm_bf16_vec_kernel<8>);
#define ALORA_PREFER_RMS(VV)                                                                                 \
  prefer_max_smem(residual_rmsnorm_kernel<VV, 0>); prefer_max_smem(residual_rmsnorm_kernel<VV, 1>);             \
  prefer_max_smem(residual_rmsnorm_kernel<VV, 2>); prefer_max_smem(residual_rmsnorm_kernel<VV, 3>);             \
  prefer_max_smem(residual_rmsnorm_kernel<VV, 4>); prefer_max_smem(residual_rmsnorm_kernel<VV, 5>);             \
  prefer_max_smem(residual_rmsnorm_kernel<VV, 6>); prefer_max_smem(residual_rmsnorm_kernel<VV, 7>);             \
  prefer_max_smem(residual_rmsnorm_kernel<VV, 8>);
  ALORA_PREFER_RMS(1) ALORA_PREFER_RMS(2) ALORA_PREFER_RMS(4) ALORA_PREFER_RMS(8)
#undef ALORA_PREFER_RMS
  prefer_max_smem(qkv_finalize_kernel<1>); prefer_max_smem(qkv_finalize_kernel<2>);
  prefer_max_smem(qkv_finalize_kernel<3>); prefer_max_smem(qkv_finalize_kernel<4>);
  prefer_max_smem(qkv_finalize_kernel<5>); prefer_max_smem(qkv_finalize_kernel<6>);
  prefer_max_smem(qkv_finalize_kernel<7>); prefer_max_smem(qkv_finalize_kernel<8>);
  prefer_max_smem(lora_select_finalize_kernel);
  prefer_max_smem(sum_partials_kernel);
}

int lora_tile_masks(const int32_t* row_slot, const uint8_t* row_apply, int M, uint32_t* masks, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  ALORA_CUDA_CHECK(launch_pdl(lora_tile_masks_kernel, dim3((M + 127) / 128), dim3(128), 0, st, nullptr, 0, row_slot, row_apply, M, masks));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace alora
