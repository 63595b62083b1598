// bf16-tier elementwise / row kernels around the tensor-core GEMM and attention:
// embedding gather, RMSNorm -> bf16 GEMM operand, RoPE, the segmented LoRA
// shrink and the per-tile adapter masks that let the GEMM skip absent adapters.

#include "common.cuh"
#include "kernels.h"

namespace alora {

// ----------------------------------------------------------------- embed ---
// x (fp32 residual) = embed[tok] (+ sinusoidal pos for the ref arch, model.py:263)
__global__ void embed_bf16_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                                  const __nv_bfloat16* __restrict__ embed, const float* __restrict__ pos_table, int d,
                                  float* __restrict__ x) {
  const int m = blockIdx.x;
  const __nv_bfloat16* e = embed + (int64_t)tokens[m] * d;
  const float* p = pos_table ? pos_table + (int64_t)positions[m] * d : nullptr;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = __bfloat162float(e[i]);
    x[(int64_t)m * d + i] = p ? v + p[i] : v;
  }
}

int embed_bf16(const int32_t* tokens, const int32_t* positions, const __nv_bfloat16* embed, const float* pos_table,
               int M, int d, float* x, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  embed_bf16_kernel<<<M, 256, 0, st>>>(tokens, positions, embed, pos_table, d, x);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// --------------------------------------------------------------- rmsnorm ---
// One CTA per row, fp32 sum of squares in a fixed tree order; output bf16.
__global__ void rmsnorm_bf16_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows, int d,
                                    const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float* xr = x + (int64_t)src * d;
  float ss = 0.f;
  if ((d & 3) == 0) {
    for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
      const float4 v = *reinterpret_cast<const float4*>(xr + i);
      ss = fmaf(v.x, v.x, ss); ss = fmaf(v.y, v.y, ss); ss = fmaf(v.z, v.z, ss); ss = fmaf(v.w, v.w, ss);
    }
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  }
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
  rmsnorm_bf16_kernel<<<n_rows, 256, 0, st>>>(x, rows, d, w, eps, out);
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
    const uint8_t* __restrict__ slot_targets, __nv_bfloat16* __restrict__ s) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  const int m = blockIdx.x;
  const int KS = n_slots * R;
  const int slot = row_slot[m];
  const bool take = slot >= 0 && row_apply[m];
  // zero the row's 3 * KS entries (other slots, untargeted projections)
  for (int i = threadIdx.x; i < 3 * KS; i += blockDim.x) {
    const int t = i / KS, c = i % KS;
    const bool mine = take && (c / R == slot) && ((slot_targets[slot] >> t) & 1);
    if (!mine) s[((int64_t)t * M + m) * KS + c] = __float2bfloat16_rn(0.f);
  }
  if (!take) return;
  const __nv_bfloat16* xr = h + (int64_t)m * K;
  for (int i = threadIdx.x * 8; i < K; i += blockDim.x * 8) *reinterpret_cast<int4*>(xs + i) = *reinterpret_cast<const int4*>(xr + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int o = warp; o < 3 * R; o += nwarps) {
    const int t = o / R, j = o % R;
    if (!((slot_targets[slot] >> t) & 1)) continue;
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
                     cudaStream_t st) {
  if (M == 0 || n_slots == 0) return ALORA_OK;
  if (K % 8 != 0) return ALORA_EINVAL;
  lora_shrink_bf16_kernel<<<M, kShrinkThreads, K * 2, st>>>(h, M, K, row_slot, row_apply, down, n_slots, R,
                                                            slot_targets, s);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// One 32-bit mask per 128-row GEMM tile: bit `slot` set when any row of the tile takes that adapter's delta.
__global__ void lora_tile_masks_kernel(const int32_t* __restrict__ row_slot, const uint8_t* __restrict__ row_apply,
                                       int M, uint32_t* __restrict__ masks) {
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
}

int lora_tile_masks(const int32_t* row_slot, const uint8_t* row_apply, int M, uint32_t* masks, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  lora_tile_masks_kernel<<<(M + 127) / 128, 128, 0, st>>>(row_slot, row_apply, M, masks);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace alora
