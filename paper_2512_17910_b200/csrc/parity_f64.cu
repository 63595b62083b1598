// fp32-storage / fp64-accumulation kernels: the reference's numerics on the GPU.
//
// Every product the reference computes as fp32(fp64(a) @ fp64(b))
// (model.py:95-98) is computed here with fp64 FMA chains in a fixed,
// M-independent order and rounded once to fp32, so each output row is a
// function of its input row only (batch-, chunk- and placement-invariant, the
// property test_model.py:167-202 pins). Softmax, RMSNorm, RoPE and SiLU also
// run in fp64 like model.py:101-104, 179-186. These are SIMT kernels: the
// ALORA_F32 dtype is the parity tier; the tensor-core tier is ALORA_BF16.

#include "common.cuh"
#include "kernels.h"

namespace alora {

// ----------------------------------------------------------------- embed ---
__global__ void embed_f32_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                                 const float* __restrict__ embed, const float* __restrict__ pos_table, int d,
                                 float* __restrict__ x, const int32_t* __restrict__ prev_ids) {
  const int m = blockIdx.x;
  int tok = tokens[m];
  if (tok < 0) tok = prev_ids[-tok - 1];  // the previous forward's greedy id of that span (see embed_bf16)
  const float* e = embed + (int64_t)tok * d;
  const float* p = pos_table ? pos_table + (int64_t)positions[m] * d : nullptr;
  for (int i = threadIdx.x; i < d; i += blockDim.x) x[(int64_t)m * d + i] = p ? e[i] + p[i] : e[i];
}

int embed_f32(const int32_t* tokens, const int32_t* positions, const float* embed, const float* pos_table,
              int M, int d, float* x, cudaStream_t st, const int32_t* prev_ids) {
  if (M == 0) return ALORA_OK;
  embed_f32_kernel<<<M, 256, 0, st>>>(tokens, positions, embed, pos_table, d, x, prev_ids);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// --------------------------------------------------------------- rmsnorm ---
// out[r] = fp32( x64 / sqrt(mean(x64^2) + eps) * w64 ), rows gathered through `rows` (or identity).
__global__ void rmsnorm_f64_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows, int d,
                                   const float* __restrict__ w, float eps, float* __restrict__ out) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float* xr = x + (int64_t)src * d;
  double ss = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double v = xr[i];
    ss = fma(v, v, ss);
  }
  ss = block_sum(ss, red);
  const double scale = sqrt(ss / (double)d + (double)eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double y = (double)xr[i] / scale;
    if (w) y *= (double)w[i];
    out[(int64_t)r * d + i] = (float)y;
  }
}

int rmsnorm_f64(const float* x, const int32_t* rows, int n_rows, int d, const float* w, float eps, float* out,
                cudaStream_t st) {
  if (n_rows == 0) return ALORA_OK;
  rmsnorm_f64_kernel<<<n_rows, 256, 0, st>>>(x, rows, d, w, eps, out);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------ gemm ---
// C[m, n] = epi( fp32( sum_k fp64(A[m,k]) * fp64(Bt[n,k]) ) ), k ascending per element.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f64_kernel(const float* __restrict__ A, int lda,
                                                       const float* __restrict__ Bt, int ldb, float* __restrict__ C,
                                                       int ldc, int M, int N, int K) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ double As[BK][BM + 1];
  __shared__ double Bs[BK][BN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      int mm = i / BK, kk = i % BK;
      int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? (double)A[(int64_t)gm * lda + gk] : 0.0;
      int gn = n0 + mm;
      Bs[kk][mm] = (gn < N && gk < K) ? (double)Bt[(int64_t)gn * ldb + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = (float)acc[i][j];
      float* c = C + (int64_t)gm * ldc + gn;
      if (EPI == kEpiStore) *c = v;
      else if (EPI == kEpiAdd) *c = *c + v;
      else if (EPI == kEpiRelu) *c = fmaxf(v, 0.0f);
    }
  }
}

int gemm_f64(int epi, const float* A, int lda, const float* Bt, int ldb, float* C, int ldc, int M, int N, int K,
             cudaStream_t st) {
  if (M == 0 || N == 0) return ALORA_OK;
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  switch (epi) {
    case kEpiStore: gemm_f64_kernel<kEpiStore><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, C, ldc, M, N, K); break;
    case kEpiAdd: gemm_f64_kernel<kEpiAdd><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, C, ldc, M, N, K); break;
    case kEpiRelu: gemm_f64_kernel<kEpiRelu><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, C, ldc, M, N, K); break;
    default: return ALORA_EINVAL;
  }
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------ lora ---
// Shrink: s[t][m][j] = fp32( sum_k h[m,k] * down[t][slot][j][k] ) for rows that take the delta;
// one warp per (m, t, j), lane-strided k, fixed shuffle tree.
__global__ void lora_shrink_f64_kernel(const float* __restrict__ h, int K, const int32_t* __restrict__ row_slot,
                                       const uint8_t* __restrict__ row_apply, const float* __restrict__ down,
                                       int n_slots, int R, const uint8_t* __restrict__ slot_targets, int M,
                                       float* __restrict__ s) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = M * 3 * R;
  if (warp >= total) return;
  const int j = warp % R, t = (warp / R) % 3, m = warp / (3 * R);
  const int slot = row_slot[m];
  float* dst = s + ((int64_t)t * M + m) * R + j;
  if (slot < 0 || !row_apply[m] || !((slot_targets[slot] >> t) & 1)) {
    if (lane == 0) *dst = 0.0f;
    return;
  }
  const float* x = h + (int64_t)m * K;
  const float* dn = down + (((int64_t)t * n_slots + slot) * R + j) * K;
  double acc = 0.0;
  for (int k = lane; k < K; k += 32) acc = fma((double)x[k], (double)dn[k], acc);
  acc = warp_sum(acc);
  if (lane == 0) *dst = (float)acc;
}

// Expand + row select: out[m,n] = base + fp32( sum_j s[t][m][j] * up_t[n][slot*R + j] ) where the row
// takes the delta and the adapter targets column n's projection; other rows keep the base bits.
__global__ void lora_expand_select_f64_kernel(const float* __restrict__ s, const int32_t* __restrict__ row_slot,
                                              const uint8_t* __restrict__ row_apply,
                                              const float* __restrict__ up_t, int n_slots, int R,
                                              const uint8_t* __restrict__ slot_targets, int M, int Nq, int Nkv,
                                              float* __restrict__ out, int ld_out) {
  const int m = blockIdx.y;
  const int slot = row_slot[m];
  if (slot < 0 || !row_apply[m]) return;
  const int N = Nq + 2 * Nkv;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const int t = n < Nq ? 0 : (n < Nq + Nkv ? 1 : 2);
    if (!((slot_targets[slot] >> t) & 1)) continue;
    const float* sr = s + ((int64_t)t * M + m) * R;
    const float* ur = up_t + (int64_t)n * n_slots * R + (int64_t)slot * R;
    double acc = 0.0;
    for (int j = 0; j < R; ++j) acc = fma((double)sr[j], (double)ur[j], acc);
    float* o = out + (int64_t)m * ld_out + n;
    *o = *o + (float)acc;
  }
}

int lora_f64(const float* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply, const float* down,
             const float* up_t, int n_slots, int R, const uint8_t* slot_targets, float* s_ws, int Nq, int Nkv,
             float* out, int ld_out, cudaStream_t st) {
  if (M == 0 || n_slots == 0 || R == 0) return ALORA_OK;
  const int warps = M * 3 * R;
  lora_shrink_f64_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(h, K, row_slot, row_apply, down, n_slots, R,
                                                                   slot_targets, M, s_ws);
  ALORA_LAUNCH_CHECK();
  const int N = Nq + 2 * Nkv;
  dim3 grid((N + 255) / 256, M);
  lora_expand_select_f64_kernel<<<grid, 256, 0, st>>>(s_ws, row_slot, row_apply, up_t, n_slots, R, slot_targets,
                                                      M, Nq, Nkv, out, ld_out);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------ rope ---
// Rotate-half RoPE in fp64 on fp32 q (H heads) and k (Hkv heads) of the packed qkv rows.
__global__ void rope_f64_kernel(float* __restrict__ qkv, int ld, const int32_t* __restrict__ positions, int H,
                                int Hkv, int D, const float* __restrict__ cos_t, const float* __restrict__ sin_t) {
  const int m = blockIdx.x;
  const int half = D / 2;
  const int pos = positions[m];
  const int pairs = (H + Hkv) * half;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int head = i / half, j = i % half;
    float* base = qkv + (int64_t)m * ld + head * D;  // k heads follow q heads contiguously
    const double c = cos_t[(int64_t)pos * half + j], s = sin_t[(int64_t)pos * half + j];
    const double x1 = base[j], x2 = base[j + half];
    base[j] = (float)(x1 * c - x2 * s);
    base[j + half] = (float)(x2 * c + x1 * s);
  }
}

int rope_f64(float* qkv, int ld, const int32_t* positions, int M, int H, int Hkv, int D, const float* cos_t,
             const float* sin_t, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  rope_f64_kernel<<<M, 128, 0, st>>>(qkv, ld, positions, H, Hkv, D, cos_t, sin_t);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------------ silu ---
// a[m, f] = fp32( silu(g64) * u64 ); gate/up interleaved in blocks of kGluBlock columns.
__global__ void silu_mul_f64_kernel(const float* __restrict__ gu, int F, float* __restrict__ a) {
  const int m = blockIdx.y;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    const int blk = f / kGluBlock, off = f % kGluBlock;
    const float* row = gu + (int64_t)m * 2 * F;
    const double g = row[blk * 2 * kGluBlock + off];
    const double u = row[blk * 2 * kGluBlock + kGluBlock + off];
    a[(int64_t)m * F + f] = (float)(g / (1.0 + exp(-g)) * u);
  }
}

int silu_mul_f64(const float* gu, int M, int F, float* a, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  dim3 grid((F + 255) / 256, M);
  silu_mul_f64_kernel<<<grid, 256, 0, st>>>(gu, F, a);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ------------------------------------------------------------- attention ---
// One CTA per (query row, head). Three passes over the keys in a fixed order
// (max, normaliser, weighted sum), all fp64, weights normalised before the
// V product like model.py:183-186.
constexpr int kAttnThreads = 128;
constexpr int kAttnChunk = 512;

__global__ void __launch_bounds__(kAttnThreads) attn_f64_kernel(
    const float* __restrict__ q, int64_t ld_q, int n_seqs, const int32_t* __restrict__ cu_q,
    const int32_t* __restrict__ start_pos, const int32_t* __restrict__ block_table, int max_blocks,
    const float* __restrict__ kv, int n_layers, int layer, int B, int H, int Hkv, int D, double sqrt_d,
    float* __restrict__ out, int64_t ld_out) {
  __shared__ double qs[256];
  __shared__ double w[kAttnChunk];
  __shared__ double red[32];
  __shared__ int blk_cache[kAttnChunk];
  const int m = blockIdx.x, h = blockIdx.y;
  const int s = seq_of_row(cu_q, n_seqs, m);
  const int pos = start_pos[s] + (m - cu_q[s]);
  const int T = pos + 1;
  const int kvh = h / (H / Hkv);
  const int kvw = Hkv * D;
  const int32_t* bt = block_table + (int64_t)s * max_blocks;
  for (int i = threadIdx.x; i < D; i += blockDim.x) qs[i] = (double)q[(int64_t)m * ld_q + h * D + i];
  __syncthreads();
  auto key_ptr = [&](int t, int kvsel) -> const float* {
    const int64_t blk = bt[t / B];
    return kv + ((((blk * n_layers + layer) * 2 + kvsel) * B + (t % B)) * (int64_t)kvw) + kvh * D;
  };
  // pass 1: max score
  double mx = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float* k = key_ptr(t, 0);
    double dot = 0.0;
    for (int i = 0; i < D; ++i) dot = fma(qs[i], (double)k[i], dot);
    mx = fmax(mx, dot / sqrt_d);
  }
  mx = block_max(mx, red, (double)-INFINITY);
  // pass 2: normaliser
  double z = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float* k = key_ptr(t, 0);
    double dot = 0.0;
    for (int i = 0; i < D; ++i) dot = fma(qs[i], (double)k[i], dot);
    z += exp(dot / sqrt_d - mx);
  }
  z = block_sum(z, red);
  // pass 3: context, keys in ascending order per output dim
  double acc0 = 0.0;  // thread d < D accumulates dim d
  for (int c0 = 0; c0 < T; c0 += kAttnChunk) {
    const int cn = min(kAttnChunk, T - c0);
    for (int i = threadIdx.x; i < cn; i += blockDim.x) {
      const float* k = key_ptr(c0 + i, 0);
      double dot = 0.0;
      for (int e = 0; e < D; ++e) dot = fma(qs[e], (double)k[e], dot);
      w[i] = exp(dot / sqrt_d - mx) / z;
    }
    __syncthreads();
    if (threadIdx.x < D) {
      for (int i = 0; i < cn; ++i) acc0 = fma(w[i], (double)key_ptr(c0 + i, 1)[threadIdx.x], acc0);
    }
    __syncthreads();
  }
  if (threadIdx.x < D) out[(int64_t)m * ld_out + h * D + threadIdx.x] = (float)acc0;
  (void)blk_cache;
}

int attn_f64(const float* q, int64_t ld_q, int M, int n_seqs, const int32_t* cu_q, const int32_t* start_pos,
             const int32_t* block_table, int max_blocks, const float* kv, int n_layers, int layer, int B, int H,
             int Hkv, int D, float out_scale_unused, float* out, int64_t ld_out, cudaStream_t st) {
  (void)out_scale_unused;
  if (M == 0) return ALORA_OK;
  if (D > 128 || H % Hkv != 0) return ALORA_EINVAL;
  dim3 grid(M, H);
  attn_f64_kernel<<<grid, kAttnThreads, 0, st>>>(q, ld_q, n_seqs, cu_q, start_pos, block_table, max_blocks, kv,
                                                 n_layers, layer, B, H, Hkv, D, sqrt((double)D), out, ld_out);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace alora
