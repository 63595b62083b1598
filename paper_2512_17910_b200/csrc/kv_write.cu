// Paged KV scatter (model.py:217-222) and greedy argmax (model.py:190-195).
//
// kv_write: row m of k/v goes to kv[blk, layer, 0|1, row, :] with
// blk = slot / B, row = slot % B, slot = slot_mapping[m] (< 0 = skip). Each
// destination row is a contiguous kv_width run, so one CTA handles several
// rows and moves them in 16-byte vectors: coalesced, one read + one write per
// byte (algorithmic traffic 2 * M * kv_width * elem * 2 bytes).

#include "common.cuh"
#include "kernels.h"

namespace alora {

constexpr int kKvThreads = 256;

__global__ void __launch_bounds__(kKvThreads) kv_write_vec_kernel(
    const uint8_t* __restrict__ k, const uint8_t* __restrict__ v, int64_t ld_src_bytes,
    const int32_t* __restrict__ slot_mapping, int M, int row_bytes, uint8_t* __restrict__ pool, int n_layers,
    int layer, int B, int rows_per_cta) {
  pdl_wait();
  pdl_trigger();
  const int vec_per_row = row_bytes / 16;
  const int per_row = 2 * vec_per_row;  // K then V
  const int m0 = blockIdx.x * rows_per_cta;
  const int total = rows_per_cta * per_row;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int m = m0 + i / per_row;
    if (m >= M) break;
    const int slot = slot_mapping[m];
    if (slot < 0) continue;
    const int r = i % per_row;
    const int sel = r / vec_per_row, c = r % vec_per_row;
    const int64_t blk = slot / B, row = slot % B;
    const uint8_t* src = (sel == 0 ? k : v) + (int64_t)m * ld_src_bytes + (int64_t)c * 16;
    uint8_t* dst = pool + ((((blk * n_layers + layer) * 2 + sel) * B + row) * (int64_t)row_bytes) + (int64_t)c * 16;
    const int4 val = __ldg(reinterpret_cast<const int4*>(src));
    __stcs(reinterpret_cast<int4*>(dst), val);  // streaming store: the pool is not re-read by this step's writer
  }
}

__global__ void kv_write_scalar_kernel(const uint8_t* __restrict__ k, const uint8_t* __restrict__ v,
                                       int64_t ld_src_bytes, const int32_t* __restrict__ slot_mapping,
                                       int row_bytes, int elem, uint8_t* __restrict__ pool, int n_layers, int layer,
                                       int B) {
  const int m = blockIdx.x;
  const int slot = slot_mapping[m];
  if (slot < 0) return;
  const int64_t blk = slot / B, row = slot % B;
  for (int i = threadIdx.x; i < 2 * row_bytes / elem; i += blockDim.x) {
    const int sel = i / (row_bytes / elem), c = i % (row_bytes / elem);
    const uint8_t* src = (sel == 0 ? k : v) + (int64_t)m * ld_src_bytes + (int64_t)c * elem;
    uint8_t* dst = pool + ((((blk * n_layers + layer) * 2 + sel) * B + row) * (int64_t)row_bytes) + (int64_t)c * elem;
    for (int b = 0; b < elem; ++b) dst[b] = src[b];
  }
}

int kv_write(int dtype, const void* k, const void* v, int64_t ld_src, const int32_t* slot_mapping, int M,
             int kv_width, void* kv_pool, int n_layers, int layer, int B, cudaStream_t st) {
  if (M == 0) return ALORA_OK;
  if (M < 0 || kv_width <= 0 || B <= 0 || layer < 0 || layer >= n_layers) return ALORA_EINVAL;
  const int elem = dtype == ALORA_BF16 ? 2 : 4;
  const int row_bytes = kv_width * elem;
  const int64_t ld_bytes = ld_src * elem;
  const bool aligned = (row_bytes % 16 == 0) && (ld_bytes % 16 == 0) &&
                       ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                         reinterpret_cast<uintptr_t>(kv_pool)) % 16 == 0);
  if (aligned) {
    const int per_row = 2 * row_bytes / 16;
    int rows_per_cta = kKvThreads / per_row;
    if (rows_per_cta < 1) rows_per_cta = 1;
    const int grid = (M + rows_per_cta - 1) / rows_per_cta;
    ALORA_CUDA_CHECK(launch_pdl(kv_write_vec_kernel, dim3(grid), dim3(kKvThreads), 0, st, nullptr, 0,
                                static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v), ld_bytes,
                                slot_mapping, M, row_bytes, static_cast<uint8_t*>(kv_pool), n_layers, layer, B,
                                rows_per_cta));
  } else {
    kv_write_scalar_kernel<<<M, 128, 0, st>>>(static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v),
                                              ld_bytes, slot_mapping, row_bytes, elem,
                                              static_cast<uint8_t*>(kv_pool), n_layers, layer, B);
  }
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

// ---------------------------------------------------------------- argmax ---
// Ties -> lowest index: compare (value, -index) lexicographically.
__global__ void argmax_kernel(const float* __restrict__ logits, int vocab, int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + (int64_t)blockIdx.x * vocab;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float x = row[i];
    if (x > best || (x == best && i < bi)) { best = x; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sv[wid] = best; si[wid] = bi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}

void configure_kv_ops() {
  prefer_max_smem(kv_write_vec_kernel);
  prefer_max_smem(kv_write_scalar_kernel);
  prefer_max_smem(argmax_kernel);
}

// next_ids[r] from the packed (orderable value, ~index) maxima the lm_head epilogue accumulated.
__global__ void argmax_unpack_kernel(const unsigned long long* __restrict__ packed, int rows, int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) out[r] = (int32_t)(0xFFFFFFFFu - (uint32_t)(packed[r] & 0xFFFFFFFFull));
}

int argmax_unpack(const unsigned long long* packed, int rows, int32_t* out_ids, cudaStream_t st) {
  if (rows <= 0) return ALORA_OK;
  ALORA_CUDA_CHECK(launch_pdl(argmax_unpack_kernel, dim3((rows + 127) / 128), dim3(128), 0, st, nullptr, 0, packed,
                              rows, out_ids));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

int argmax_rows(const float* logits, int rows, int vocab, int32_t* out_ids, cudaStream_t st) {
  if (rows == 0) return ALORA_OK;
  if (vocab <= 0) return ALORA_EINVAL;
  ALORA_CUDA_CHECK(launch_pdl(argmax_kernel, dim3(rows), dim3(1024), 0, st, nullptr, 0, logits, vocab, out_ids));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace alora
