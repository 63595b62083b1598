// Internal launchers (host functions) shared by capi.cu and runtime.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace alora {

// One-time kernel attribute setup (shared-memory carveout, dynamic smem limits); idempotent.
void configure_kernels();
void configure_bf16_ops();
void configure_kv_ops();
void configure_attention();
void configure_gemm();

// Batch-invariant mode (AloraModelDesc.batch_invariant; set by the executor for the duration of a forward on
// its thread): GEMMs use one kernel and one K range for every row, attention one kernel and one partition
// per row, so a token's KV and logits do not depend on the step it was computed in.
inline thread_local bool g_batch_invariant = false;

enum Epi : int { kEpiStore = 0, kEpiAdd = 1, kEpiRelu = 2, kEpiSwiglu = 3, kEpiRope = 4, kEpiLoraSelect = 5 };

// ---- fp32 storage / fp64 accumulation (parity tier), parity_f64.cu
int embed_f32(const int32_t* tokens, const int32_t* positions, const float* embed, const float* pos_table, int M,
              int d, float* x, cudaStream_t st,
              const int32_t* prev_ids = nullptr);
int rmsnorm_f64(const float* x, const int32_t* rows, int n_rows, int d, const float* w, float eps, float* out,
                cudaStream_t st);
int gemm_f64(int epi, const float* A, int lda, const float* Bt, int ldb, float* C, int ldc, int M, int N, int K,
             cudaStream_t st);
int lora_f64(const float* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply, const float* down,
             const float* up_t, int n_slots, int R, const uint8_t* slot_targets, float* s_ws, int Nq, int Nkv,
             float* out, int ld_out, cudaStream_t st);
int rope_f64(float* qkv, int ld, const int32_t* positions, int M, int H, int Hkv, int D, const float* cos_t,
             const float* sin_t, cudaStream_t st);
int silu_mul_f64(const float* gu, int M, int F, float* a, cudaStream_t st);
int attn_f64(const float* q, int64_t ld_q, int M, int n_seqs, const int32_t* cu_q, const int32_t* start_pos,
             const int32_t* block_table, int max_blocks, const float* kv, int n_layers, int layer, int B, int H,
             int Hkv, int D, float unused, float* out, int64_t ld_out, cudaStream_t st);

// ---- dtype-generic, kv_write.cu / misc.cu
int kv_write(int dtype, const void* k, const void* v, int64_t ld_src, const int32_t* slot_mapping, int M,
             int kv_width, void* kv_pool, int n_layers, int layer, int B, cudaStream_t st);
int argmax_rows(const float* logits, int rows, int vocab, int32_t* out_ids, cudaStream_t st);

// ---- bf16 storage / fp32 accumulation (tensor-core tier)
int embed_bf16(const int32_t* tokens, const int32_t* positions, const __nv_bfloat16* embed, const float* pos_table,
               int M, int d, float* x, cudaStream_t st,
               const int32_t* prev_ids = nullptr);
// out_bf16[r] = bf16( rmsnorm(x[rows[r]]) * w )
int rmsnorm_bf16(const float* x, const int32_t* rows, int n_rows, int d, const float* w, float eps,
                 __nv_bfloat16* out, cudaStream_t st);
// Shrink planes: down [P][n_slots][R][K] -> s [P][M][n_slots*R]; plane t serves target bit tbit0 + t of
// slot_targets (q 0, k 1, v 2 | o 3 | gate 4, up 5 | down 6).
int lora_shrink_bf16(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                     const __nv_bfloat16* down, int n_slots, int R, const uint8_t* slot_targets, __nv_bfloat16* s,
                     cudaStream_t st, int n_planes = 3, int tbit0 = 0);
// Segmented shrink for steps with at most a few hundred delta rows per adapter: one CTA cluster per (slot,
// chunk of 64 of its rows) streams the adapter's down rows of every plane (K split over the cluster, DSMEM
// reduction in rank order), mma.sync over the slot's active rows; writes the same [n_planes][M][n_slots*R]
// layout (zeros elsewhere). R in {8, 16, 32, 64}, n_planes in {1, 2, 3}; max_rows bounds any slot's row count.
int lora_shrink_seg_bf16(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
                         const __nv_bfloat16* down, int n_slots, int R, const uint8_t* slot_targets,
                         __nv_bfloat16* s, cudaStream_t st, int n_planes, int tbit0, int max_rows);
bool lora_shrink_seg_fits(int K);  // K splits into whole 128-wide slices over the cluster
constexpr int kSegMaxRows = 128;  // the executor's switch: at most this many delta rows per adapter slot
int rope_bf16(__nv_bfloat16* qkv, int ld, const int32_t* positions, int M, int H, int Hkv, int D,
              const float* cos_t, const float* sin_t, cudaStream_t st);
int attn_bf16(const __nv_bfloat16* q, int64_t ld_q, int M, int n_seqs, const int32_t* cu_q,
              const int32_t* start_pos, const int32_t* block_table, int max_blocks, int max_q, int max_ctx,
              const __nv_bfloat16* kv, int n_layers, int layer, int B, int H, int Hkv, int D,
              __nv_bfloat16* out, int64_t ld_out, void* ws, int64_t ws_bytes, cudaStream_t st,
              int total_blocks = 0 /* > 0 enables the TMA / tcgen05 kernel */);
int64_t attn_bf16_workspace(int M, int n_seqs, int max_q, int max_ctx, int H, int Hkv, int D);
// Shared-prefix attention over an alora_plan_attention work list (on the device): query sets of requests
// that hold the same physical prefix blocks stream that prefix once; KV-partition partials (max_np > 1) are
// combined by a merge launch in partition order.
int attn_grouped(const __nv_bfloat16* q, int64_t ld_q, int M, int S, const int32_t* positions, const int32_t* row_seq,
                 const int32_t* block_table, int max_blocks, const int32_t* plan, int n_items, int n_segs, int n_sets,
                 int max_np, bool merge, const __nv_bfloat16* kv, int total_blocks, int n_layers, int layer, int B,
                 int H, int Hkv, int D, __nv_bfloat16* out, int64_t ld_out, void* ws, int64_t ws_bytes,
                 cudaStream_t st);
int64_t attn_bf16_workspace_bound(int H, int D);

// tcgen05 GEMM: C = epi(A[M,K] @ Bt[N,K]^T (+ S_t[M,Ks] @ Ut[N,Ks]^T lora part)), bf16 in, fp32 accumulate.
struct GemmLora {
  const __nv_bfloat16* s = nullptr;    // [s_planes][M][Ks] shrink output (K-major), nullptr = no LoRA
  const __nv_bfloat16* up_t = nullptr; // [N][Ks] (select mode) or [N][planes * Ks] (concat mode)
  int ks = 0;                          // n_slots * rank
  int n_q = 0, n_kv = 0;               // select mode: column ranges of the q|k|v targets (planes 0 | 1 | 2)
  int planes = 0;                      // > 1: concat mode, every tile adds all planes (SwiGLU gate|up tiles)
  int s_planes = 3;                    // planes allocated in s
  int s_rows = 0;                      // rows between planes of s (0 = M)
  const uint32_t* tile_slot_mask = nullptr;  // [ceil(M/128)] bitmask of slots present (taking the delta)
  int rank = 0;
  // kEpiRope: rotate-half RoPE in fp32 on the accumulator of columns < rope_cols (q and k heads), one rounding
  const int32_t* positions = nullptr;
  const float* rope_cos = nullptr;  // [max_seq_len, head_dim/2]
  const float* rope_sin = nullptr;
  int rope_cols = 0;
  int head_dim = 0;
  // kEpiLoraSelect (the shrink as a GEMM over all adapters' stacked down rows): column c of [M, 3*SR]
  // is (t = c / SR, slot = (c % SR) / rank); it is kept only where the row takes slot's delta and slot
  // targets t, and stored to the 3-plane shrink layout C[t][m][c % SR]; everything else is written 0.
  const int32_t* sel_row_slot = nullptr;
  const uint8_t* sel_row_apply = nullptr;
  const uint8_t* sel_targets = nullptr;
  int sel_sr = 0;
  int sel_rank = 0;
  int sel_planes = 3;  // N = sel_planes * sel_sr
  int sel_tbit0 = 0;   // target bit of plane 0 in sel_targets (q 0, k 1, v 2, o 3, gate 4, up 5, down 6)
  // fp32-store epilogue of a weight-streaming launch: per row, atomicMax of (orderable logit << 32 | ~col),
  // i.e. the greedy token with ties to the lowest id (model.py:190-195), fused into the lm_head
  unsigned long long* argmax = nullptr;
  // Paged KV scatter in the QKV epilogue (large-M tile / persistent kernels, one K split): columns
  // [kv_q, kv_q + kv_w) (K, after RoPE) and [kv_q + kv_w, kv_q + 2 kv_w) (V) of row m also go to slot
  // kv_slots[m] of the pool [NB, kv_layers, 2, kv_block, kv_w] at layer kv_layer (model.py:217-222); the GEMM
  // reports it through GemmDefer::kv_written
  __nv_bfloat16* kv_pool = nullptr;
  const int32_t* kv_slots = nullptr;
  int kv_q = 0, kv_w = 0, kv_layer = 0, kv_layers = 0, kv_block = 0;
};
// Split-K scratch: fp32 partial rows + 2 arrival counters per output tile (zeroed once, self-resetting).
constexpr int kGemmCounters = 16384;
struct GemmWs {
  void* partial = nullptr;
  int64_t partial_bytes = 0;
  int* counters = nullptr;
  int n_counters = 0;
};
int64_t gemm_bf16_workspace_bytes();
// Carves a GemmWs out of a caller buffer of gemm_bf16_workspace_bytes() bytes (counters at the end).
inline GemmWs gemm_ws_from(void* base, int64_t bytes) {
  GemmWs w;
  if (base == nullptr || bytes < gemm_bf16_workspace_bytes()) return w;
  w.n_counters = kGemmCounters;
  w.partial = base;
  w.partial_bytes = bytes - (int64_t)kGemmCounters * 4;
  w.counters = reinterpret_cast<int*>(static_cast<char*>(base) + w.partial_bytes);
  return w;
}
// Deferred split-K for weight-streaming launches (M <= 256) of the kEpiAdd / kEpiRope epilogues: when the
// plan splits K, the GEMM writes fp32 partials [splits][M][N] to `partial` (capacity bytes) and skips its
// epilogue; the consuming kernel (residual_rmsnorm_bf16 / qkv_finalize_bf16) sums the splits in order and
// applies it. splits_out reports the split count (1 = the epilogue ran inside the GEMM).
struct GemmDefer {
  float* partial = nullptr;
  int64_t capacity = 0;
  int splits_out = 1;
  bool deferred = false;  // partials [splits_out][M][N] were written and the epilogue is the consumer's job
  bool kv_written = false;  // the epilogue scattered K / V into the paged pool (GemmLora::kv_pool)
};
// ws enables split-K of the per-tile kernel (M > 256; max_splits caps it) when the output tiles cannot fill
// the 148 SMs.
int gemm_bf16(int epi, const __nv_bfloat16* A, int lda, const __nv_bfloat16* Bt, int ldb, void* C, int ldc,
              int M, int N, int K, const GemmLora* lora, cudaStream_t st, const GemmWs* ws = nullptr,
              int max_splits = 8, GemmDefer* defer = nullptr);
// x[r] (+)= sum_p partials[p][r] (split order), then out[r] = bf16(rmsnorm(x[r]) * w); rows as rmsnorm_bf16.
// zero_rows (optional, [n_rows]) is cleared: the packed argmax accumulator of the lm_head that follows.
int residual_rmsnorm_bf16(float* x, const float* partials, int nparts, int M, const int32_t* rows, int n_rows, int d,
                          const float* w, float eps, __nv_bfloat16* out, cudaStream_t st,
                          unsigned long long* zero_rows = nullptr);
// out[i] = sum_p partials[p * n + i] in split order (n % 4 == 0): the local split-K sum before a TP all-reduce.
int sum_partials_f32(const float* partials, int nparts, int64_t n, float* out, cudaStream_t st);
int argmax_unpack(const unsigned long long* packed, int rows, int32_t* out_ids, cudaStream_t st);
// qkv[m] = bf16(RoPE(sum_p partials[p][m])) on q/k heads (plain sum on v), and the row's k/v scattered into
// the paged pool (the kv_write of the step) -- the deferred epilogue of a split-K QKV projection.
int qkv_finalize_bf16(const float* partials, int nparts, int M, int Nq, int Nkv, int D, const int32_t* positions,
                      const float* cos_t, const float* sin_t, __nv_bfloat16* qkv, int ldq, const int32_t* slot_mapping,
                      __nv_bfloat16* kv_pool, int n_layers, int layer, int B, cudaStream_t st);
// Deferred epilogue of a split-K LoRA shrink (kEpiLoraSelect): s[t][m][off] = bf16(sum_p partials[p][m][t*SR+off])
// where row m takes slot (off / rank)'s delta on target t, else 0.
int lora_select_finalize_bf16(const float* partials, int nparts, int M, int SR, int rank, const int32_t* row_slot,
                              const uint8_t* row_apply, const uint8_t* slot_targets, __nv_bfloat16* s,
                              cudaStream_t st, int n_planes = 3, int tbit0 = 0);
// Fused TP all-reduce + residual + RMSNorm over peer buffers (tp_allreduce.cu).
void configure_tp();
int64_t tp_buffer_bytes(int max_tokens, int d);
float* tp_partial_slot(void* own, int max_tokens, int d, int slot);
int tp_allreduce_norm(void* const* peers, int n, int rank, int colocated, int max_tokens, int slot, int M, int d,
                      float* x, const float* w, float eps, __nv_bfloat16* h, cudaStream_t st);
int lora_tile_masks(const int32_t* row_slot, const uint8_t* row_apply, int M, uint32_t* masks, cudaStream_t st);

}  // namespace alora
