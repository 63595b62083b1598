/*
 * libalora_sm100a.so — C ABI of the B200 (sm_100a) aLoRA hot path.
 *
 * Drop-in boundary for /root/reference/pkg/src/aloraserve (pure Python/numpy).
 * The reference has no FFI; every entry point below replaces one Python
 * function of its hot path (file:line into /root/reference/pkg/src/aloraserve):
 *
 *   alora_hash_block / alora_hash_chain  <- kv_cache.py:41-69 hash_block, and the chain
 *                                           walks of kv_cache.py:166-182, 253-260
 *   alora_qkv_proj                       <- model.py:117-146 project_qkv_masked
 *   alora_kv_write                       <- model.py:217-222 _write_kv
 *   alora_paged_prefill_attn             <- model.py:149-187 paged_attention
 *   alora_model_* (native executor)      <- model.py:233-272 Model.forward_step /
 *                                           _forward_one, batched over all spans of a step
 *   alora_argmax                         <- model.py:190-195 greedy_next_token
 *
 * Conventions
 *   - Plain pointers and sizes only. Device pointers are CUDA global memory owned
 *     by the caller; no entry point allocates device memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Return 0 (ALORA_OK) or a negative status; the Python shim maps
 *     ALORA_EINVAL to ValueError and the rest to RuntimeError (the reference
 *     raises ValueError for bad shapes, model.py:134-135, 162-163, 250-258).
 *   - dtype: ALORA_F32 = fp32 storage with fp64 accumulation (the reference's
 *     numerics, model.py:95-98); ALORA_BF16 = bf16 storage, fp32 accumulation
 *     on tcgen05 tensor cores.
 *   - KV pool layout is the reference's block-major [NB, L, 2, B, kv_width]
 *     (kv_cache.py:143); a slot is block_id * B + (pos % B).
 */
#ifndef ALORA_SM100A_H
#define ALORA_SM100A_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALORA_OK 0
#define ALORA_EINVAL (-1)
#define ALORA_ECUDA (-2)
#define ALORA_EUNSUPPORTED (-3)
#define ALORA_ENOSPC (-4) /* block pool: not enough free blocks (PoolExhaustedError) */
#define ALORA_ESTATE (-5) /* block pool: an invariant the call relies on does not hold */

#define ALORA_F32 0
#define ALORA_BF16 1

#define ALORA_ARCH_REF 0   /* aloraserve model.py: sinusoidal pos, no-gain RMSNorm, MHA, ReLU 4x MLP */
#define ALORA_ARCH_LLAMA 1 /* RoPE, GQA, SwiGLU, weighted RMSNorm, tied lm_head */

/* ---------------------------------------------------------------- host ---- */

/* Version string of the build (architecture, nvcc). */
const char* alora_version(void);

/* One block digest: blake2b-128 over the kv_cache.py:41-69 encoding.
 * parent: 16 bytes or NULL (first block). tokens: block_size u32 ids. */
int alora_hash_block(const uint8_t* parent, const uint32_t* tokens, int32_t block_size,
                     const char* key, int32_t key_len, uint8_t* out_digest);

/* Chain of n_blocks digests; block i hashes tokens[i*B, (i+1)*B) with key
 * key_blob[key_off[i], key_off[i+1]) and parent = digest i-1 (or `parent`
 * for i = 0, NULL = chain start). out_digests: n_blocks * 16 bytes. */
int alora_hash_chain(const uint8_t* parent, const uint32_t* tokens, int64_t n_blocks,
                     int32_t block_size, const char* key_blob, const int64_t* key_off,
                     uint8_t* out_digests);

/* n_chains independent alora_hash_chain calls (arguments per chain, parents
 * may be NULL = every chain starts fresh), spread over up to n_threads host
 * threads. Replaces the per-request chain walks of one scheduler step
 * (kv_cache.py:166-182 called from scheduler.py admission, 253-260 at retire). */
int alora_hash_chains(int32_t n_chains, const uint8_t* const* parents, const uint32_t* const* tokens,
                      const int64_t* n_blocks, int32_t block_size, const char* const* key_blobs,
                      const int64_t* const* key_offs, uint8_t* const* out_digests, int32_t n_threads);

/* The admission lookup chains of n_req requests in one call: request r's prompt
 * (int64 token ids, validated < 2^32) gives n_blocks[r] digests; blocks
 * [0, n_base[r]) carry the base key "" and the rest keys[r] (compute_block_keys,
 * kv_cache.py:72-96). Digests land back to back in out_digests (sum n_blocks * 16). */
int alora_hash_requests(int32_t n_req, const int64_t* const* tokens, const int64_t* n_blocks, const int64_t* n_base,
                        const char* const* keys, const int32_t* key_lens, int32_t block_size,
                        uint8_t* out_digests, int32_t n_threads);

/* ------------------------------------------------------- block manager ---- */
/* Per-block state of the paged KV pool and its digest index (kv_cache.py:126-326
 * BlockPool; the per-request maps stay with the caller). Digests are 16 bytes. */
void* alora_pool_create(int32_t n_blocks, int32_t block_size);
void alora_pool_destroy(void* pool);
/* Host pointers to the pool's own arrays: ref_count[nb], fill[nb], has_hash[nb], hash[nb*16]. */
int alora_pool_views(void* pool, int32_t** ref, int32_t** fill, uint8_t** has_hash, uint8_t** hash);
int32_t alora_pool_num_free(void* pool);
/* find_cached_prefix walk (kv_cache.py:154-183): pins and returns the hit count (>= 0). */
int64_t alora_pool_lookup(void* pool, const uint8_t* digests, int64_t n, int32_t* out_ids);
/* allocate (kv_cache.py:192-218): ALORA_ENOSPC and no change when n > free blocks. */
int alora_pool_allocate(void* pool, int64_t n, int32_t* out_ids);
/* release of a request's blocks, tail first (kv_cache.py:258-270). */
int alora_pool_release(void* pool, const int32_t* ids, int64_t n);
/* commit: digest i -> block ids[i] (full blocks only), index overwritten (kv_cache.py:250-257). */
int alora_pool_publish(void* pool, const int32_t* ids, const uint8_t* digests, int64_t n);
/* set_fill (kv_cache.py:220-223) for the n blocks ids[0..n) of a request that hold its
 * block positions first .. first+n-1. */
int alora_pool_set_fill(void* pool, const int32_t* ids, int64_t n, int64_t first, int64_t n_tokens);
/* Free blocks in eviction order (least recently released first); returns the count. */
int64_t alora_pool_free_list(void* pool, int32_t* out, int64_t cap);
/* Block id indexed under `digest`, or -1. */
int32_t alora_pool_index_get(void* pool, const uint8_t* digest);
/* Index entries (cap <= 0: just the count). */
int64_t alora_pool_index_dump(void* pool, uint8_t* digests, int32_t* ids, int64_t cap);

/* ------------------------------------------------------ native admission ---- */
/* The engine's scheduler and per-request block tables on top of a block manager (csrc/sched_core.cpp):
 * scheduler.py:139-265 (intake, schedule_step, prefix lookup, block allocation, on_span_done) and the
 * per-request half of kv_cache.py:154-271 (lookup walk, set_fill, commit_and_free, release). */
void* alora_sched_create(void* pool, int32_t block_size, int32_t token_budget, int32_t max_batch,
                         int32_t chunked, int32_t prefix_caching, int32_t hash_threads);
void alora_sched_destroy(void* sched);
/* Thread-safe intake (ticket order = call order). mode: 0 base, 1 standard LoRA, 2 activated (inv_start
 * = invocation start). key = the adapter id (block-hash extra key). Returns the request handle (>= 0). */
int32_t alora_sched_submit(void* sched, const int64_t* prompt, int64_t n, int32_t max_new, int32_t mode,
                           const char* key, int32_t key_len, int64_t inv_start);
int32_t alora_sched_has_work(void* sched);
/* One schedule_step. spans[i] = {handle, start, end, kind} (kind: 0 prefill, 1 decode, +256 = the request's
 * first scheduled work); failed = requests failed this step (pool exhausted during decode); looked = requests
 * whose prefix lookup ran this step; counts = {n_spans, n_failed, n_looked, budget_used}; blocks/block_off =
 * each span's block table (the request's block ids in position order), concatenated. */
int alora_sched_step(void* sched, int32_t* spans, int32_t span_cap, int32_t* failed, int32_t failed_cap,
                     int32_t* looked, int32_t looked_cap, int32_t* counts, int32_t* blocks, int64_t block_cap,
                     int64_t* block_off);
/* The step's spans are done (on_span_done + set_fill for each): emitted token (if has_emitted; a
 * placeholder is fixed later with alora_sched_set_token). flags_out: bit 0 prompt completed (-> decoding),
 * bit 1 finished. */
int alora_sched_step_done(void* sched, int32_t n, const int32_t* handles, const int32_t* starts,
                          const int32_t* ends, const int64_t* emitted, const uint8_t* has_emitted,
                          uint8_t* flags_out);
int alora_sched_set_token(void* sched, int32_t handle, int64_t gen_index, int64_t token);
/* Retire a finished request: commit_and_free (publish its full blocks, release tail first) or, for a
 * failed request, release. */
int alora_sched_retire(void* sched, int32_t handle);
/* {processed, hit tokens, computed tokens, generated, state, blocks held, blocks reused, failed} */
int alora_sched_info(void* sched, int32_t handle, int64_t* out8);
int64_t alora_sched_blocks(void* sched, int32_t handle, int32_t* out, int64_t cap);
int64_t alora_sched_owned_total(void* sched);

/* ------------------------------------------------------ hot-path kernels ---- */

/* Masked multi-adapter aLoRA Q/K/V projection (model.py:117-146).
 *   x          [M, K] (dtype), row stride K
 *   w_qkv_t    [Nq + 2*Nkv, K] (dtype): Wq|Wk|Wv transposed (K contiguous)
 *   row_slot   [M] int32 adapter slot of the row, -1 = no adapter
 *   row_apply  [M] uint8 1 = add the delta (activated: pos >= inv_start; standard: all rows)
 *   lora_down  [3, n_slots, rank, K] (dtype) zero padded beyond each adapter's rank
 *   lora_up_t  [Nq + 2*Nkv, n_slots*rank] (dtype): up_t^T for the target owning the column
 *   slot_targets [n_slots] uint8 bit0 q, bit1 k, bit2 v
 *   s_ws       workspace, >= 3*M*n_slots*rank elements (dtype) (shrink output)
 *   out        [M, ld_out] (dtype): q at col 0, k at Nq, v at Nq+Nkv
 * Rows with row_apply = 0 (or slot -1, or untargeted projections) are exactly
 * the base product — row select, not blend (model.py:145). */
int alora_qkv_proj(int32_t dtype, const void* x, int32_t M, int32_t K, const void* w_qkv_t,
                   int32_t Nq, int32_t Nkv, const int32_t* row_slot, const uint8_t* row_apply,
                   const void* lora_down, const void* lora_up_t, int32_t n_slots, int32_t rank,
                   const uint8_t* slot_targets, void* s_ws, void* out, int32_t ld_out, void* stream);

/* Paged KV scatter (model.py:217-222): for m < M with slot_mapping[m] >= 0,
 * kv[blk, layer, 0, row, :] = k[m, :], kv[blk, layer, 1, row, :] = v[m, :],
 * blk = slot / block_size, row = slot % block_size. Vectorised 16-byte stores. */
int alora_kv_write(int32_t dtype, const void* k, const void* v, int64_t ld_src,
                   const int32_t* slot_mapping, int32_t M, int32_t kv_width, void* kv_pool,
                   int32_t n_layers, int32_t layer, int32_t block_size, void* stream);

/* Paged causal prefill attention over the cache (model.py:149-187, GQA):
 * sequence s owns query rows [cu_q[s], cu_q[s+1]) at absolute positions
 * start_pos[s] + i and attends keys [0, start_pos[s] + i] read through
 * block_table[s, :] (their K/V must already be in the pool: alora_kv_write).
 *   q [n_rows, ld_q] (dtype) heads contiguous, out [n_rows, ld_out] (dtype); n_rows == cu_q[n_seqs].
 * Scale is 1/sqrt(head_dim) as in model.py:179. Keys are visited in a fixed
 * order of absolute positions, so results do not depend on chunking. */
int alora_paged_prefill_attn(int32_t dtype, const void* q, int64_t ld_q, int32_t n_rows,
                             int32_t n_seqs, const int32_t* cu_q, const int32_t* start_pos,
                             const int32_t* block_table, int32_t max_blocks, int32_t max_q,
                             int32_t max_ctx, const void* kv_pool, int32_t total_blocks,
                             int32_t n_layers, int32_t layer, int32_t block_size, int32_t n_heads,
                             int32_t n_kv_heads, int32_t head_dim, void* out, int64_t ld_out,
                             void* workspace, int64_t workspace_bytes, void* stream);

/* Device workspace alora_paged_prefill_attn needs (bf16 split-KV partials + merge counters at
 * the end of the buffer; 0 for fp32). Zero-fill it once: the counters reset themselves. */
int64_t alora_attn_workspace_bytes(int32_t dtype, int32_t n_rows, int32_t n_seqs, int32_t max_q,
                                   int32_t max_ctx, int32_t n_heads, int32_t n_kv_heads,
                                   int32_t head_dim);

/* Host planner of the shared-prefix attention (replaces the per-span loop of model.py:243 around
 * paged_attention, model.py:149-187, for steps whose requests hold the same physical prefix blocks:
 * the base-aligned reuse of kv_cache.py:72-96). HOST arrays: cu_q [S+1], start_pos [S], block_table
 * [S, max_blocks]. flags: bit 0 group spans by shared leading blocks, bit 1 never split the keys.
 * partial_cap_bytes bounds the split-KV partials. Writes the int32 plan into out (layout in
 * csrc/attn_plan.cpp: header [n_items, n_segs, n_sets, max_parts, merge_rows, unique kv tokens,
 * total tiles, 0] then items, segments, sets, set rows, per-span partition counts) and returns its
 * length, or -(length needed) when out_cap is too small, or ALORA_EINVAL. */
int64_t alora_plan_attention(int32_t n_seqs, const int32_t* cu_q, const int32_t* start_pos,
                             const int32_t* block_table, int32_t max_blocks, int32_t block_size,
                             int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, int32_t flags,
                             int64_t partial_cap_bytes, int32_t* out, int64_t out_cap);

/* Split-KV partial bytes the executor's attention workspace holds (the partial_cap_bytes to plan with). */
int64_t alora_attn_partial_capacity(int32_t n_heads, int32_t head_dim);

/* Paged causal attention (model.py:149-187) through a plan from alora_plan_attention, uploaded to
 * the device (bf16 tier): row m at absolute position positions[m] of span row_seq[m] attends keys
 * [0, positions[m]] of its span; requests grouped by the plan read their shared prefix once.
 * Results equal alora_paged_prefill_attn's up to fp32 summation order. Workspace: the split-KV
 * partials, max_parts * n_rows * n_heads * (head_dim + 2) * 4 bytes when max_parts > 1. */
int alora_paged_prefix_attn(const void* q, int64_t ld_q, int32_t n_rows, int32_t n_seqs,
                            const int32_t* positions, const int32_t* row_seq, const int32_t* block_table,
                            int32_t max_blocks, const int32_t* plan, int32_t n_items, int32_t n_segs,
                            int32_t n_sets, int32_t max_parts, const void* kv_pool, int32_t total_blocks,
                            int32_t n_layers, int32_t layer, int32_t block_size, int32_t n_heads,
                            int32_t n_kv_heads, int32_t head_dim, void* out, int64_t ld_out,
                            void* workspace, int64_t workspace_bytes, void* stream);

/* Dense bf16 GEMM on tcgen05 (the engine behind alora_qkv_proj and the O/MLP/lm_head
 * projections of alora_model_forward): C = epi(A[M,K] . Bt[N,K]^T), fp32 accumulate.
 * epi: 0 store bf16, 1 C(fp32) += acc, 2 relu -> bf16, 3 SwiGLU of 64-interleaved
 * gate|up column blocks -> bf16 [M, N/2], 16 store fp32.
 * workspace (optional; zero-filled once, >= alora_gemm_workspace_bytes()) enables split-K
 * when the output tiles cannot fill the 148 SMs: the splits of a tile are co-resident
 * (cooperative launch), publish fp32 partials to L2 and each reduces a slice of rows in
 * split order (deterministic for a given split count). */
int alora_gemm_bf16(int32_t epi, const void* A, int32_t lda, const void* Bt, int32_t ldb, void* C,
                    int32_t ldc, int32_t M, int32_t N, int32_t K, void* workspace,
                    int64_t workspace_bytes, void* stream);
int64_t alora_gemm_workspace_bytes(void);

/* Greedy next token per row of logits [rows, V] fp32: argmax, ties -> lowest id (model.py:190-195). */
int alora_argmax(const float* logits, int32_t rows, int32_t vocab, int32_t* out_ids, void* stream);

/* ------------------------------------------------------ native executor ---- */

/* Tensor-parallel all-reduce hook (sum, in place) of `count` fp32 values at device pointer `buf`,
 * stream-ordered on `stream`. alora_model_forward calls it twice per layer when tp_size > 1: on the
 * row-parallel O-projection output and on the MLP-down output, before the residual add + RMSNorm
 * (reference model.py:269-271, sharded as in SURVEY.md §8(e)). Returns 0 on success. */
typedef int32_t (*alora_allreduce_fn)(void* ctx, float* buf, int64_t count, void* stream);

/* Model description: shapes plus device pointers (caller-owned). Per-layer
 * pointers are arrays of n_layers device pointers living in HOST memory. */
typedef struct AloraModelDesc {
  int32_t arch, dtype;
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn_dim, vocab, max_seq_len;
  float rms_eps, rope_theta;
  int32_t max_tokens;            /* workspace capacity in rows per step */
  int32_t max_seqs;              /* workspace capacity in spans per step */
  /* weights (dtype), transposed to [out, in] */
  const void* embed;             /* [V, d] */
  const void* unembed_t;         /* [V, d] (ref: unembed^T; llama: == embed when tied) */
  const float* pos_table;        /* ref: [max_seq_len, d] fp32 sinusoidal */
  const float* rope_cos;         /* llama: [max_seq_len, head_dim/2] fp32 */
  const float* rope_sin;
  const float* final_norm;       /* llama: [d] fp32, ref: NULL */
  const void* const* w_qkv_t;    /* [L] -> [Nq+2Nkv, d] */
  const void* const* w_o_t;      /* [L] -> [d, Nq] */
  const void* const* w_in_t;     /* [L] -> ref [4d, d] (ReLU) / llama [2F, d] gate|up interleaved per 64 */
  const void* const* w_out_t;    /* [L] -> [d, F] */
  const float* const* attn_norm; /* [L] -> [d] fp32 or NULL */
  const float* const* mlp_norm;  /* [L] -> [d] fp32 or NULL */
  /* adapters */
  int32_t n_slots, lora_rank;
  const void* const* lora_down;  /* [L] -> [3, n_slots, rank, d] */
  const void* const* lora_up_t;  /* [L] -> [Nq+2Nkv, n_slots*rank] */
  const uint8_t* slot_targets;   /* [n_slots] device */
  /* paged KV pool */
  void* kv_pool;                 /* [NB, L, 2, B, Hkv*D] (dtype) */
  int32_t total_blocks, block_size;
  /* workspace (caller-owned device memory, >= alora_model_workspace_bytes) */
  void* workspace;
  int64_t workspace_bytes;
  /* tensor parallelism (bf16 tier): this rank holds n_heads / n_kv_heads / ffn_dim of a tp_size-way
   * sharded model (column-parallel q|k|v and gate|up, row-parallel o and down); 0 or 1 = unsharded */
  int32_t tp_size;
  void* tp_ctx;
  alora_allreduce_fn tp_allreduce;
  /* aLoRA on the O / MLP projections: an extension of the reference, whose adapters target q/k/v only
   * (adapters.py:26, 61-63). bf16 tier. NULL arrays = no adapter targets that projection. The delta is
   * the same masked base + (x . down) . up of model.py:141-145, fused as extra K of the O / gate|up /
   * down GEMM. slot_targets bits: q 0, k 1, v 2, o 3, gate 4, up 5, down 6. */
  const void* const* lora_o_down;    /* [L] -> [1, n_slots, rank, Nq] */
  const void* const* lora_o_up_t;    /* [L] -> [d, n_slots*rank] */
  const void* const* lora_in_down;   /* [L] -> [P, n_slots, rank, d]; P = 2 (llama: gate, up) or 1 (ref: up) */
  const void* const* lora_in_up_t;   /* [L] -> [rows of w_in_t, P*n_slots*rank], plane p in columns p*n_slots*rank.. */
  const void* const* lora_out_down;  /* [L] -> [1, n_slots, rank, F] */
  const void* const* lora_out_up_t;  /* [L] -> [d, n_slots*rank] */
  /* fused tensor-parallel all-reduce (tp_size > 1 and tp_peers != NULL; replaces the tp_allreduce hook):
   * tp_peers[r] = rank r's symmetric buffer of alora_tp_buffer_bytes(max_tokens, d_model) bytes, zeroed
   * before first use, mapped into this process (CUDA IPC: alora_ipc_get_handle / alora_ipc_open, or the
   * same device pointers when the ranks are threads on one GPU: tp_colocated = 1). The O-projection and
   * MLP-down write their fp32 partials into this rank's buffer and one kernel per rank sums every rank's
   * partial in rank order, adds the residual and applies the next RMSNorm (graph-capturable). */
  int32_t tp_rank;
  void* const* tp_peers;
  int32_t tp_colocated;
  /* batch-invariant numerics (bf16 tier): every row of every step goes through the same kernels with the
   * same reduction order -- one weight-streaming GEMM kernel and K range (no M-dependent split-K or
   * swap-AB decode GEMM), the segmented (or per-row) LoRA shrink, one tcgen05 attention kernel with a single
   * KV partition per row -- so a token's KV and logits are bitwise independent of batching, chunking and
   * decode vs prefill (the reference's property, model.py:95-98; tests/test_model.py:167-202). Slower. */
  int32_t batch_invariant;
} AloraModelDesc;

/* One engine step: all spans packed back to back (varlen). Device arrays. */
typedef struct AloraStepDesc {
  int32_t n_tokens, n_seqs, max_blocks, max_q, max_ctx;
  const int32_t* tokens;        /* [M]; a negative entry t is next_ids[-t-1] of the PREVIOUS forward on this
                                   buffer (a decode step launched before the host read that step's output) */
  const int32_t* positions;     /* [M] absolute */
  const int32_t* slot_mapping;  /* [M] */
  const int32_t* row_slot;      /* [M] adapter slot or -1 */
  const uint8_t* row_apply;     /* [M] */
  const int32_t* cu_q;          /* [S+1] */
  const int32_t* start_pos;     /* [S] */
  const int32_t* block_table;   /* [S, max_blocks] */
  const int32_t* last_row;      /* [S] row whose logits are produced */
  float* logits;                /* [S, V] fp32 out */
  int32_t* next_ids;            /* [S] argmax out (read first for negative tokens, written last) */
  /* host-side shape summary, used only for the profiler's algorithmic bytes/flops */
  double attn_kv_tokens;        /* distinct keys read (a shared prefix counted once) */
  double attn_qk_pairs;         /* sum over spans of n * (start_pos + (n + 1) / 2) */
  /* optional shared-prefix attention plan (alora_plan_attention output, on the device); NULL = per span */
  const int32_t* row_seq;       /* [M] span of each row */
  const int32_t* attn_plan;
  int32_t attn_items, attn_segs, attn_sets, attn_max_parts;
  /* most rows taking one adapter's delta in this step (host count): few -> the segmented LoRA shrink */
  int32_t lora_rows_max;
} AloraStepDesc;

/* Tensor-parallel peer buffers: bytes of one rank's symmetric buffer, device allocation (zeroed, a whole
 * cudaMalloc allocation so that its IPC handle covers it), and the CUDA IPC handle exchange (64-byte
 * handles; alora_ipc_open maps a peer's buffer with lazy peer access over NVLink). */
int64_t alora_tp_buffer_bytes(int32_t max_tokens, int32_t d_model);
/* Byte offset of partial slot `slot` (0 | 1) in a rank's buffer: [max_tokens, d_model] fp32 rows. */
int64_t alora_tp_partial_offset(int32_t max_tokens, int32_t d_model, int32_t slot);
int alora_device_alloc(int64_t bytes, void** out);
int alora_device_free(void* p);
int alora_ipc_get_handle(void* dev_ptr, uint8_t* out64);
int alora_ipc_open(const uint8_t* handle64, void** out_ptr);
int alora_ipc_close(void* ptr);
/* The fused all-reduce + residual + RMSNorm on its own (what alora_model_forward launches after the
 * row-parallel O-projection / MLP-down): x[M, d] += sum over ranks (rank order) of the partial in slot
 * `slot` of every peer buffer; h = bf16(rmsnorm(x) * w) unless h is NULL. Every rank must make the same
 * sequence of calls. */
int alora_tp_allreduce_norm(void* const* peers, int32_t n_ranks, int32_t rank, int32_t colocated,
                            int32_t max_tokens, int32_t slot, int32_t M, int32_t d, float* x, const float* w,
                            float eps, void* h, void* stream);

int64_t alora_model_workspace_bytes(const AloraModelDesc* desc);
int alora_model_create(const AloraModelDesc* desc, void** out_handle);
int alora_model_destroy(void* handle);
/* Run every layer for one packed step: embed -> L x [norm, masked QKV (+LoRA),
 * KV write, paged attention, O-proj, MLP] -> last-row logits -> argmax. */
int alora_model_forward(void* handle, const AloraStepDesc* step, void* stream);
/* alora_model_forward captured as a CUDA graph (with its programmatic-launch edges) and replayed: the first
 * call for a step shape (n_tokens, n_seqs, max_blocks, max_q, max_ctx) captures on `stream` (which must not
 * be the legacy default stream), later calls with the same shape AND the same staged step buffers replay it.
 * Kernels read every per-step length from the device arrays, so one capture serves all decode steps whose
 * padded block-table width and context bound fall in the same bucket. Falls back to alora_model_forward
 * while profiling. */
int alora_model_forward_graph(void* handle, const AloraStepDesc* step, void* stream);
/* Capture (if not cached yet) the graph alora_model_forward_graph would replay for this step, without
 * launching it: tensor-parallel ranks sharing one GPU capture before any rank starts spinning in the fused
 * all-reduce (graph instantiation may wait for the device). */
int alora_model_graph_prepare(void* handle, const AloraStepDesc* step, void* stream);
/* Count of kernel launches issued by the last alora_model_forward. */
int32_t alora_model_last_launches(void* handle);

/* Per-kernel profiling with CUDA events on the launch stream: while enabled,
 * every launch of alora_model_forward is bracketed by events and tagged with
 * its algorithmic bytes and flops. profile_read (after a stream sync)
 * aggregates by kernel kind: names (max_kinds x 32 chars), total ms, launch
 * counts, bytes and flops; returns the number of kinds. */
int alora_model_set_profiling(void* handle, int32_t enable);
int alora_model_profile_read(void* handle, int32_t max_kinds, char* names, float* ms, int32_t* counts,
                             double* bytes, double* flops);
/* The kernels behind the profiled launches: one text line per distinct (kind, kernel, grid),
 * "kind<TAB>demangled kernel name<TAB>grid CTAs<TAB>launches\n", NUL-terminated into buf (cap bytes).
 * Returns the size the full text needs (call with buf = NULL to size it). Tests use it to assert
 * which kernel variant (tile width, split count, decode/prefill attention) served a step. */
int64_t alora_model_profile_kernels(void* handle, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* ALORA_SM100A_H */
