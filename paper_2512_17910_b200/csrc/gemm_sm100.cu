// tcgen05 / TMEM / TMA GEMM for the bf16 tier, with the aLoRA delta fused into the accumulator.
//
//   C[M, N] = epi( A[M, K] . Bt[N, K]^T  +  S_t[M, Ks] . Ut[N, Ks]^T )
//
// The second product is the LoRA expand (model.py:141: adapted = base + (x@down)@up):
// S_t is the shrink output of projection t (q|k|v, chosen by the N tile), laid
// out [slot*rank + j] so that a row only has non-zeros in its own adapter's
// slot, and only if the row takes the delta (pos >= inv_start). Rows before
// the invocation therefore add exact zeros to the fp32 accumulator and come out
// bit-identical to a base-only GEMM — the row-select of model.py:145 without a
// second pass. K-blocks of the LoRA range whose adapters are absent from the
// 128-row tile (per-tile slot mask) are skipped entirely.
//
// Structure (one 128 x BN output tile per CTA and K split, 192 threads):
//   warp 0      TMA producer: A/B (or S/U) 64-wide K slabs -> smem ring (SW128)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 cols -> fused epilogue -> global
// mbarrier ring: full[s] (TMA tx bytes) / empty[s] (tcgen05.commit), tmem_full.
//
// Kernels by step shape (gemm_bf16 at the end of this file picks one):
//   M <= 32    gemm_dec_kernel: swap-AB (128 weight rows as the MMA's M, the tokens as N = 16 / 32)
//   M <= 256   gemm_ws_kernel: weight streaming, one CTA per (N tile, K split) covering every token row;
//              K splits are deferred: fp32 partials are TMA-stored and summed in split order by the consuming
//              kernel (residual RMSNorm / QKV finalize), so every SM streams a disjoint weight slab once
//   M > 256    gemm_bf16_persist_kernel (more tiles than SMs: one CTA per SM, two TMEM accumulators, grouped
//              tile order) or gemm_bf16_kernel (one tile per CTA; co-resident split-K through global partials
//              and arrival counters when the tiles cannot fill half the SMs); 128 x 128 or 128 x 256 tiles
// Epilogues: bf16 store, fp32 store, residual add (C += acc), ReLU, SwiGLU of
// 64-interleaved gate|up blocks, rotate-half RoPE on q/k columns, and the
// LoRA-shrink row/slot select.

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace alora {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 192;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kMaxSplits = 8;  // portable cluster size

struct GemmArgs {
  void* C;
  int ldc;
  int M, N, K;
  int epi;        // Epi | 16 => fp32 output for kEpiStore
  int ks;         // LoRA K (n_slots * rank), 0 = none
  int rank;
  int n_q, n_kv;  // q | k | v column ranges (select mode)
  int lora_planes; // > 1: concat mode, every tile reads all planes (up_t columns [p*ks, (p+1)*ks) for plane p)
  const uint32_t* tile_slot_mask;
  const int32_t* positions;  // kEpiRope
  const float* rope_cos;
  const float* rope_sin;
  int rope_cols, head_dim;
  const int32_t* sel_row_slot;  // kEpiLoraSelect
  const uint8_t* sel_row_apply;
  const uint8_t* sel_targets;
  int sel_sr, sel_rank;
  int sel_tbit0;  // target bit of plane 0 in sel_targets
  unsigned long long* argmax;  // fused greedy argmax of the fp32-store epilogue (ws kernel, S == 1)
  __nv_bfloat16* kv_pool;      // paged KV scatter of the K / V columns (GemmLora::kv_pool)
  const int32_t* kv_slots;
  int kv_q, kv_w, kv_layer, kv_layers, kv_block;
  int splits;                 // K splits (blockIdx.z); grid <= SM count, cooperative launch
  float* partial;             // [splits][m_tiles*128][N] fp32 when splits > 1
  int* counters;              // 2 per output tile (arrive, depart); zero between launches
  unsigned long long* trace;  // optional per-CTA %globaltimer stamps (ALORA_GEMM_TRACE=1)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot)                                                                                   \
  do {                                                                                                \
    if (args.trace) args.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 6 + (slot)] = gtime(); \
  } while (0)

template <int BN>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStage) > 10 ? 10 : (kSmemBudget / kStage);
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kRedStride = BN + 4;  // fp32 partial-tile row stride (floats) in smem
  static_assert(kBM * kRedStride * 4 <= kStages * kStage, "partial tile must fit in the stage ring");
  static constexpr int kSmem = 1024 + kStages * kStage + 256;
};

// LoRA K-block j covers slots [j*64/R, ((j+1)*64-1)/R]; present if any of them is in the tile mask.
__device__ __forceinline__ bool lora_block_present(int j, int rank, uint32_t mask) {
  const int s0 = (j * kBK) / rank, s1 = (j * kBK + kBK - 1) / rank;
  for (int s = s0; s <= s1 && s < 32; ++s)
    if ((mask >> s) & 1u) return true;
  return false;
}

// The LoRA K range of an output tile. Select mode (lora_planes <= 1, the q|k|v projection): one plane of the
// shrink output, chosen by the tile's column range. Concat mode (lora_planes = P > 1, e.g. the SwiGLU gate|up
// GEMM whose tiles hold both targets' columns): all P planes in turn against up_t columns [p*ks + j*64, +64).
template <typename Args>
__device__ __forceinline__ int lora_np(const Args& a) { return a.lora_planes > 1 ? a.lora_planes : 1; }
template <typename Args>
__device__ __forceinline__ int lora_target(const Args& a, int n0) {
  return n0 < a.n_q ? 0 : (n0 < a.n_q + a.n_kv ? 1 : 2);
}
// K block i of the tile's LoRA range (i < np * nkl): S plane and up_t column of block j = i % nkl
template <typename Args>
__device__ __forceinline__ void lora_block(const Args& a, int i, int nkl, int target, int& j, int& plane, int& ucol) {
  const int p = i / nkl;
  j = i - p * nkl;
  plane = a.lora_planes > 1 ? p : target;
  ucol = p * a.ks + j * 64;
}
__device__ __forceinline__ int lora_blocks_present(int nkl, int np, int rank, uint32_t mask) {
  int n = 0;
  for (int j = 0; j < nkl; ++j) n += lora_block_present(j, rank, mask) ? 1 : 0;
  return n * np;
}

// fast SiLU: __fdividef (MUFU.RCP + FMUL, no IEEE-division slow path / divergence); -> 0 for very negative g
__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32], bool relu) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __align__(16) __nv_bfloat162 o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float a0 = v[q * 8 + e * 2], a1 = v[q * 8 + e * 2 + 1];
      if (relu) { a0 = fmaxf(a0, 0.f); a1 = fmaxf(a1, 0.f); }
      o[e] = __floats2bfloat162_rn(a0, a1);
    }
    *reinterpret_cast<int4*>(dst + q * 8) = *reinterpret_cast<int4*>(o);
  }
}

// Epilogue work is cut into units of 32 (or paired 2x32) columns of one row.
template <int BN>
__device__ __forceinline__ int units_per_row(const GemmArgs& a, int n0) {
  const int epi = a.epi & 15;
  if (epi == kEpiRope && n0 < a.rope_cols) return (BN / a.head_dim) * (a.head_dim / 64);
  if (epi == kEpiSwiglu) return (BN / 128) * 2;
  return BN / 32;
}

// Emit one unit for `row`; fetch(c0, v) provides the 32 fp32 accumulators of tile columns [c0, c0+32).
// 32 bf16 output columns [col, col + 32) of `row` that fall in the K or V section also go to the row's pool slot
__device__ __forceinline__ void kv_scatter(const GemmArgs& a, int row, int col, const float (&v)[32]) {
  const int c = col - a.kv_q;
  if (!a.kv_pool || c < 0 || c >= 2 * a.kv_w) return;
  const int slot = a.kv_slots[row];
  if (slot < 0) return;
  const int sel = c >= a.kv_w ? 1 : 0;
  const int64_t blk = slot / a.kv_block, off = slot % a.kv_block;
  store_bf16x32(a.kv_pool + (((blk * a.kv_layers + a.kv_layer) * 2 + sel) * a.kv_block + off) * a.kv_w +
                    (c - sel * a.kv_w), v, false);
}

template <int BN, typename Fetch>
__device__ __forceinline__ void emit_unit(const GemmArgs& a, int n0, int row, int u, Fetch&& fetch) {
  const bool live = row < a.M;
  const int epi = a.epi & 15;
  if (epi == kEpiRope && n0 < a.rope_cols) {
    // q/k heads: x1 = cols [i*32, +32), x2 = cols [half + i*32, +32) of the head; fp32 rotate, one rounding
    const int D = a.head_dim, half = D / 2, per_head = half / 32;
    const int hb = (u / per_head) * D, i = u % per_head;
    float x1[32], x2[32];
    fetch(hb + i * 32, x1);
    fetch(hb + half + i * 32, x2);
    if (!live) return;
    const int pos = a.positions[row];
    const float* cs = a.rope_cos + (int64_t)pos * half + i * 32;
    const float* sn = a.rope_sin + (int64_t)pos * half + i * 32;
    float r1[32], r2[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float c = __ldg(cs + j), s = __ldg(sn + j);
      r1[j] = x1[j] * c - x2[j] * s;
      r2[j] = x2[j] * c + x1[j] * s;
    }
    __nv_bfloat16* d1 = static_cast<__nv_bfloat16*>(a.C) + (int64_t)row * a.ldc + n0 + hb + i * 32;
    store_bf16x32(d1, r1, false);
    store_bf16x32(d1 + half, r2, false);
    kv_scatter(a, row, n0 + hb + i * 32, r1);
    kv_scatter(a, row, n0 + hb + half + i * 32, r2);
    return;
  }
  if (epi == kEpiSwiglu) {
    // tile columns [c*128, +64) gate, [c*128+64, +64) up -> 64 outputs at column n0/2 + c*64
    const int c = u / 2, h = u % 2;
    float g[32], v[32];
    fetch(c * 128 + h * 32, g);
    fetch(c * 128 + 64 + h * 32, v);
    if (!live) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) g[j] = silu(g[j]) * v[j];
    store_bf16x32(static_cast<__nv_bfloat16*>(a.C) + (int64_t)row * a.ldc + n0 / 2 + c * 64 + h * 32, g, false);
    return;
  }
  float v[32];
  const int c0 = u * 32;
  fetch(c0, v);
  const int col = n0 + c0;
  if (!live || col >= a.N) return;
  if (epi == kEpiLoraSelect) {
    const int slot = a.sel_row_slot[row];
    const bool takes = slot >= 0 && a.sel_row_apply[row];
    const int t = col / a.sel_sr, off = col % a.sel_sr;  // 32-col units never straddle a plane
    const bool tgt = takes && ((a.sel_targets[slot] >> (a.sel_tbit0 + t)) & 1u);
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (!(tgt && (off + e) / a.sel_rank == slot)) v[e] = 0.f;
    store_bf16x32(static_cast<__nv_bfloat16*>(a.C) + ((int64_t)t * a.M + row) * a.sel_sr + off, v, false);
  } else if (epi == kEpiAdd) {
    float* dst = static_cast<float*>(a.C) + (int64_t)row * a.ldc + col;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 x = *reinterpret_cast<float4*>(dst + q * 4);
      x.x += v[q * 4]; x.y += v[q * 4 + 1]; x.z += v[q * 4 + 2]; x.w += v[q * 4 + 3];
      *reinterpret_cast<float4*>(dst + q * 4) = x;
    }
  } else if (a.epi & 16) {
    float* dst = static_cast<float*>(a.C) + (int64_t)row * a.ldc + col;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(dst + q * 4) = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
  } else {
    store_bf16x32(static_cast<__nv_bfloat16*>(a.C) + (int64_t)row * a.ldc + col, v, epi == kEpiRelu);
    if (epi == kEpiRope) kv_scatter(a, row, col, v);  // the V columns (past the rotated q | k heads)
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_u,
                     const GemmArgs args) {
  using C = Cfg<BN>;
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m_tile = blockIdx.y, m0 = m_tile * kBM;
  const int split = blockIdx.z;  // == cluster rank when splits > 1
  const int S = args.splits;
  if (threadIdx.x == 0) TRACE(0);
  // this split's base K range (LoRA blocks ride with the last split)
  const int nkb_all = (args.K + kBK - 1) / kBK;
  const int per = (nkb_all + S - 1) / S;
  const int kb0 = min(nkb_all, split * per), kb1 = min(nkb_all, kb0 + per);
  int target = 0, nkl = 0;
  uint32_t mask = 0;
  if (args.ks > 0 && split == S - 1) {
    target = lora_target(args, n0);
    nkl = (args.ks + kBK - 1) / kBK;
    mask = args.tile_slot_mask[m_tile];
  }

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_a);
    sm100::prefetch_tmap(&tm_b);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<C::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int n_iters = kb1 - kb0;
  n_iters += lora_blocks_present(nkl, lora_np(args), args.rank, mask);

  // warp-converged loops, one elected lane per operation (see gemm_ws_kernel / gemm_bf16_persist_kernel)
  if (warp == 0) {
    const uint64_t pol_act = sm100::policy_evict_last();  // activations: re-read by every N tile
    const uint64_t pol_w = sm100::policy_evict_first();   // weights: streamed once per forward
    int s = 0;
    uint32_t phase = 0;
    auto next = [&] { if (++s == C::kStages) { s = 0; phase ^= 1; } };
    for (int kb = kb0; kb < kb1; ++kb) {
      sm100::mbar_wait(&empty[s], phase ^ 1);
      if (sm100::elect_one()) {
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_2d(sa, &tm_a, &full[s], kb * kBK, m0, pol_act);
        sm100::tma_load_2d(sa + C::kABytes, &tm_b, &full[s], kb * kBK, n0, pol_w);
      }
      __syncwarp();
      next();
    }
    for (int i = 0; i < lora_np(args) * nkl; ++i) {
      int j, plane, ucol;
      lora_block(args, i, nkl, target, j, plane, ucol);
      if (!lora_block_present(j, args.rank, mask)) continue;
      sm100::mbar_wait(&empty[s], phase ^ 1);
      if (sm100::elect_one()) {
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_3d(sa, &tm_s, &full[s], j * kBK, m0, plane, pol_act);
        sm100::tma_load_2d(sa + C::kABytes, &tm_u, &full[s], ucol, n0, pol_w);
      }
      __syncwarp();
      next();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
    int s = 0;
    uint32_t phase = 0;
    for (int it = 0; it < n_iters; ++it) {
      sm100::mbar_wait(&full[s], phase);
      sm100::tc_fence_after();
      if (it == 0 && lane == 0) TRACE(1);
      if (sm100::elect_one()) {
        const uint8_t* sa = smem + s * C::kStage;
        const uint64_t da = sm100::umma_desc_sw128(sa);
        const uint64_t db = sm100::umma_desc_sw128(sa + C::kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // +32 bytes per K=16 step inside the 128B swizzle atom
          sm100::mma_bf16_ss(tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc,
                             (it > 0 || k > 0) ? 1u : 0u);
        sm100::mma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == C::kStages) { s = 0; phase ^= 1; }
    }
    if (sm100::elect_one()) sm100::mma_commit(tmem_full);
    __syncwarp();
  } else {
    // epilogue warps: warp w owns TMEM lanes [32*(w%4), +32) = tile rows
    const int quarter = warp & 3;
    const int trow_idx = quarter * 32 + lane;
    sm100::mbar_wait(tmem_full, 0);
    sm100::tc_fence_after();
    if (threadIdx.x == 64) TRACE(2);
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    auto tmem_fetch = [&](int c0, float (&v)[32]) {  // warp-collective
      uint32_t r[32];
      sm100::tmem_ld_32x32b_x32(trow + c0, r);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = n_iters > 0 ? __uint_as_float(r[i]) : 0.f;
    };
    const bool quarter_live = m0 + quarter * 32 < args.M;  // warp-uniform: skip all-padding lane quarters
    if (S == 1) {
      const int units = units_per_row<BN>(args, n0);
      if (quarter_live)
        for (int u = 0; u < units; ++u) emit_unit<BN>(args, n0, m0 + trow_idx, u, tmem_fetch);
    } else if (quarter_live) {
      // publish this split's fp32 partial rows (L2-resident workspace [S][m_tiles*128][N])
      float* part = args.partial + ((int64_t)(split * gridDim.y + m_tile) * kBM + trow_idx) * args.N + n0;
      const bool row_live = m0 + trow_idx < args.M;
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_fetch(c, v);
        if (!row_live) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          __stcg(reinterpret_cast<float4*>(part + c + q * 4), make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]));
      }
    }
  }
  if (threadIdx.x == 64) TRACE(3);
  if (S > 1 && warp >= 2) {
    // all S splits of this tile are co-resident (cooperative launch, grid <= SM count): wait for every
    // partial, then split k reduces rows [k*R/S, (k+1)*R/S) in split order and runs their epilogue
    int* arrive = args.counters + 2 * (m_tile * gridDim.x + blockIdx.x);
    __threadfence();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 64) {
      atomicAdd(arrive, 1);
      while (*reinterpret_cast<volatile int*>(arrive) < S) __nanosleep(32);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    __threadfence();
    if (threadIdx.x == 64) TRACE(4);
    const int valid_rows = min(kBM, args.M - m0);
    const int r_beg = split * valid_rows / S, r_end = (split + 1) * valid_rows / S;
    const int my_rows = r_end - r_beg;
    float* red = reinterpret_cast<float*>(smem);  // [my_rows][kRedStride] in the idle stage ring
    constexpr int G4 = BN / 4;
    const int64_t pstride = (int64_t)gridDim.y * kBM * args.N;
    for (int g = threadIdx.x - 64; g < my_rows * G4; g += kThreads - 64) {
      const int rl = g / G4, c4 = (g % G4) * 4;
      const float* src = args.partial + ((int64_t)m_tile * kBM + r_beg + rl) * args.N + n0 + c4;
      float4 p[kMaxSplits];
#pragma unroll
      for (int k = 0; k < kMaxSplits; ++k)
        if (k < S) p[k] = __ldcg(reinterpret_cast<const float4*>(src + k * pstride));
      float4 acc = p[0];
#pragma unroll
      for (int k = 1; k < kMaxSplits; ++k)
        if (k < S) { acc.x += p[k].x; acc.y += p[k].y; acc.z += p[k].z; acc.w += p[k].w; }
      *reinterpret_cast<float4*>(red + rl * C::kRedStride + c4) = acc;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int units = units_per_row<BN>(args, n0);
    for (int w = threadIdx.x - 64; w < my_rows * units; w += kThreads - 64) {
      const int rl = w / units, u = w % units;
      auto smem_fetch = [&](int c0, float (&v)[32]) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 t = *reinterpret_cast<const float4*>(red + rl * C::kRedStride + c0 + q * 4);
          v[q * 4] = t.x; v[q * 4 + 1] = t.y; v[q * 4 + 2] = t.z; v[q * 4 + 3] = t.w;
        }
      };
      emit_unit<BN>(args, n0, m0 + r_beg + rl, u, smem_fetch);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 64 && atomicAdd(arrive + 1, 1) == S - 1) {  // last one out resets for the next launch
      arrive[0] = 0;
      arrive[1] = 0;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<C::kTmemCols>(tmem);
  if (threadIdx.x == 64) TRACE(5);
}

// ============================================================================================================
// Persistent large-M GEMM (prefill / LoRA recompute, no split-K): one CTA per SM walks the output tiles
// (N-fastest, so the tiles in flight share A row blocks and B column blocks through L2) and keeps TWO TMEM
// accumulators: the epilogue of tile i (TMEM -> registers -> fused epilogue -> global) runs while the MMA warp
// accumulates tile i+1, instead of every CTA paying its epilogue, setup and TMEM allocation serially.
//   warp 0   TMA producer over (tile, K block) through one smem ring
//   warp 1   TMEM allocator (2 x BN columns) + tcgen05.mma issuer; waits tmem_empty[b] before reusing b
//   warps 2-5 epilogue: wait tmem_full[b], emit, arrive tmem_empty[b]
// ============================================================================================================
template <int BN>
struct PCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStage) > 10 ? 10 : (kSmemBudget / kStage);
  static constexpr int kTmemCols = 2 * BN;  // two accumulators
  static constexpr int kSmem = 1024 + kStages * kStage + 256;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_persist_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                             const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_u,
                             const GemmArgs args) {
  using C = PCfg<BN>;
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_n = (args.N + BN - 1) / BN, n_m = (args.M + kBM - 1) / kBM;
  const int n_tiles = n_n * n_m;
  const int nkb = (args.K + kBK - 1) / kBK;
  const int nkl = args.ks > 0 ? (args.ks + kBK - 1) / kBK : 0;
  if (threadIdx.x == 0) TRACE(0);

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_a);
    sm100::prefetch_tmap(&tm_b);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&tmem_full[b], 1);
      sm100::mbar_init(&tmem_empty[b], 4);  // one arrival per epilogue warp
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<C::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // LoRA extra K of a tile: the m tile's slot mask decides which K blocks are present
  // Tile order: groups of up to kGroupM M tiles, M-fastest inside a group. The 148 CTAs in flight then cover
  // ~148 / group N tiles with every M tile of the group, so each weight tile is fetched from HBM once and
  // served to the group's CTAs from L2 (N-fastest order re-read the weights from HBM once per M tile: 5.8x
  // the weight bytes for the C3 MLP-in GEMM at M = 1024, which made it HBM-bound); the group's activation
  // rows (<= 2048 x K bf16) stay L2-resident across its N tiles.
  constexpr int kGroupM = 16;
  auto tile_of = [&](int t, int& m_tile, int& n0) {
    const int gm = min(n_m, kGroupM);
    const int g = t / (gm * n_n), r = t - g * gm * n_n;
    const int gs = min(gm, n_m - g * gm);
    m_tile = g * gm + r % gs;
    n0 = (r / gs) * BN;
  };

  // Producer and MMA loops run warp-converged with one elected lane per operation (see gemm_ws_kernel: a lone
  // lane looping while its siblings wait let ptxas clobber the MMA's uniform TMEM operand).
  if (warp == 0) {
    const uint64_t pol_act = sm100::policy_evict_last();
    const uint64_t pol_w = sm100::policy_evict_normal();  // re-read by the m tiles in flight
    int s = 0;
    uint32_t phase = 0;
    auto next = [&] { if (++s == C::kStages) { s = 0; phase ^= 1; } };
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      int m_tile, n0;
      tile_of(t, m_tile, n0);
      const int m0 = m_tile * kBM;
      for (int kb = 0; kb < nkb; ++kb) {
        sm100::mbar_wait(&empty[s], phase ^ 1);
        if (sm100::elect_one()) {
          uint8_t* sa = smem + s * C::kStage;
          sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
          sm100::tma_load_2d(sa, &tm_a, &full[s], kb * kBK, m0, pol_act);
          sm100::tma_load_2d(sa + C::kABytes, &tm_b, &full[s], kb * kBK, n0, pol_w);
        }
        __syncwarp();
        next();
      }
      if (nkl > 0) {
        const int target = lora_target(args, n0);
        const uint32_t mask = args.tile_slot_mask[m_tile];
        for (int i = 0; i < lora_np(args) * nkl; ++i) {
          int j, plane, ucol;
          lora_block(args, i, nkl, target, j, plane, ucol);
          if (!lora_block_present(j, args.rank, mask)) continue;
          sm100::mbar_wait(&empty[s], phase ^ 1);
          if (sm100::elect_one()) {
            uint8_t* sa = smem + s * C::kStage;
            sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
            sm100::tma_load_3d(sa, &tm_s, &full[s], j * kBK, m0, plane, pol_act);
            sm100::tma_load_2d(sa + C::kABytes, &tm_u, &full[s], ucol, n0, pol_w);
          }
          __syncwarp();
          next();
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
    int s = 0;
    uint32_t phase = 0;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      int m_tile, n0;
      tile_of(t, m_tile, n0);
      const int b = i & 1;
      if (i >= 2) sm100::mbar_wait(&tmem_empty[b], ((i >> 1) - 1) & 1);  // epilogue drained accumulator b
      sm100::tc_fence_after();
      const uint32_t acc_t = tmem + (uint32_t)(b * BN);
      int n_iters = nkb;
      if (nkl > 0) {
        n_iters += lora_blocks_present(nkl, lora_np(args), args.rank, args.tile_slot_mask[m_tile]);
      }
      for (int it = 0; it < n_iters; ++it) {
        sm100::mbar_wait(&full[s], phase);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          const uint8_t* sa = smem + s * C::kStage;
          const uint64_t da = sm100::umma_desc_sw128(sa);
          const uint64_t db = sm100::umma_desc_sw128(sa + C::kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            sm100::mma_bf16_ss(acc_t, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, (it > 0 || k > 0) ? 1u : 0u);
          sm100::mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == C::kStages) { s = 0; phase ^= 1; }
      }
      if (sm100::elect_one()) sm100::mma_commit(&tmem_full[b]);
      __syncwarp();
    }
  } else {
    const int quarter = warp & 3;
    const int trow_idx = quarter * 32 + lane;
    int i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      int m_tile, n0;
      tile_of(t, m_tile, n0);
      const int m0 = m_tile * kBM;
      const int b = i & 1;
      sm100::mbar_wait(&tmem_full[b], (i >> 1) & 1);
      sm100::tc_fence_after();
      const uint32_t trow = tmem + (uint32_t)(b * BN) + ((uint32_t)(quarter * 32) << 16);
      auto tmem_fetch = [&](int c0, float (&v)[32]) {  // warp-collective
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(trow + c0, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
      };
      if (m0 + quarter * 32 < args.M) {  // warp-uniform: skip all-padding lane quarters
        const int units = units_per_row<BN>(args, n0);
        for (int u = 0; u < units; ++u) emit_unit<BN>(args, n0, m0 + trow_idx, u, tmem_fetch);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tmem_empty[b]);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<C::kTmemCols>(tmem);
  if (threadIdx.x == 64) TRACE(5);
}

template <int BN>
int launch_persist(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& s, const CUtensorMap& u,
                   const GemmArgs& args, cudaStream_t st) {
  using C = PCfg<BN>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_bf16_persist_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  const int tiles = ((args.N + BN - 1) / BN) * ((args.M + kBM - 1) / kBM);
  const dim3 grid(std::min(tiles, kNumSMs));
  ALORA_CUDA_CHECK(launch_pdl(gemm_bf16_persist_kernel<BN>, grid, dim3(kThreads), C::kSmem, st, nullptr, 0, a, b, s, u,
                              args));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

template <int BN>
int launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& s, const CUtensorMap& u,
           const GemmArgs& args, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_bf16_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  const dim3 grid((args.N + BN - 1) / BN, (args.M + kBM - 1) / kBM, args.splits);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // split-K tiles spin-wait on each other: co-residency required
  attr[0].val.cooperative = 1;
  GemmArgs targs = args;
  static unsigned long long* trace_buf = nullptr;
  static const bool tracing = getenv("ALORA_GEMM_TRACE") != nullptr;
  const int n_ctas = grid.x * grid.y * grid.z;
  if (tracing) {
    if (!trace_buf) cudaMalloc(&trace_buf, sizeof(unsigned long long) * 6 * 65536);
    cudaMemsetAsync(trace_buf, 0, sizeof(unsigned long long) * 6 * n_ctas, st);
    targs.trace = trace_buf;
  }
  if (args.splits > 1) {  // cooperative (co-resident split-K): no programmatic overlap with the previous kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launch(reinterpret_cast<const void*>(gemm_bf16_kernel<BN>), grid);
    if (cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<BN>, a, b, s, u, targs) != cudaSuccess) return ALORA_ECUDA;
  } else if (launch_pdl(gemm_bf16_kernel<BN>, grid, dim3(kThreads), C::kSmem, st, nullptr, 0, a, b, s, u, targs) !=
             cudaSuccess) {
    return ALORA_ECUDA;
  }
  ALORA_LAUNCH_CHECK();
  if (tracing) {  // phase timings relative to the earliest CTA start (debug only)
    std::vector<unsigned long long> h(6 * n_ctas);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tend = 0;
    double ph[5] = {0, 0, 0, 0, 0};
    for (int c = 0; c < n_ctas; ++c) {
      t0 = std::min(t0, h[6 * c]);
      tend = std::max(tend, h[6 * c + 5]);
      for (int p = 0; p < 5; ++p)
        if (h[6 * c + p + 1] && h[6 * c + p]) ph[p] += double(h[6 * c + p + 1] - h[6 * c + p]);
    }
    unsigned long long last_start = 0;
    for (int c = 0; c < n_ctas; ++c) last_start = std::max(last_start, h[6 * c]);
    fprintf(stderr,
            "[gemm trace] M=%d N=%d K=%d BN=%d splits=%d ctas=%d span %.2f us, last CTA start +%.2f us; mean "
            "setup->1st data %.2f, mainloop %.2f, epi %.2f, sync %.2f, reduce+exit %.2f us\n",
            args.M, args.N, args.K, BN, args.splits, n_ctas, (tend - t0) / 1e3, (last_start - t0) / 1e3,
            ph[0] / n_ctas / 1e3, ph[1] / n_ctas / 1e3, ph[2] / n_ctas / 1e3, ph[3] / n_ctas / 1e3,
            ph[4] / n_ctas / 1e3);
  }
  return ALORA_OK;
}


// ============================================================================================================
// Weight-streaming GEMM for small M (M <= 256: aLoRA suffix steps, decode).
//
// One CTA owns an N tile of BN weight rows and a K slab, and ALL MT (<= 2) 128-row token tiles, so each
// weight byte enters exactly one SM once and the activations are re-read only N/BN times (the per-SM
// L2->SM ingest, not HBM, is what bounds narrow tiles). K is split over a thread-block cluster of S CTAs
// (cluster dims 1x1xS); each parks its fp32 partial tile in its own shared memory and, after a cluster
// barrier, CTA r reduces token rows [r*M/S, (r+1)*M/S) over distributed shared memory, summing the S
// partials in rank order (deterministic for a given S), and runs the fused epilogue on them.
//   warp 0           TMA producer; weight slabs of the first stages are issued BEFORE griddepcontrol.wait
//                    (weights do not depend on the previous kernel), activations after it
//   warp 1           TMEM allocator + single-thread tcgen05.mma issuer (MT accumulators of 128 x BN)
//   warps 2..2+4MT   epilogue: warp w reads TMEM lanes 32*(w%4) of token tile (w-2)/4
// ============================================================================================================
#ifndef ALORA_WS_MT2_STAGES
#define ALORA_WS_MT2_STAGES 4
#endif
template <int BN, int MT>
struct WsCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = MT * kABytes + kBBytes;
  static constexpr int kMaxStages = MT == 2 ? ALORA_WS_MT2_STAGES : 12;
  static constexpr int kStages = (kSmemBudget / kStage) > kMaxStages ? kMaxStages : (kSmemBudget / kStage);
  static constexpr int kAcc = MT * BN;
  static constexpr int kTmemCols = kAcc <= 32 ? 32 : kAcc <= 64 ? 64 : kAcc <= 128 ? 128 : kAcc <= 256 ? 256 : 512;
  static constexpr int kRedStride = BN + 4;
  static constexpr int kRedBytes = MT * kBM * kRedStride * 4;
  static constexpr bool kCanSplit = kRedBytes <= kStages * kStage;
  static constexpr int kThreads = 64 + 128 * MT;
  static constexpr int kSmem = 1024 + kStages * kStage + 256;
};

template <int BN, int MT>
__global__ void __launch_bounds__(WsCfg<BN, MT>::kThreads, 1)
    gemm_ws_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_u,
                   const __grid_constant__ CUtensorMap tm_p, const GemmArgs args) {
  using C = WsCfg<BN, MT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int S = args.splits;
  const int split = blockIdx.z;
  if (threadIdx.x == 0) TRACE(0);
  const int nkb_all = (args.K + kBK - 1) / kBK;
  // The LoRA K blocks ride with the last split: size the splits over base + LoRA blocks so that split does not
  // run ~nkl blocks longer than the others, keeping at least one base block in it
  int per = (nkb_all + S - 1) / S;
  if (args.ks > 0 && S > 1) {
    const int nkl_all = lora_np(args) * ((args.ks + kBK - 1) / kBK);
    per = max(per, min((nkb_all + nkl_all + S - 1) / S, (nkb_all - 1) / (S - 1)));
  }
  const int kb0 = min(nkb_all, split * per), kb1 = split == S - 1 ? nkb_all : min(nkb_all, kb0 + per);
  const int n_base = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_a);
    sm100::prefetch_tmap(&tm_b);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<C::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Producer and MMA warps run their loops warp-converged and elect one lane per operation: a lone lane
  // looping while the other 31 wait in __syncwarp lets ptxas reuse uniform registers of the diverged
  // path (observed: the MMA's TMEM operand clobbered -> out-of-range TMEM address).
  if (warp == 0) {
    const uint64_t pol_act = sm100::policy_evict_last();
    const uint64_t pol_w = sm100::policy_evict_first();
    // weights of the first stages go out before the dependency wait: they overlap the previous kernel
    const int n_pre = min(C::kStages, n_base);
    for (int i = 0; i < n_pre; ++i) {
      if (sm100::elect_one()) {
        uint8_t* sa = smem + i * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[i], C::kStage);
        sm100::tma_load_2d(sa + MT * C::kABytes, &tm_b, &full[i], (kb0 + i) * kBK, n0, pol_w);
      }
      __syncwarp();
    }
    pdl_wait();
    pdl_trigger();
    int target = 0, nkl = 0;
    uint32_t mask = 0;
    if (args.ks > 0 && split == S - 1) {
      target = lora_target(args, n0);
      nkl = (args.ks + kBK - 1) / kBK;
      for (int mt = 0; mt < MT; ++mt) mask |= args.tile_slot_mask[mt];
    }
    for (int i = 0; i < n_pre; ++i) {
      if (sm100::elect_one()) {
        uint8_t* sa = smem + i * C::kStage;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          sm100::tma_load_2d(sa + mt * C::kABytes, &tm_a, &full[i], (kb0 + i) * kBK, mt * kBM, pol_act);
      }
      __syncwarp();
    }
    int s = n_pre % C::kStages;
    uint32_t phase = n_pre == C::kStages ? 1u : 0u;
    auto next = [&] { if (++s == C::kStages) { s = 0; phase ^= 1; } };
    for (int kb = kb0 + n_pre; kb < kb1; ++kb) {
      sm100::mbar_wait(&empty[s], phase ^ 1);
      if (sm100::elect_one()) {
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_2d(sa + MT * C::kABytes, &tm_b, &full[s], kb * kBK, n0, pol_w);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          sm100::tma_load_2d(sa + mt * C::kABytes, &tm_a, &full[s], kb * kBK, mt * kBM, pol_act);
      }
      __syncwarp();
      next();
    }
    for (int i = 0; i < lora_np(args) * nkl; ++i) {
      int j, plane, ucol;
      lora_block(args, i, nkl, target, j, plane, ucol);
      if (!lora_block_present(j, args.rank, mask)) continue;
      sm100::mbar_wait(&empty[s], phase ^ 1);
      if (sm100::elect_one()) {
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_2d(sa + MT * C::kABytes, &tm_u, &full[s], ucol, n0, pol_w);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          sm100::tma_load_3d(sa + mt * C::kABytes, &tm_s, &full[s], j * kBK, mt * kBM, plane, pol_act);
      }
      __syncwarp();
      next();
    }
  } else {
    pdl_wait();
    if (warp == 1) {
      int n_iters = n_base;
      if (args.ks > 0 && split == S - 1) {
        uint32_t mask = 0;
        for (int mt = 0; mt < MT; ++mt) mask |= args.tile_slot_mask[mt];
        n_iters += lora_blocks_present((args.ks + kBK - 1) / kBK, lora_np(args), args.rank, mask);
      }
      constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
      int s = 0;
      uint32_t phase = 0;
      for (int it = 0; it < n_iters; ++it) {
        sm100::mbar_wait(&full[s], phase);
        sm100::tc_fence_after();
        if (it == 0 && lane == 0) TRACE(1);
        if (sm100::elect_one()) {
          const uint8_t* sa = smem + s * C::kStage;
          const uint64_t db = sm100::umma_desc_sw128(sa + MT * C::kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint64_t da = sm100::umma_desc_sw128(sa + mt * C::kABytes);
              sm100::mma_bf16_ss(tmem + mt * BN, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc,
                                 (it > 0 || k > 0) ? 1u : 0u);
            }
          }
          sm100::mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == C::kStages) { s = 0; phase ^= 1; }
      }
      if (sm100::elect_one()) sm100::mma_commit(tmem_full);
      __syncwarp();
    } else {
      // epilogue warps
      const int ew = warp - 2;
      const int mt = ew >> 2, quarter = warp & 3;
      const int trow = mt * kBM + quarter * 32 + lane;  // token row (the CTA spans all token tiles)
      const bool has_acc = n_base > 0 || (args.ks > 0 && split == S - 1);
      sm100::mbar_wait(tmem_full, 0);
      sm100::tc_fence_after();
      if (threadIdx.x == 64) TRACE(2);
      const uint32_t taddr = tmem + mt * BN + ((uint32_t)(quarter * 32) << 16);
      auto tmem_fetch = [&](int c0, float (&v)[32]) {  // warp-collective
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(taddr + c0, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = has_acc ? __uint_as_float(r[i]) : 0.f;
      };
      const bool quarter_live = mt * kBM + quarter * 32 < args.M;
      if (S == 1) {
        const int units = units_per_row<BN>(args, n0);
        if (quarter_live) {
          if (args.argmax != nullptr) {
            unsigned long long best = 0ull;
            auto fetch_am = [&](int c0, float (&v)[32]) {
              tmem_fetch(c0, v);
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                uint32_t u32 = __float_as_uint(v[j]);
                u32 = (u32 & 0x80000000u) ? ~u32 : (u32 | 0x80000000u);
                const unsigned long long key =
                    ((unsigned long long)u32 << 32) | (0xFFFFFFFFu - (uint32_t)(n0 + c0 + j));
                best = key > best ? key : best;
              }
            };
            for (int u = 0; u < units; ++u) emit_unit<BN>(args, n0, trow, u, fetch_am);
            if (trow < args.M) atomicMax(args.argmax + trow, best);
          } else {
            for (int u = 0; u < units; ++u) emit_unit<BN>(args, n0, trow, u, tmem_fetch);
          }
        }
      } else if (quarter_live) {
        // deferred split-K: this split's fp32 partial rows -> partial[split][row][n]; the consuming kernel
        // (residual RMSNorm / QKV finalize) sums the splits in order and applies the epilogue
        // (32 x 32 fp32 boxes staged in the idle stage ring with the 128B swizzle, written by TMA stores;
        // two staging buffers per warp, rows >= M clipped by the tensor map)
        uint8_t* stg = smem + ew * 8192;
        const int row0 = mt * kBM + quarter * 32;
        int ci = 0;
        for (int c = 0; c < BN; c += 32, ++ci) {
          float v[32];
          tmem_fetch(c, v);
          uint8_t* buf = stg + (ci & 1) * 4096;
          if (ci >= 2) {
            if (lane == 0) sm100::bulk_wait_read<1>();
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_3d(&tm_p, buf, n0 + c, row0, split);
            sm100::bulk_commit();
          }
          __syncwarp();
        }
        if (lane == 0) sm100::bulk_wait<0>();
        __syncwarp();
      }
    }
  }
  if (threadIdx.x == 64) TRACE(3);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<C::kTmemCols>(tmem);
  if (threadIdx.x == 64) TRACE(5);
}

template <int BN, int MT>
int launch_ws(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& s, const CUtensorMap& u,
              const GemmArgs& args, cudaStream_t st) {
  CUtensorMap p = a;  // deferred split-K partials [splits][M][N] fp32 (TMA-store target)
  if (args.splits > 1 && !make_tmap_3d_f32(&p, args.partial, args.splits, args.M, args.N, 32)) return ALORA_ECUDA;
  using C = WsCfg<BN, MT>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_ws_kernel<BN, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  GemmArgs targs = args;
  static unsigned long long* trace_buf = nullptr;
  static const bool tracing = getenv("ALORA_GEMM_TRACE") != nullptr;
  const dim3 grid(args.N / BN, 1, args.splits);
  const int n_ctas = grid.x * grid.z;
  if (tracing) {
    if (!trace_buf) cudaMalloc(&trace_buf, sizeof(unsigned long long) * 6 * 65536);
    cudaMemsetAsync(trace_buf, 0, sizeof(unsigned long long) * 6 * n_ctas, st);
    targs.trace = trace_buf;
  }
  if (launch_pdl(gemm_ws_kernel<BN, MT>, grid, dim3(C::kThreads), C::kSmem, st, nullptr, 0, a, b, s, u, p, targs) !=
      cudaSuccess)
    return ALORA_ECUDA;
  ALORA_LAUNCH_CHECK();
  if (tracing) {
    std::vector<unsigned long long> h(6 * n_ctas);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tend = 0;
    double ph[5] = {0, 0, 0, 0, 0};
    for (int c = 0; c < n_ctas; ++c) {
      t0 = std::min(t0, h[6 * c]);
      tend = std::max(tend, h[6 * c + 5]);
      for (int p = 0; p < 5; ++p)
        if (h[6 * c + p + 1] && h[6 * c + p]) ph[p] += double(h[6 * c + p + 1] - h[6 * c + p]);
    }
    fprintf(stderr,
            "[gemm_ws trace] M=%d N=%d K=%d BN=%d MT=%d splits=%d ctas=%d span %.2f us; mean setup->1st data %.2f, "
            "mainloop %.2f, epi %.2f, sync %.2f, reduce+exit %.2f us\n",
            args.M, args.N, args.K, BN, MT, args.splits, n_ctas, (tend - t0) / 1e3, ph[0] / n_ctas / 1e3,
            ph[1] / n_ctas / 1e3, ph[2] / n_ctas / 1e3, ph[3] / n_ctas / 1e3, ph[4] / n_ctas / 1e3);
  }
  return ALORA_OK;
}


// ============================================================================================================
// Decode GEMM (M <= 32 token rows): swap-AB weight streaming. The MMA's 128-row A operand is a tile of 128
// WEIGHT rows and the B operand the (zero-padded) token rows, N = MN in {16, 32}, so a stage is 16 KB of
// weights + MN*128 B of activations: ~11 stages (~176 KB of weights in flight per SM) instead of the
// half-empty 128-row token tiles of gemm_ws_kernel. TMEM lane = output column, TMEM column = token.
//   warp 0 TMA producer (weights of the first stages before griddepcontrol.wait), warp 1 MMA issuer,
//   warps 2..5 epilogue. Epilogues: fp32 split-K partials [split][M][N] (consumed by residual RMSNorm /
//   QKV finalize / LoRA select), C(fp32) += acc, fp32 store (+ fused greedy argmax), SwiGLU.
// ============================================================================================================
enum DecEpi : int { kDecPartial = 0, kDecAdd = 1, kDecStoreF32 = 2, kDecSwiglu = 3 };

template <int MN>
struct DecCfg {
  static constexpr int kWBytes = kBM * kBK * 2;   // 128 weight rows x 64 K
  static constexpr int kXBytes = MN * kBK * 2;    // MN token rows x 64 K
  static constexpr int kStage = kWBytes + kXBytes;
  static constexpr int kStages = (kSmemBudget / kStage) > 12 ? 12 : (kSmemBudget / kStage);
  static constexpr int kSmem = 1024 + kStages * kStage + 256 + 128 * 33 * 4;  // + SwiGLU exchange tile
};

struct DecArgs {
  int M, N, K, splits, mode;
  float* out;          // partial base / C (fp32) / logits
  int ldc;
  __nv_bfloat16* out_bf16;  // SwiGLU output [M, N/2]
  int ld_bf16;
  unsigned long long* argmax;
  int ks, rank, n_q, n_kv;  // LoRA expand as extra K (last split)
  int lora_planes;
  const uint32_t* tile_slot_mask;
};

template <int MN>
__global__ void __launch_bounds__(192, 1)
    gemm_dec_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                    const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_s,
                    const DecArgs args) {
  // Persistent over N tiles (tile = blockIdx.x + j * gridDim.x): the stage ring runs on across tiles and two
  // TMEM accumulators alternate, so tile j's epilogue overlaps tile j+1's weight stream (no wave tail on
  // the 128256-row lm_head).
  using C = DecCfg<MN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  float* xch = reinterpret_cast<float*>(smem + C::kStages * C::kStage + 256);  // [128][33]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = args.N / kBM;
  const int S = args.splits, split = blockIdx.z;
  const int nkb_all = (args.K + kBK - 1) / kBK;
  const int per = (nkb_all + S - 1) / S;
  const int kb0 = min(nkb_all, split * per), kb1 = min(nkb_all, kb0 + per);
  const int n_base = kb1 - kb0;
  const bool lora_here = args.ks > 0 && split == S - 1;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_w);
    sm100::prefetch_tmap(&tm_x);
    for (int i = 0; i < C::kStages; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&tmem_full[b], 1);
      sm100::mbar_init(&tmem_empty[b], 128);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<64>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    const uint64_t pol_act = sm100::policy_evict_last();
    const uint64_t pol_w = sm100::policy_evict_first();
    const int n_pre = min(C::kStages, n_base);
    const int first = blockIdx.x;
    for (int i = 0; i < n_pre; ++i) {  // first tile's weights before the dependency wait
      if (sm100::elect_one()) {
        sm100::mbar_arrive_expect_tx(&full[i], C::kStage);
        sm100::tma_load_2d(smem + i * C::kStage, &tm_w, &full[i], (kb0 + i) * kBK, first * kBM, pol_w);
      }
      __syncwarp();
    }
    pdl_wait();
    pdl_trigger();
    uint32_t mask = 0;
    const int nkl = lora_here ? (args.ks + kBK - 1) / kBK : 0;
    if (lora_here) mask = args.tile_slot_mask[0];
    for (int i = 0; i < n_pre; ++i) {
      if (sm100::elect_one())
        sm100::tma_load_2d(smem + i * C::kStage + C::kWBytes, &tm_x, &full[i], (kb0 + i) * kBK, 0, pol_act);
      __syncwarp();
    }
    int st = n_pre % C::kStages;
    uint32_t phase = n_pre == C::kStages ? 1u : 0u;
    auto next = [&] { if (++st == C::kStages) { st = 0; phase ^= 1; } };
    for (int tile = first; tile < n_tiles; tile += gridDim.x) {
      const int n0 = tile * kBM;
      for (int kb = (tile == first ? kb0 + n_pre : kb0); kb < kb1; ++kb) {
        sm100::mbar_wait(&empty[st], phase ^ 1);
        if (sm100::elect_one()) {
          uint8_t* sa = smem + st * C::kStage;
          sm100::mbar_arrive_expect_tx(&full[st], C::kStage);
          sm100::tma_load_2d(sa, &tm_w, &full[st], kb * kBK, n0, pol_w);
          sm100::tma_load_2d(sa + C::kWBytes, &tm_x, &full[st], kb * kBK, 0, pol_act);
        }
        __syncwarp();
        next();
      }
      const int target = lora_target(args, n0);
      for (int i = 0; i < lora_np(args) * nkl; ++i) {
        int j, plane, ucol;
        lora_block(args, i, nkl, target, j, plane, ucol);
        if (!lora_block_present(j, args.rank, mask)) continue;
        sm100::mbar_wait(&empty[st], phase ^ 1);
        if (sm100::elect_one()) {
          uint8_t* sa = smem + st * C::kStage;
          sm100::mbar_arrive_expect_tx(&full[st], C::kStage);
          sm100::tma_load_2d(sa, &tm_u, &full[st], ucol, n0, pol_w);
          sm100::tma_load_3d(sa + C::kWBytes, &tm_s, &full[st], j * kBK, 0, plane, pol_act);
        }
        __syncwarp();
        next();
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    int n_iters = n_base;
    if (lora_here) {
      n_iters += lora_blocks_present((args.ks + kBK - 1) / kBK, lora_np(args), args.rank, args.tile_slot_mask[0]);
    }
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, MN);
    int st = 0;
    uint32_t phase = 0;
    int j = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
      const int b = j & 1;
      if (j >= 2) {  // the epilogue has drained this accumulator (tile j-2)
        sm100::mbar_wait(&tmem_empty[b], ((j - 2) >> 1) & 1);
        sm100::tc_fence_after();
      }
      for (int it = 0; it < n_iters; ++it) {
        sm100::mbar_wait(&full[st], phase);
        sm100::tc_fence_after();
        if (sm100::elect_one()) {
          const uint8_t* sa = smem + st * C::kStage;
          const uint64_t da = sm100::umma_desc_sw128(sa);
          const uint64_t db = sm100::umma_desc_sw128(sa + C::kWBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            sm100::mma_bf16_ss(tmem + b * 32, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc,
                               (it > 0 || k > 0) ? 1u : 0u);
          sm100::mma_commit(&empty[st]);
        }
        __syncwarp();
        if (++st == C::kStages) { st = 0; phase ^= 1; }
      }
      if (sm100::elect_one()) sm100::mma_commit(&tmem_full[b]);
      __syncwarp();
    }
  } else {
    pdl_wait();
    const int quarter = warp & 3;
    const bool has_acc = n_base > 0 || lora_here;
    const int M = args.M;
    int j = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
      const int b = j & 1;
      const int n0 = tile * kBM;
      const int ncol = n0 + quarter * 32 + lane;  // this thread's output column (TMEM lane)
      sm100::mbar_wait(&tmem_full[b], (j >> 1) & 1);
      sm100::tc_fence_after();
      uint32_t r[32];
      sm100::tmem_ld_32x32b_x32(tmem + b * 32 + ((uint32_t)(quarter * 32) << 16), r);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tmem_empty[b]);  // the accumulator may be reused while the stores below run
      float v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = has_acc ? __uint_as_float(r[q]) : 0.f;
      if (args.mode == kDecPartial) {
        float* dst = args.out + (int64_t)split * M * args.N + ncol;
#pragma unroll
        for (int m = 0; m < MN; ++m)
          if (m < M) dst[(int64_t)m * args.N] = v[m];
      } else if (args.mode == kDecAdd) {
#pragma unroll
        for (int m = 0; m < MN; ++m)
          if (m < M) args.out[(int64_t)m * args.ldc + ncol] += v[m];
      } else if (args.mode == kDecStoreF32) {
#pragma unroll
        for (int m = 0; m < MN; ++m)
          if (m < M) args.out[(int64_t)m * args.ldc + ncol] = v[m];
        if (args.argmax) {
#pragma unroll
          for (int m = 0; m < MN; ++m) {
            if (m >= M) break;
            uint32_t u32 = __float_as_uint(v[m]);
            u32 = (u32 & 0x80000000u) ? ~u32 : (u32 | 0x80000000u);
            unsigned long long key = ((unsigned long long)u32 << 32) | (0xFFFFFFFFu - (uint32_t)ncol);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
              key = other > key ? other : key;
            }
            if (lane == 0) atomicMax(args.argmax + m, key);
          }
        }
      } else {  // kDecSwiglu: lanes 0-63 of the 128-row tile are gate rows, 64-127 the matching up rows
        const int row = quarter * 32 + lane;
#pragma unroll
        for (int m = 0; m < MN; ++m) xch[row * 33 + m] = v[m];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (quarter < 2) {
#pragma unroll
          for (int m = 0; m < MN; ++m)
            if (m < M)
              args.out_bf16[(int64_t)m * args.ld_bf16 + n0 / 2 + row] =
                  __float2bfloat16_rn(silu(xch[row * 33 + m]) * xch[(row + 64) * 33 + m]);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // xch is rewritten by the next tile
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<64>(tmem);
}

template <int MN>
int launch_dec(const CUtensorMap& w, const CUtensorMap& x, const CUtensorMap& u, const CUtensorMap& sm,
               const DecArgs& args, cudaStream_t st) {
  using C = DecCfg<MN>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_dec_kernel<MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  const int tiles = args.N / kBM;
  const int per_split = std::max(1, kNumSMs / args.splits);  // persistent: at most one CTA per SM
  const dim3 grid(std::min(tiles, per_split), 1, args.splits);
  if (launch_pdl(gemm_dec_kernel<MN>, grid, dim3(192), C::kSmem, st, nullptr, 0, w, x, u, sm, args) != cudaSuccess)
    return ALORA_ECUDA;
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

struct WsChoice {
  int bn = 0, splits = 1;
  double cost = 1e30;
};

// Modelled time of one weight-streaming launch. A CTA moves weight bytes at most at
//   min(SM ingest ~170 GB/s, stage-ring bytes in flight / ~1.2 us loaded latency) x BN / (BN + token rows)
// capped at the ~60 GB/s a CTA was measured to sustain; the launch is further bounded by HBM. K splits (S > 1) are only planned when the caller can defer the
// reduction to the consuming kernel, which then re-reads S fp32 partials from L2.
template <int BN, int MT>
void ws_consider(WsChoice& best, int M, int N, int K, bool can_defer, int64_t defer_cap) {
  using C = WsCfg<BN, MT>;
  const int nkb = (K + kBK - 1) / kBK;
  const int tiles = N / BN;
  const double mrows = std::min(M, MT * kBM);
  for (int S = 1; S <= kMaxSplits; ++S) {
    if (S > 1 && (!can_defer || (int64_t)S * M * N * 4 > defer_cap)) break;
    if (S > nkb) break;
    const int per = (nkb + S - 1) / S;
    if ((nkb + per - 1) / per != S) continue;  // no empty trailing splits
    const int ctas = tiles * S;
    const int waves = (ctas + kNumSMs - 1) / kNumSMs;
    const int active = std::min(ctas, kNumSMs);
    const double inflight = (double)C::kStages * (mrows + BN) * kBK * 2.0;
    const double ingest_rate = std::min(170e9, inflight / 1.2e-6);
    // measured on the B200: a lone weight-streaming CTA sustains ~30-60 GB/s of weights, so the SM count
    // engaged matters more than the tile shape
    const double w_rate = std::min(ingest_rate * BN / (BN + mrows), 60e9);
    const double wbytes = (double)N * K * 2.0;
    (void)active;
    double t = std::max(waves * ((double)BN * per * kBK * 2.0 / w_rate), wbytes / 6.5e12) + waves * 1.5e-6;
    if (S > 1) t += (double)S * M * N * 4.0 / 8e12 + 0.3e-6;
    if (t < best.cost * 0.97) {  // prefer the first (wider) tile unless clearly faster
      best.cost = t;
      best.bn = BN;
      best.splits = S;
    }
  }
}

template <int MT>
int dispatch_ws(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& s, const CUtensorMap& u,
                GemmArgs& args, int bn, cudaStream_t st) {
  switch (bn) {
    case 256: return launch_ws<256, MT>(a, b, s, u, args, st);
    case 128: return launch_ws<128, MT>(a, b, s, u, args, st);
    case 64: return launch_ws<64, MT>(a, b, s, u, args, st);
    default: return launch_ws<32, MT>(a, b, s, u, args, st);
  }
}

}  // namespace

void configure_gemm() {
  prefer_max_smem(gemm_bf16_kernel<32>);
  prefer_max_smem(gemm_bf16_kernel<64>);
  prefer_max_smem(gemm_bf16_kernel<128>);
  prefer_max_smem(gemm_bf16_kernel<256>);
  prefer_max_smem(gemm_ws_kernel<32, 1>);
  prefer_max_smem(gemm_ws_kernel<64, 1>);
  prefer_max_smem(gemm_ws_kernel<128, 1>);
  prefer_max_smem(gemm_ws_kernel<256, 1>);
  prefer_max_smem(gemm_ws_kernel<32, 2>);
  prefer_max_smem(gemm_ws_kernel<64, 2>);
  prefer_max_smem(gemm_ws_kernel<128, 2>);
  prefer_max_smem(gemm_ws_kernel<256, 2>);
  prefer_max_smem(gemm_dec_kernel<16>);
  prefer_max_smem(gemm_dec_kernel<32>);
}

int gemm_bf16(int epi, const __nv_bfloat16* A, int lda, const __nv_bfloat16* Bt, int ldb, void* Cout, int ldc, int M,
              int N, int K, const GemmLora* lora, cudaStream_t st, const GemmWs* ws, int max_splits,
              GemmDefer* defer) {
  if (defer) {
    defer->splits_out = 1;
    defer->deferred = false;
  }
  if (M == 0 || N == 0) return ALORA_OK;
  if (M < 0 || N < 0 || K < 1 || lda % 8 || ldb % 8 || ldc % 8) return ALORA_EINVAL;
  const int base_epi = epi & 15;
  if (g_batch_invariant && M > 2 * kBM) {
    // batch-invariant mode: every row goes through the same weight-streaming kernel with one K range, so
    // rows larger steps are cut into 256-row launches (row offsets into A, C, the shrink planes, the tile
    // slot masks and the positions)
    if (base_epi == kEpiLoraSelect) return ALORA_EINVAL;
    const int esz = (base_epi == kEpiAdd || (epi & 16)) ? 4 : 2;
    for (int r0 = 0; r0 < M; r0 += 2 * kBM) {
      const int mc = std::min(2 * kBM, M - r0);
      GemmLora lc;
      if (lora) {
        lc = *lora;
        if (lc.s) {
          lc.s_rows = lora->s_rows > 0 ? lora->s_rows : M;
          lc.s = lora->s + (int64_t)r0 * lora->ks;
        }
        if (lc.tile_slot_mask) lc.tile_slot_mask = lora->tile_slot_mask + r0 / kBM;
        if (lc.positions) lc.positions = lora->positions + r0;
        if (lc.argmax) lc.argmax = lora->argmax + r0;
      }
      void* cc = static_cast<char*>(Cout) + (int64_t)r0 * ldc * esz;
      const int rc = gemm_bf16(epi, A + (int64_t)r0 * lda, lda, Bt, ldb, cc, ldc, mc, N, K, lora ? &lc : nullptr, st,
                               ws, max_splits, nullptr);
      if (rc != ALORA_OK) return rc;
    }
    return ALORA_OK;
  }
  if (N % 32 != 0) return ALORA_EINVAL;
  if (base_epi == kEpiSwiglu && N % 128 != 0) return ALORA_EINVAL;
  // Tile width: large M keeps 128 (256 for SwiGLU); small M (weight streaming, <= 2 row tiles) picks the
  // widest BN that still gives ~one full wave of CTAs, so every SM streams weights without a K split.
  const int m_tiles_ = (M + kBM - 1) / kBM;
  int bn_min = 32;
  if (base_epi == kEpiSwiglu) bn_min = 128;
  if (base_epi == kEpiRope) bn_min = std::max(64, lora ? lora->head_dim : 64);
  if (lora && lora->s && lora->ks > 0) {
    while (bn_min < 128 && ((lora->n_q % bn_min) || (lora->n_kv % bn_min))) bn_min *= 2;
  }
  auto fits = [&](int bn) {
    return bn >= bn_min && N % bn == 0 && (base_epi != kEpiSwiglu || bn % 128 == 0) &&
           (!lora || !lora->s || lora->ks == 0 || ((lora->n_q % bn) == 0 && (lora->n_kv % bn) == 0)) &&
           (base_epi != kEpiRope || (lora->rope_cols % bn == 0 && bn % lora->head_dim == 0));
  };
  int BN = 0;
  if (m_tiles_ <= 2) {
    for (int bn : {256, 128, 64, 32})
      if (fits(bn) && m_tiles_ * (N / bn) >= (kNumSMs * 3) / 4) { BN = bn; break; }
    if (BN == 0)
      for (int bn : {32, 64, 128, 256})
        if (fits(bn)) { BN = bn; break; }
  } else {
    // 128 x 256 tiles when they cost fewer tile rounds: a 128 x 128 tile's K-block brings 32 KB through the
    // L2 -> SM crossbar per 256 MMA cycles, which held the M = 1024 projections near 50% of the tensor pipe
    // (ncu); a 256-wide tile does the same work in ~1.63x the time of a 128-wide one (measured), so it wins
    // unless it adds a round of tiles over the 148 SMs (C3: o-proj / MLP-down 256 -> 128 tiles, one round;
    // QKV stays at 128: 384 tiles in 3 rounds vs 192 in 2 x 1.63)
    static const int large_bn = getenv("ALORA_LARGE_BN") ? atoi(getenv("ALORA_LARGE_BN")) : 0;  // A/B override
    auto rounds = [&](int bn) { return (double)((m_tiles_ * (N / bn) + kNumSMs - 1) / kNumSMs); };
    if (base_epi == kEpiSwiglu) {
      if (fits(256)) BN = 256;
    } else if (large_bn > 0) {
      if (fits(large_bn)) BN = large_bn;
    } else if (fits(256) && fits(128) && rounds(256) * 1.63 < rounds(128)) {
      BN = 256;
    }
    if (BN == 0)
      for (int bn : {128, 64, 32})
        if (fits(bn)) { BN = bn; break; }
  }
  if (BN == 0) return ALORA_EINVAL;
  GemmArgs args{};
  args.C = Cout; args.ldc = ldc; args.M = M; args.N = N; args.K = K; args.epi = epi; args.rank = 1; args.splits = 1;
  if (base_epi == kEpiRope) {
    if (!lora || !lora->positions || !lora->rope_cos || !lora->rope_sin || lora->head_dim < 64 ||
        lora->head_dim % 64 || lora->rope_cols % BN || BN % lora->head_dim)
      return ALORA_EINVAL;
    args.positions = lora->positions;
    args.rope_cos = lora->rope_cos;
    args.rope_sin = lora->rope_sin;
    args.rope_cols = lora->rope_cols;
    args.head_dim = lora->head_dim;
  }
  if (lora && lora->argmax) {
    if (epi != (kEpiStore | 16) || M > 2 * kBM) return ALORA_EINVAL;
    args.argmax = lora->argmax;
  }
  if (base_epi == kEpiLoraSelect) {
    if (!lora || !lora->sel_row_slot || !lora->sel_row_apply || !lora->sel_targets || lora->sel_sr % 32 ||
        lora->sel_rank < 1 || lora->sel_planes < 1 || N != lora->sel_planes * lora->sel_sr)
      return ALORA_EINVAL;
    args.sel_row_slot = lora->sel_row_slot;
    args.sel_row_apply = lora->sel_row_apply;
    args.sel_targets = lora->sel_targets;
    args.sel_sr = lora->sel_sr;
    args.sel_rank = lora->sel_rank;
    args.sel_tbit0 = lora->sel_tbit0;
  }
  CUtensorMap ta, tb, ts, tu;
  const int up_planes = lora && lora->planes > 1 ? lora->planes : 1;  // up_t width = up_planes * ks
  if (!make_tmap_2d(&ta, A, M, K, lda, kBM, kBK)) return ALORA_ECUDA;
  if (!make_tmap_2d(&tb, Bt, N, K, ldb, BN, kBK)) return ALORA_ECUDA;
  ts = ta;
  tu = tb;
  if (lora != nullptr && lora->s != nullptr && lora->ks > 0) {
    if (lora->ks % 8 || (lora->n_q % BN) || (lora->n_kv % BN) || lora->rank < 1) return ALORA_EINVAL;
    if (lora->s_planes < 1 || lora->planes > lora->s_planes) return ALORA_EINVAL;
    if (!make_tmap_3d(&ts, lora->s, lora->s_planes, M, lora->ks, kBM, kBK, lora->s_rows)) return ALORA_ECUDA;
    if (!make_tmap_2d(&tu, lora->up_t, N, lora->ks * up_planes, lora->ks * up_planes, BN, kBK)) return ALORA_ECUDA;
    args.ks = lora->ks;
    args.rank = lora->rank;
    args.n_q = lora->n_q;
    args.n_kv = lora->n_kv;
    args.lora_planes = lora->planes;
    args.tile_slot_mask = lora->tile_slot_mask;
  }
  static const bool no_dec = getenv("ALORA_GEMM_NO_DEC") != nullptr;  // A/B switch off the swap-AB decode GEMM
  if (M <= 32 && !no_dec && !g_batch_invariant && N % kBM == 0 && K % kBK == 0) {
    const bool defer_ok = defer != nullptr && defer->partial != nullptr;
    int mode = -1;
    if (base_epi == kEpiAdd && !(epi & 16)) mode = defer_ok ? kDecPartial : kDecAdd;
    else if ((base_epi == kEpiRope || base_epi == kEpiLoraSelect) && defer_ok) mode = kDecPartial;
    else if (epi == (kEpiStore | 16)) mode = kDecStoreF32;
    else if (base_epi == kEpiSwiglu) mode = kDecSwiglu;
    if (mode >= 0) {
      DecArgs da{};
      da.M = M; da.N = N; da.K = K; da.mode = mode; da.splits = 1;
      const int tiles = N / kBM, nkb = K / kBK;
      if (mode == kDecPartial) {
        int sp = std::max(1, std::min({8, (2 * kNumSMs + tiles - 1) / tiles / 2 > 0 ? kNumSMs / tiles : 1, nkb / 4}));
        while (sp > 1 && (int64_t)sp * M * N * 4 > defer->capacity) --sp;
        const int per = (nkb + sp - 1) / sp;
        sp = (nkb + per - 1) / per;  // no empty trailing splits
        da.splits = sp;
        da.out = defer->partial;
        defer->splits_out = sp;
        defer->deferred = true;
      } else if (mode == kDecSwiglu) {
        da.out_bf16 = static_cast<__nv_bfloat16*>(Cout);
        da.ld_bf16 = ldc;
      } else {
        da.out = static_cast<float*>(Cout);
        da.ldc = ldc;
        da.argmax = lora ? lora->argmax : nullptr;
      }
      const int MN = M <= 16 ? 16 : 32;
      CUtensorMap tw, tx, tu, tsm;
      if (!make_tmap_2d(&tw, Bt, N, K, ldb, kBM, kBK)) return ALORA_ECUDA;
      if (!make_tmap_2d(&tx, A, M, K, lda, MN, kBK)) return ALORA_ECUDA;
      tu = tw;
      tsm = tx;
      if (lora != nullptr && lora->s != nullptr && lora->ks > 0) {
        if (lora->ks % 8 || (lora->n_q % kBM) || (lora->n_kv % kBM) || lora->rank < 1) return ALORA_EINVAL;
        if (!make_tmap_2d(&tu, lora->up_t, N, lora->ks * up_planes, lora->ks * up_planes, kBM, kBK)) return ALORA_ECUDA;
        if (!make_tmap_3d(&tsm, lora->s, lora->s_planes, M, lora->ks, MN, kBK, lora->s_rows)) return ALORA_ECUDA;
        da.ks = lora->ks;
        da.rank = lora->rank;
        da.n_q = lora->n_q;
        da.n_kv = lora->n_kv;
        da.lora_planes = lora->planes;
        da.tile_slot_mask = lora->tile_slot_mask;
      }
      return MN == 16 ? launch_dec<16>(tw, tx, tu, tsm, da, st) : launch_dec<32>(tw, tx, tu, tsm, da, st);
    }
  }
  static const bool no_ws = getenv("ALORA_GEMM_NO_WS") != nullptr;  // A/B switch to the per-tile kernel
  if (M <= 2 * kBM && !no_ws) {
    // weight streaming: one CTA per (N tile, K split) covering every token row
    const int mt = (M + kBM - 1) / kBM;
    const bool can_defer = !g_batch_invariant && defer != nullptr && defer->partial != nullptr && !(epi & 16) &&
                           (base_epi == kEpiAdd || base_epi == kEpiRope || base_epi == kEpiLoraSelect);
    const int64_t defer_cap = can_defer ? defer->capacity : 0;
    WsChoice best;
    auto consider = [&](int bn) {
      if (!fits(bn) || mt * bn > 512) return;
      if (mt == 1) {
        switch (bn) {
          case 256: ws_consider<256, 1>(best, M, N, K, can_defer, defer_cap); break;
          case 128: ws_consider<128, 1>(best, M, N, K, can_defer, defer_cap); break;
          case 64: ws_consider<64, 1>(best, M, N, K, can_defer, defer_cap); break;
          default: ws_consider<32, 1>(best, M, N, K, can_defer, defer_cap);
        }
      } else {
        switch (bn) {
          case 256: ws_consider<256, 2>(best, M, N, K, can_defer, defer_cap); break;
          case 128: ws_consider<128, 2>(best, M, N, K, can_defer, defer_cap); break;
          case 64: ws_consider<64, 2>(best, M, N, K, can_defer, defer_cap); break;
          default: ws_consider<32, 2>(best, M, N, K, can_defer, defer_cap);
        }
      }
    };
    for (int bn : {256, 128, 64, 32}) consider(bn);
    static const int force_bn = getenv("ALORA_WS_BN") ? atoi(getenv("ALORA_WS_BN")) : 0;  // debug overrides
    static const int force_s = getenv("ALORA_WS_S") ? atoi(getenv("ALORA_WS_S")) : 0;
    if (force_bn > 0 && fits(force_bn) && mt * force_bn <= 512) best.bn = force_bn;
    if (force_s > 0 && (force_s == 1 || can_defer)) best.splits = force_s;
    if (g_batch_invariant) best.splits = 1;  // one K range: the row's sum order never depends on the step
    if (best.bn > 0) {
      if (base_epi == kEpiRope && (lora->rope_cols % best.bn || best.bn % lora->head_dim)) return ALORA_EINVAL;
      CUtensorMap tb2, tu2 = tu;
      if (!make_tmap_2d(&tb2, Bt, N, K, ldb, best.bn, kBK)) return ALORA_ECUDA;
      if (args.ks > 0 && !make_tmap_2d(&tu2, lora->up_t, N, lora->ks * up_planes, lora->ks * up_planes, best.bn, kBK))
        return ALORA_ECUDA;
      if (args.ks == 0) tu2 = tb2;
      args.splits = best.splits;
      if (best.splits > 1) {
        if (!can_defer) return ALORA_EINVAL;
        args.partial = defer->partial;
        defer->splits_out = best.splits;
        defer->deferred = true;
      }
      return mt == 1 ? dispatch_ws<1>(ta, tb2, ts, tu2, args, best.bn, st)
                     : dispatch_ws<2>(ta, tb2, ts, tu2, args, best.bn, st);
    }
  }
  // split K when the tile grid cannot fill the machine (weight-streaming small-M launches): the largest
  // split count with tiles * splits <= 148 (one co-resident CTA per SM) and >= 4 K-blocks per split
  const int m_tiles = (M + kBM - 1) / kBM;
  const int tiles = m_tiles * (N / BN);
  const int nkb = (K + kBK - 1) / kBK;
  int splits = 1;
  if (ws != nullptr && ws->partial != nullptr && tiles * 2 <= kNumSMs) {
    splits = std::min({max_splits, kMaxSplits, kNumSMs / tiles, nkb / 4});
    splits = std::max(1, splits);
    const int per = (nkb + splits - 1) / splits;
    splits = (nkb + per - 1) / per;  // no empty trailing splits
    if ((int64_t)splits * m_tiles * kBM * N * 4 > ws->partial_bytes || 2 * tiles > ws->n_counters) splits = 1;
  }
  args.splits = splits;
  if (splits > 1) {
    args.partial = static_cast<float*>(ws->partial);
    args.counters = ws->counters;
  }
  if (splits == 1 && base_epi == kEpiRope && lora && lora->kv_pool && lora->kv_slots && lora->kv_w % 32 == 0 &&
      lora->kv_q % 32 == 0 && lora->kv_block > 0 && defer) {
    args.kv_pool = lora->kv_pool;
    args.kv_slots = lora->kv_slots;
    args.kv_q = lora->kv_q;
    args.kv_w = lora->kv_w;
    args.kv_layer = lora->kv_layer;
    args.kv_layers = lora->kv_layers;
    args.kv_block = lora->kv_block;
    defer->kv_written = true;
  }
  static const bool no_persist = getenv("ALORA_GEMM_NO_PERSIST") != nullptr;  // A/B switch
  if (splits == 1 && !no_persist && tiles > kNumSMs) {  // several tiles per SM: overlap epilogues with MMAs
    switch (BN) {
      case 256: return launch_persist<256>(ta, tb, ts, tu, args, st);
      case 128: return launch_persist<128>(ta, tb, ts, tu, args, st);
      case 64: return launch_persist<64>(ta, tb, ts, tu, args, st);
      default: return launch_persist<32>(ta, tb, ts, tu, args, st);
    }
  }
  switch (BN) {
    case 256: return launch<256>(ta, tb, ts, tu, args, st);
    case 128: return launch<128>(ta, tb, ts, tu, args, st);
    case 64: return launch<64>(ta, tb, ts, tu, args, st);
    default: return launch<32>(ta, tb, ts, tu, args, st);
  }
}

int64_t gemm_bf16_workspace_bytes() {
  // splits * m_tiles <= 148 partial tile rows of 128 x N(<= 148 * 128 cols per split group) fp32, plus counters
  return (int64_t)kNumSMs * kBM * 128 * 4 + (int64_t)kGemmCounters * 4;
}

}  // namespace alora
