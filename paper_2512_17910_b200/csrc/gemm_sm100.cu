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
// Structure (one 128 x BN output tile per CTA, 192 threads):
//   warp 0      TMA producer: A/B (or S/U) 64-wide K slabs -> smem ring (SW128)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 cols -> fused epilogue -> global
// mbarrier ring: full[s] (TMA tx bytes) / empty[s] (tcgen05.commit), tmem_full.
// Each output element accumulates its K range in a fixed order (no split-K):
// the result of a row does not depend on M or on its neighbours.

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

struct GemmArgs {
  void* C;
  int ldc;
  int M, N, K;
  int epi;        // Epi | 16 => fp32 output for kEpiStore
  int ks;         // LoRA K (n_slots * rank), 0 = none
  int rank;
  int n_q, n_kv;  // q | k | v column ranges
  const uint32_t* tile_slot_mask;
  const int32_t* positions;  // kEpiRope
  const float* rope_cos;
  const float* rope_sin;
  int rope_cols, head_dim;
};

template <int BN>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStage) > 8 ? 8 : (kSmemBudget / kStage);
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kSmem = 1024 + kStages * kStage + 256;
};

// LoRA K-block j covers slots [j*64/R, ((j+1)*64-1)/R]; present if any of them is in the tile mask.
__device__ __forceinline__ bool lora_block_present(int j, int rank, uint32_t mask) {
  const int s0 = (j * kBK) / rank, s1 = (j * kBK + kBK - 1) / rank;
  for (int s = s0; s <= s1 && s < 32; ++s)
    if ((mask >> s) & 1u) return true;
  return false;
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_u,
                     const GemmArgs args) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m_tile = blockIdx.y, m0 = m_tile * kBM;
  const int nkb = (args.K + kBK - 1) / kBK;
  // LoRA range of this N tile
  int target = 0, nkl = 0;
  uint32_t mask = 0;
  if (args.ks > 0) {
    target = n0 < args.n_q ? 0 : (n0 < args.n_q + args.n_kv ? 1 : 2);
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

  if (warp == 0) {
    if (sm100::elect_one()) {
      const uint64_t pol_act = sm100::policy_evict_last();   // activations: re-read by every N tile
      const uint64_t pol_w = sm100::policy_evict_first();    // weights: streamed once per forward
      int s = 0;
      uint32_t phase = 0;
      auto next = [&] { if (++s == C::kStages) { s = 0; phase ^= 1; } };
      for (int kb = 0; kb < nkb; ++kb) {
        sm100::mbar_wait(&empty[s], phase ^ 1);
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_2d(sa, &tm_a, &full[s], kb * kBK, m0, pol_act);
        sm100::tma_load_2d(sa + C::kABytes, &tm_b, &full[s], kb * kBK, n0, pol_w);
        next();
      }
      for (int j = 0; j < nkl; ++j) {
        if (!lora_block_present(j, args.rank, mask)) continue;
        sm100::mbar_wait(&empty[s], phase ^ 1);
        uint8_t* sa = smem + s * C::kStage;
        sm100::mbar_arrive_expect_tx(&full[s], C::kStage);
        sm100::tma_load_3d(sa, &tm_s, &full[s], j * kBK, m0, target, pol_act);
        sm100::tma_load_2d(sa + C::kABytes, &tm_u, &full[s], j * kBK, n0, pol_w);
        next();
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
      int s = 0;
      uint32_t phase = 0;
      uint32_t acc = 0;
      auto consume = [&] {
        sm100::mbar_wait(&full[s], phase);
        sm100::tc_fence_after();
        const uint8_t* sa = smem + s * C::kStage;
        const uint64_t da = sm100::umma_desc_sw128(sa);
        const uint64_t db = sm100::umma_desc_sw128(sa + C::kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {  // +32 bytes per K=16 step inside the 128B swizzle atom
          sm100::mma_bf16_ss(tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, acc);
          acc = 1;
        }
        sm100::mma_commit(&empty[s]);
        if (++s == C::kStages) { s = 0; phase ^= 1; }
      };
      for (int kb = 0; kb < nkb; ++kb) consume();
      for (int j = 0; j < nkl; ++j)
        if (lora_block_present(j, args.rank, mask)) consume();
      sm100::mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // epilogue: warp w owns TMEM lanes [32*(w%4), +32) = tile rows
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    sm100::mbar_wait(tmem_full, 0);
    sm100::tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const int epi = args.epi & 15;
    const bool out_f32 = (args.epi & 16) != 0;
    const bool live = row < args.M;
    if (epi == kEpiRope && n0 < args.rope_cols) {
      // q/k heads: x1 = cols [i*32, +32), x2 = cols [half + i*32, +32) of each head; fp32 rotate, one bf16 rounding
      const int D = args.head_dim, half = D / 2;
      const int pos = live ? args.positions[row] : 0;
      const float* cs = args.rope_cos + (int64_t)pos * half;
      const float* sn = args.rope_sin + (int64_t)pos * half;
      for (int hb = 0; hb < BN; hb += D) {
        for (int i = 0; i < half / 32; ++i) {
          uint32_t x1[32], x2[32];
          sm100::tmem_ld_32x32b_x32(trow + hb + i * 32, x1);
          sm100::tmem_ld_32x32b_x32(trow + hb + half + i * 32, x2);
          sm100::tmem_ld_wait();
          if (!live) continue;
          __nv_bfloat16* d1 = static_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc + n0 + hb + i * 32;
          __nv_bfloat16* d2 = d1 + half;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            __align__(16) __nv_bfloat162 o1[4], o2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float r1[2], r2[2];
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int j = v * 8 + e * 2 + q;
                const float c = __ldg(cs + i * 32 + j), s = __ldg(sn + i * 32 + j);
                const float a = __uint_as_float(x1[j]), b = __uint_as_float(x2[j]);
                r1[q] = a * c - b * s;
                r2[q] = b * c + a * s;
              }
              o1[e] = __floats2bfloat162_rn(r1[0], r1[1]);
              o2[e] = __floats2bfloat162_rn(r2[0], r2[1]);
            }
            *reinterpret_cast<int4*>(d1 + v * 8) = *reinterpret_cast<int4*>(o1);
            *reinterpret_cast<int4*>(d2 + v * 8) = *reinterpret_cast<int4*>(o2);
          }
        }
      }
    } else if (epi == kEpiSwiglu) {
      // tile columns [0,64) gate, [64,128) up -> 64 outputs at column n0/2
      for (int c = 0; c < BN / 128; ++c) {
        for (int h = 0; h < 2; ++h) {
          uint32_t g[32], u[32];
          sm100::tmem_ld_32x32b_x32(trow + c * 128 + h * 32, g);
          sm100::tmem_ld_32x32b_x32(trow + c * 128 + 64 + h * 32, u);
          sm100::tmem_ld_wait();
          if (live) {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc + n0 / 2 + c * 64 + h * 32;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              __align__(16) __nv_bfloat162 o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int i = v * 8 + e * 2;
                const float a0 = silu(__uint_as_float(g[i])) * __uint_as_float(u[i]);
                const float a1 = silu(__uint_as_float(g[i + 1])) * __uint_as_float(u[i + 1]);
                o[e] = __floats2bfloat162_rn(a0, a1);
              }
              *reinterpret_cast<int4*>(dst + v * 8) = *reinterpret_cast<int4*>(o);
            }
          }
        }
      }
    } else {
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(trow + c * 32, r);
        sm100::tmem_ld_wait();
        if (!live) continue;
        const int col = n0 + c * 32;
        if (col >= args.N) continue;
        if (epi == kEpiAdd) {
          float* dst = static_cast<float*>(args.C) + (int64_t)row * args.ldc + col;
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 x = *reinterpret_cast<float4*>(dst + v * 4);
            x.x += __uint_as_float(r[v * 4 + 0]);
            x.y += __uint_as_float(r[v * 4 + 1]);
            x.z += __uint_as_float(r[v * 4 + 2]);
            x.w += __uint_as_float(r[v * 4 + 3]);
            *reinterpret_cast<float4*>(dst + v * 4) = x;
          }
        } else if (out_f32) {
          float* dst = static_cast<float*>(args.C) + (int64_t)row * args.ldc + col;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<float4*>(dst + v * 4) =
                make_float4(__uint_as_float(r[v * 4]), __uint_as_float(r[v * 4 + 1]), __uint_as_float(r[v * 4 + 2]),
                            __uint_as_float(r[v * 4 + 3]));
        } else {
          __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc + col;
          const bool relu = epi == kEpiRelu;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            __align__(16) __nv_bfloat162 o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float a0 = __uint_as_float(r[v * 8 + e * 2]), a1 = __uint_as_float(r[v * 8 + e * 2 + 1]);
              if (relu) { a0 = fmaxf(a0, 0.f); a1 = fmaxf(a1, 0.f); }
              o[e] = __floats2bfloat162_rn(a0, a1);
            }
            *reinterpret_cast<int4*>(dst + v * 8) = *reinterpret_cast<int4*>(o);
          }
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<C::kTmemCols>(tmem);
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
  dim3 grid((args.N + BN - 1) / BN, (args.M + kBM - 1) / kBM);
  gemm_bf16_kernel<BN><<<grid, kThreads, C::kSmem, st>>>(a, b, s, u, args);
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace

int gemm_bf16(int epi, const __nv_bfloat16* A, int lda, const __nv_bfloat16* Bt, int ldb, void* Cout, int ldc, int M,
              int N, int K, const GemmLora* lora, cudaStream_t st) {
  if (M == 0 || N == 0) return ALORA_OK;
  if (M < 0 || N < 0 || K < 1 || lda % 8 || ldb % 8 || ldc % 8) return ALORA_EINVAL;
  const int base_epi = epi & 15;
  int BN = (N % 128 == 0) ? 128 : 64;
  if (N % 64 != 0) return ALORA_EINVAL;
  if (base_epi == kEpiSwiglu && N % 128 != 0) return ALORA_EINVAL;
  if (base_epi == kEpiSwiglu) BN = 128;
  GemmArgs args{Cout, ldc, M, N, K, epi, 0, 1, 0, 0, nullptr, nullptr, nullptr, nullptr, 0, 0};
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
  CUtensorMap ta, tb, ts, tu;
  if (!make_tmap_2d(&ta, A, M, K, lda, kBM, kBK)) return ALORA_ECUDA;
  if (!make_tmap_2d(&tb, Bt, N, K, ldb, BN, kBK)) return ALORA_ECUDA;
  ts = ta;
  tu = tb;
  if (lora != nullptr && lora->s != nullptr && lora->ks > 0) {
    if (lora->ks % 8 || (lora->n_q % BN) || (lora->n_kv % BN) || lora->rank < 1) return ALORA_EINVAL;
    if (!make_tmap_3d(&ts, lora->s, 3, M, lora->ks, kBM, kBK)) return ALORA_ECUDA;
    if (!make_tmap_2d(&tu, lora->up_t, N, lora->ks, lora->ks, BN, kBK)) return ALORA_ECUDA;
    args.ks = lora->ks;
    args.rank = lora->rank;
    args.n_q = lora->n_q;
    args.n_kv = lora->n_kv;
    args.tile_slot_mask = lora->tile_slot_mask;
  }
  return BN == 128 ? launch<128>(ta, tb, ts, tu, args, st) : launch<64>(ta, tb, ts, tu, args, st);
}

}  // namespace alora
