// Paged causal prefill attention, bf16 tier (model.py:149-187 generalised to GQA).
//
// Work item = (sequence, kv head, 128-row query tile, KV partition). Query rows
// are GQA-packed: row r of a sequence's tile space is (token r / G, q head
// kvh*G + r % G), so one K/V tile read from HBM serves all G query heads that
// share it. A CTA runs 8 warps of 16 rows; only ceil(rows/16) warps compute, so
// a 20-token aLoRA suffix (80 packed rows at G=4) costs 5 warps, not two full
// 64-row tiles. K/V tiles of 64 keys are gathered page by page through the
// block table with cp.async (one table lookup per key row, 16-byte chunks,
// XOR-swizzled smem rows, 3-stage ring); QK^T and PV use mma.sync m16n8k16 bf16
// with fp32 accumulation and an fp32 online softmax (ex2.approx). Causal masks
// are evaluated only on tiles that cross the diagonal or the partition end.
//
// When a step has too few work items to fill the 148 SMs (the aLoRA suffix turn
// and decode: few query rows, long cached prefix) the key range is split into
// partitions; each partition CTA publishes (m, l, O) partials and the last one
// to arrive for a query tile merges them in partition order (deterministic),
// so no separate combine kernel runs.

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

constexpr int kQT = 128;      // packed query rows per CTA (8 warps x 16)
constexpr int kKT = 64;       // keys per KV tile
constexpr int kThreadsA = 256;
constexpr int kTargetCtas = 2 * kNumSMs;  // two resident CTAs per SM
constexpr int kStagesA = 3;               // cp.async ring depth for K/V tiles
constexpr int kMinPartKeys = 128;
constexpr int kMaxCounters = 4096;
constexpr int kMaxParts = 8;  // split-KV partitions per query tile (merge keeps them all in registers)

struct AttnArgs {
  const __nv_bfloat16* q;
  int64_t ld_q;
  const int32_t* cu_q;
  const int32_t* start_pos;
  const int32_t* block_table;
  int max_blocks;
  const __nv_bfloat16* kv;
  int n_layers, layer, B, H, Hkv, D;
  float scale_log2;  // log2(e) / sqrt(D)
  int part_size;     // keys per partition (multiple of kKT)
  int n_parts;
  int n_qtiles;      // gridDim.x
  __nv_bfloat16* out;
  int64_t ld_out;
  float* ws_o;   // [n_parts][M*H][D] when split
  float* ws_ml;  // [n_parts][M*H][2]
  int* counters; // [n_seqs * Hkv * n_qtiles], zero between launches
  unsigned long long* trace;  // optional per-CTA %globaltimer stamps (ALORA_ATTN_TRACE=1)
  int M;
  int exp;  // debug experiments (ALORA_ATTN_EXP): 3 = softmax skips its math (timing only)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// shared-window address form: no generic->shared conversion per copy
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
// arrive on an mbarrier once every cp.async this thread issued so far has completed (no pending-count increment:
// the barrier's expected count includes this arrival)
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 2^x on the SFU (ex2.approx.ftz): exp2(-inf) = +0, as the softmax needs for masked keys.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// paired fp32 arithmetic (sm_100 FFMA2 / FADD2 on a 64-bit register pair)
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled [rows][D] bf16 tile: 16-byte chunk c of row r lives at chunk (c ^ (r & 7)).
template <int D>
__device__ __forceinline__ __nv_bfloat16* tile_ptr(__nv_bfloat16* base, int row, int col) {
  constexpr int chunks = D / 8;
  const int c = (col >> 3) ^ (row & 7);
  return base + row * D + ((c & (chunks - 1)) << 3) + (col & 7);
}

template <int D>
__device__ void merge_partials(const AttnArgs& a, int s, int kvh, int qt, int row0, int start, int rows_here,
                               int parts_here, int G, int* s_last);

template <int D>
__global__ void __launch_bounds__(kThreadsA, D == 64 ? 2 : 1) attn_bf16_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_attn[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sK = sQ + kQT * D;             // [kStagesA][kKT][D]
  __nv_bfloat16* sV = sK + kStagesA * kKT * D;  // [kStagesA][kKT][D]
  __shared__ int s_last;

  const int G = a.H / a.Hkv;
  const int s = blockIdx.z / a.Hkv, kvh = blockIdx.z % a.Hkv;
  const int qt = blockIdx.x, part = blockIdx.y;
  const int row0 = a.cu_q[s];
  const int n_tok = a.cu_q[s + 1] - row0;
  const int R = n_tok * G;
  if (qt * kQT >= R) return;
  const int rows_here = min(kQT, R - qt * kQT);
  const int start = a.start_pos[s];
  const int last_tok = (qt * kQT + rows_here - 1) / G;
  const int tile_end = start + last_tok + 1;  // exclusive key bound of the whole tile
  const int key_begin = part * a.part_size;
  const int key_end = min(tile_end, key_begin + a.part_size);
  if (key_begin >= key_end) return;  // nothing visible in this partition for any row of the tile
  const int parts_here = min(a.n_parts, (tile_end + a.part_size - 1) / a.part_size);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool active = warp * 16 < rows_here;  // warp-uniform
  const int kvw = a.Hkv * D;
  const int32_t* bt = a.block_table + (int64_t)s * a.max_blocks;
  constexpr int CH = D / 8;  // 16-byte chunks per row

  // ---- Q tile (packed rows) -> smem
  for (int i = tid; i < kQT * CH; i += kThreadsA) {
    const int r = i / CH, c = i % CH;
    const bool valid = r < rows_here;
    const int pr = qt * kQT + r;
    const int tok = valid ? pr / G : 0, g = valid ? pr % G : 0;
    const __nv_bfloat16* src = a.q + (int64_t)(row0 + tok) * a.ld_q + (kvh * G + g) * D + c * 8;
    cp_async16(tile_ptr<D>(sQ, r, c * 8), valid ? src : a.q, valid);
  }
  // K/V loader: thread owns key row tid/4 and a quarter of its chunks (one block-table lookup per row)
  const int lrow = tid >> 2, lq = tid & 3;
  const int64_t vstep = (int64_t)a.B * kvw;
  auto load_kv = [&](int buf, int k0) {
    __nv_bfloat16* dk = sK + buf * kKT * D;
    __nv_bfloat16* dv = sV + buf * kKT * D;
    const int t = k0 + lrow;
    const bool valid = t < key_end;
    const __nv_bfloat16* ksrc = a.kv;
    if (valid) {
      const int bi = t / a.B;
      const int64_t blk = bt[bi];
      ksrc = a.kv + ((((blk * a.n_layers + a.layer) * 2) * a.B + (t - bi * a.B)) * (int64_t)kvw) + kvh * D;
    }
#pragma unroll
    for (int cc = 0; cc < CH / 4; ++cc) {
      const int c = lq * (CH / 4) + cc;
      cp_async16(tile_ptr<D>(dk, lrow, c * 8), valid ? ksrc + c * 8 : a.kv, valid);
      cp_async16(tile_ptr<D>(dv, lrow, c * 8), valid ? ksrc + vstep + c * 8 : a.kv, valid);
    }
  };
  const int n_tiles = (key_end - key_begin + kKT - 1) / kKT;
#pragma unroll
  for (int p = 0; p < kStagesA - 1; ++p) {  // prologue (Q rides with tile 0's group)
    if (p < n_tiles) load_kv(p, key_begin + p * kKT);
    cp_async_commit();
  }

  // per-thread rows: lane/4 and lane/4 + 8 of this warp's 16-row slice
  const int wr = warp * 16;
  int pos_r[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = wr + (lane >> 2) + h * 8;
    pos_r[h] = r < rows_here ? start + (qt * kQT + r) / G : -1;
  }
  const int min_pos = start + (qt * kQT + wr) / G;  // this warp's first row sees the fewest keys
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  uint32_t qf[D / 16][4];
  // Per-lane swizzled smem offsets (elements) of the ldmatrix rows: the XOR pattern depends only on the lane
  // because every fragment row block starts at a multiple of 8 rows.
  int koff[D / 16], voff[D / 16];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    koff[kk] = ((lane & 7) + (lane >> 4) * 8) * D + (((kk * 2 + ((lane >> 3) & 1)) ^ (lane & 7)) << 3);
    voff[kk] = (lane & 15) * D + (((kk * 2 + (lane >> 4)) ^ (lane & 7)) << 3);
  }

  for (int it = 0; it < n_tiles; ++it) {
    const int k0 = key_begin + it * kKT;
    cp_async_wait<kStagesA - 2>();  // tile `it` has landed
    __syncthreads();                // ... for every thread, and buffer (it-1) % kStagesA is free again
    if (it + kStagesA - 1 < n_tiles) load_kv((it + kStagesA - 1) % kStagesA, k0 + (kStagesA - 1) * kKT);
    cp_async_commit();
    if (!active) continue;
    if (it == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ldsm_x4(qf[kk], tile_ptr<D>(sQ, wr + (lane & 15), kk * 16 + (lane >> 4) * 8));
    }
    const __nv_bfloat16* cK = sK + (it % kStagesA) * kKT * D;
    const __nv_bfloat16* cV = sV + (it % kStagesA) * kKT * D;
    // S = Q K^T  (16 x 64 per warp)
    float sc[kKT / 8][4];
#pragma unroll
    for (int j = 0; j < kKT / 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int jn = 0; jn < kKT / 16; ++jn) {
        uint32_t b[4];
        ldsm_x4(b, cK + jn * 16 * D + koff[kk]);
        mma16816(sc[2 * jn], qf[kk], b[0], b[1]);
        mma16816(sc[2 * jn + 1], qf[kk], b[2], b[3]);
      }
    }
    // mask (only tiles crossing this warp's causal edge or the partition end) + online softmax (log2)
    const bool need_mask = (k0 + kKT - 1 > min_pos) || (k0 + kKT > key_end);
    float mnew[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float mx = m_r[h];
      const int lim = min(pos_r[h], key_end - 1);
#pragma unroll
      for (int j = 0; j < kKT / 8; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float v = sc[j][h * 2 + e] * a.scale_log2;
          if (need_mask && (k0 + j * 8 + 2 * (lane & 3) + e > lim)) v = -INFINITY;
          sc[j][h * 2 + e] = v;
          mx = fmaxf(mx, v);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[h] = mx;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float base = mnew[h] == -INFINITY ? 0.f : mnew[h];
      const float corr = fast_exp2(m_r[h] - base);
#pragma unroll
      for (int j = 0; j < D / 8; ++j) { o[j][h * 2] *= corr; o[j][h * 2 + 1] *= corr; }
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < kKT / 8; ++j) {
        sc[j][h * 2] = fast_exp2(sc[j][h * 2] - base);
        sc[j][h * 2 + 1] = fast_exp2(sc[j][h * 2 + 1] - base);
        rs += sc[j][h * 2] + sc[j][h * 2 + 1];
      }
      l_r[h] = l_r[h] * corr + rs;
      m_r[h] = mnew[h];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(sc[2 * kk][0], sc[2 * kk][1]);
      pa[1] = pack_bf16(sc[2 * kk][2], sc[2 * kk][3]);
      pa[2] = pack_bf16(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
      pa[3] = pack_bf16(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
      for (int jd = 0; jd < D / 16; ++jd) {
        uint32_t b[4];
        ldsm_x4_t(b, cV + kk * 16 * D + voff[jd]);
        mma16816(o[2 * jd], pa, b[0], b[1]);
        mma16816(o[2 * jd + 1], pa, b[2], b[3]);
      }
    }
  }
  cp_async_wait<0>();
  if (active) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // full row sums across the 4 lanes of a quad
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wr + (lane >> 2) + h * 8;
      if (r >= rows_here || pos_r[h] < key_begin) continue;
      const int pr = qt * kQT + r;
      const int tok = pr / G, head = kvh * G + pr % G;
      const int64_t grow = row0 + tok;
      if (parts_here == 1) {
        const float inv = 1.f / l_r[h];
        __nv_bfloat16* dst = a.out + grow * a.ld_out + head * D;
#pragma unroll
        for (int j = 0; j < D / 8; ++j)
          *reinterpret_cast<__nv_bfloat162*>(dst + j * 8 + 2 * (lane & 3)) =
              __floats2bfloat162_rn(o[j][h * 2] * inv, o[j][h * 2 + 1] * inv);
      } else {
        const int64_t slot = ((int64_t)part * a.M + grow) * a.H + head;
        float* dst = a.ws_o + slot * D;
#pragma unroll
        for (int j = 0; j < D / 8; ++j)
          __stcg(reinterpret_cast<float2*>(dst + j * 8 + 2 * (lane & 3)), make_float2(o[j][h * 2], o[j][h * 2 + 1]));
        if ((lane & 3) == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml + slot * 2), make_float2(m_r[h], l_r[h]));
      }
    }
  }
  if (parts_here == 1) return;
  merge_partials<D>(a, s, kvh, qt, row0, start, rows_here, parts_here, G, &s_last);
}

// Last partition CTA to arrive for query tile (s, kvh, qt) merges the partials in partition order.
// Called by every thread of the CTA after its own partials are stored.
template <int D>
__device__ void merge_partials(const AttnArgs& a, int s, int kvh, int qt, int row0, int start, int rows_here,
                               int parts_here, int G, int* s_last) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  __syncthreads();  // CTA-scope: every thread's partial stores happen-before thread 0's cumulative gpu fence
  int* ctr = a.counters + ((int64_t)s * a.Hkv + kvh) * a.n_qtiles + qt;
  if (tid == 0) {
    __threadfence();
    const int prev = atomicAdd(ctr, 1);
    *s_last = prev == parts_here - 1;
    if (*s_last) {
      *ctr = 0;  // ready for the next launch
      __threadfence();
    }
  }
  __syncthreads();
  if (!*s_last) return;
  constexpr int G8 = D / 8;
  const int n_items = rows_here * G8;
  if (parts_here <= 4) {
  // two work items per thread per round: all partial loads of both are in flight before any is consumed
  // (the merge is a chain of L2 round trips on the kernel's tail)
  for (int i0 = tid; i0 < n_items; i0 += 2 * nthr) {
    float2 ml[2][4];
    float4 x0[2][4], x1[2][4];
    int64_t grow2[2];
    int head2[2], c82[2], np2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * nthr;
      np2[u] = 0;
      if (i >= n_items) continue;
      const int r = i / G8, c8 = (i % G8) * 8;
      const int pr = qt * kQT + r;
      const int tok = pr / G, head = kvh * G + pr % G;
      const int64_t grow = row0 + tok;
      const int np_row = min(parts_here, (start + tok) / a.part_size + 1);
      grow2[u] = grow;
      head2[u] = head;
      c82[u] = c8;
      np2[u] = np_row;
      const int64_t slot0 = (int64_t)grow * a.H + head, pstride = (int64_t)a.M * a.H;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (p < np_row) {
          ml[u][p] = __ldcg(reinterpret_cast<const float2*>(a.ws_ml + (slot0 + p * pstride) * 2));
          x0[u][p] = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8));
          x1[u][p] = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8 + 4));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int np_row = np2[u];
      if (np_row == 0) continue;
      float mx = -INFINITY;
#pragma unroll
      for (int p = 0; p < 4; ++p)
        if (p < np_row) mx = fmaxf(mx, ml[u][p].x);
      float l = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int p = 0; p < 4; ++p) {  // partition order: deterministic
        if (p >= np_row) break;
        const float w = fast_exp2(ml[u][p].x - mx);
        l += w * ml[u][p].y;
        acc[0] += w * x0[u][p].x; acc[1] += w * x0[u][p].y; acc[2] += w * x0[u][p].z; acc[3] += w * x0[u][p].w;
        acc[4] += w * x1[u][p].x; acc[5] += w * x1[u][p].y; acc[6] += w * x1[u][p].z; acc[7] += w * x1[u][p].w;
      }
      const float inv = __fdividef(1.f, l);
      __align__(16) __nv_bfloat162 ov[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) ov[e] = __floats2bfloat162_rn(acc[2 * e] * inv, acc[2 * e + 1] * inv);
      *reinterpret_cast<int4*>(a.out + grow2[u] * a.ld_out + head2[u] * D + c82[u]) = *reinterpret_cast<int4*>(ov);
    }
  }
    return;
  }
  for (int i = tid; i < n_items; i += nthr) {
    const int r = i / G8, c8 = (i % G8) * 8;
    const int pr = qt * kQT + r;
    const int tok = pr / G, head = kvh * G + pr % G;
    const int64_t grow = row0 + tok;
    const int np_row = min(parts_here, (start + tok) / a.part_size + 1);
    const int64_t slot0 = (int64_t)grow * a.H + head, pstride = (int64_t)a.M * a.H;
    float2 ml[kMaxParts];
    float4 x0[kMaxParts], x1[kMaxParts];
#pragma unroll
    for (int p = 0; p < kMaxParts; ++p) {
      ml[p] = p < np_row ? __ldcg(reinterpret_cast<const float2*>(a.ws_ml + (slot0 + p * pstride) * 2))
                         : make_float2(-INFINITY, 0.f);
      if (p < np_row) {
        x0[p] = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8));
        x1[p] = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8 + 4));
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int p = 0; p < kMaxParts; ++p) mx = fmaxf(mx, ml[p].x);
    float l = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int p = 0; p < kMaxParts; ++p) {  // partition order: deterministic
      if (p >= np_row) break;
      const float w = fast_exp2(ml[p].x - mx);
      l += w * ml[p].y;
      acc[0] += w * x0[p].x; acc[1] += w * x0[p].y; acc[2] += w * x0[p].z; acc[3] += w * x0[p].w;
      acc[4] += w * x1[p].x; acc[5] += w * x1[p].y; acc[6] += w * x1[p].z; acc[7] += w * x1[p].w;
    }
    const float inv = __fdividef(1.f, l);
    __align__(16) __nv_bfloat162 ov[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) ov[e] = __floats2bfloat162_rn(acc[2 * e] * inv, acc[2 * e + 1] * inv);
    *reinterpret_cast<int4*>(a.out + grow * a.ld_out + head * D + c8) = *reinterpret_cast<int4*>(ov);
  }
}

// ============================================================================================================
// tcgen05 variant: QK^T and PV on the 5th-gen tensor cores with S and O accumulated in TMEM.
//   warps 0-3  softmax: thread = query row = TMEM lane; tcgen05.ld its 64 scores per tile, online softmax
//              (lazy rescale: O in TMEM is rescaled only when the row max grows by > 2^8), P -> smem (SW128)
//   warp 4     producer: Q once (cp.async gather of the GQA-packed rows), then K/V tiles of 64 keys as TMA
//              boxes of [B keys x 64 dims], one per page (the block table is the gather index), 4-stage ring
//   warp 5     TMEM allocator + single-thread MMA issuer: S_t = Q K_t^T (M=128, N=64), O += P_t V_t (N=D,
//              V as an MN-major operand), S double-buffered so S_{t+1} overlaps softmax_t.
// Operands live in 64-column (128-byte) swizzled sub-tiles: [D/64][rows][64] bf16.
// ============================================================================================================
namespace tc {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ATTN_TRACE(slot)                                                                                    \
  do {                                                                                                      \
    if (a.trace) a.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 6 + (slot)] = gtimer(); \
  } while (0)

// K/V ring depth. A stage is held from its TMA issue until PV of its tile completes (TMA latency + S MMA +
// softmax + PV, ~2-3 us under load), so the per-tile period is that cycle over kNS. P lives in TMEM (written
// over the S columns it came from), which leaves the smem to K/V: 5 stages at ~97 KB per CTA for D=64, so
// two CTAs (two independent softmax chains) still share an SM.
template <int D>
constexpr int kNS = 5;
// S runs two tiles ahead of the softmax (three S buffers in TMEM). P_t overwrites the first 32 columns of
// its S buffer, which the MMA warp reuses for S_{t+3} only after issuing PV_t (tcgen05.mma from one thread
// execute in issue order), so neither warp waits on the other's previous step.
constexpr int kSBuf = 3;
constexpr int kThreads = 192;   // 4 softmax + 1 producer + 1 MMA warps
constexpr float kRescaleLog2 = 8.f;

template <int D>
struct Smem {
  static constexpr int kQBytes = kQT * D * 2;        // [D/64][128][64]
  static constexpr int kKVBytes = kKT * D * 2;       // one K (or V) tile [D/64][64][64]
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;
  static constexpr int kV = kK + kNS<D> * kKVBytes;
  static constexpr int kBar = kV + kNS<D> * kKVBytes;
  static constexpr int kTotal = kBar + 256 + 1024;  // barriers + TMEM slot + alignment slack
};

// byte offset of (row, 16B chunk c) inside a [D/64][rows][64] swizzled operand
__device__ __forceinline__ uint32_t sw_off(int row, int c, int rows) {
  return (uint32_t)((c >> 3) * rows * 128 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

template <int D>
__global__ void __launch_bounds__(kThreads, D == 64 ? 2 : 1) attn_tc_kernel(const AttnArgs a,
                                                              const __grid_constant__ CUtensorMap tm_kv) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw_tc[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_tc) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kBar);
  uint64_t* q_full = bars;             // 1
  uint64_t* kv_full = bars + 1;        // kNS<D>
  uint64_t* kv_empty = kv_full + kNS<D>;  // kNS<D>
  uint64_t* s_full = kv_empty + kNS<D>;   // kSBuf
  // p_full[t % 3]: P_t is in TMEM. Three deep like S: softmax_{t+3} needs S_{t+3}, which needs PV_t complete,
  // so a P barrier can never run a phase ahead of the MMA warp's parity test.
  uint64_t* p_full = s_full + kSBuf;   // kSBuf
  // s_free[i]: PV of the P held in S buffer i has completed (one phase per use of the buffer). It is also
  // the softmax's "O holds PV_t" signal: the previous phase on s_free[t % 3] (PV_{t-3}) always completed
  // before S_t was issued, so a parity wait on it can never match a stale phase (a 2-deep PV barrier could).
  uint64_t* s_free = p_full + kSBuf;   // kSBuf
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + kSBuf);
  __shared__ int s_last;

  const int G = a.H / a.Hkv;
  const int s = blockIdx.z / a.Hkv, kvh = blockIdx.z % a.Hkv;
  const int qt = blockIdx.x, part = blockIdx.y;
  const int row0 = a.cu_q[s];
  const int n_tok = a.cu_q[s + 1] - row0;
  const int R = n_tok * G;
  if (qt * kQT >= R) return;
  const int rows_here = min(kQT, R - qt * kQT);
  const int start = a.start_pos[s];
  const int tile_end = start + (qt * kQT + rows_here - 1) / G + 1;
  const int key_begin = part * a.part_size;
  const int key_end = min(tile_end, key_begin + a.part_size);
  if (key_begin >= key_end) return;
  const int parts_here = min(a.n_parts, (tile_end + a.part_size - 1) / a.part_size);
  const int n_tiles = (key_end - key_begin + kKT - 1) / kKT;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) ATTN_TRACE(0);
  constexpr int CH = D / 8;
  const int live_warps = (rows_here + 31) / 32;  // softmax warps with at least one live packed row
  if (tid == 0) {
    sm100::mbar_init(q_full, 32);
    for (int i = 0; i < kNS<D>; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_free[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) sm100::mbar_init(&p_full[i], 32 * live_warps);
    sm100::fence_barrier_init();
  }
  if (warp == 5) sm100::tmem_alloc<(D == 64 ? 256 : 512)>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: D=64 -> S0 | S1 | O | S2 in 256 columns; D=128 -> S0 | S1 | S2 | - | O in 512
  const uint32_t tO = tmem + (D == 64 ? 128 : 256);
  const uint32_t tS[kSBuf] = {tmem, tmem + 64, tmem + (D == 64 ? 192 : 128)};

  // Producer and MMA loops run warp-converged with one elected lane per operation (see gemm_ws_kernel).
  if (warp == 4) {
    // ------------------------------------------------------------------ producer warp
    const int32_t* bt = a.block_table + (int64_t)s * a.max_blocks;  // step metadata: uploaded before the forward
    const int last_blk = (key_end - 1) / a.B;
    const int per_tile = kKT / a.B;
    // KV streams through L2 with evict_first: keeping it (evict_last) pushed the next kernels' weights and
    // split-K partials out of L2 and cost ~3.5% of the forward (measured A/B)
    const uint64_t pol = sm100::policy_evict_first();
    // Block-table window: lane i holds the page id of page w0 + i, refilled with one coalesced load when a
    // tile needs a page past it (a dependent L2 load per page serialised the issue loop: ~4 us before Q).
    int w0 = -(1 << 30);
    int32_t win = 0;
    auto issue_kv = [&](int t) {  // warp-wide. K/V tile t: TMA boxes of [B keys x 64 dims], page by page
      const int st = t % kNS<D>;
      uint8_t* dk = sm + L::kK + st * L::kKVBytes;
      uint8_t* dv = sm + L::kV + st * L::kKVBytes;
      const int b0 = (key_begin + t * kKT) / a.B;
      if (a.exp & 32) {  // timing experiment: one page per tile (results wrong)
        if (sm100::elect_one()) sm100::mbar_arrive_expect_tx(&kv_full[st], 2 * L::kKVBytes / per_tile);
        const int idx = min(b0, last_blk);
        const int64_t blk = bt[idx];
        const int rowk = (int)(((blk * a.n_layers + a.layer) * 2) * a.B);
        if (sm100::elect_one()) {
#pragma unroll
          for (int sub = 0; sub < D / 64; ++sub) {
            sm100::tma_load_2d(dk + sub * kKT * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64, rowk, pol);
            sm100::tma_load_2d(dv + sub * kKT * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64, rowk + a.B, pol);
          }
        }
        __syncwarp();
        return;
      }
      if (sm100::elect_one()) sm100::mbar_arrive_expect_tx(&kv_full[st], 2 * L::kKVBytes);
      for (int j = 0; j < per_tile; ++j) {
        const int idx = min(b0 + j, last_blk);  // past the end: a valid duplicate, masked later
        if (idx >= w0 + 32) {
          w0 = idx;
          win = bt[min(w0 + lane, last_blk)];
        }
        const int64_t blk = __shfl_sync(0xffffffffu, win, idx - w0);
        const int rowk = (int)(((blk * a.n_layers + a.layer) * 2) * a.B);
        if (sm100::elect_one()) {
#pragma unroll
          for (int sub = 0; sub < D / 64; ++sub) {
            sm100::tma_load_2d(dk + sub * kKT * 128 + j * a.B * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64, rowk,
                               pol);
            sm100::tma_load_2d(dv + sub * kKT * 128 + j * a.B * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64,
                               rowk + a.B, pol);
          }
        }
        __syncwarp();
      }
    };
    // Tiles made only of pages wholly before this sequence's start position hold cached KV that no kernel of
    // this step writes: they stream in before the dependency wait, overlapping the kernels before.
    const int cached_end = (start / a.B) * a.B;
    int t = 0;
    static constexpr int kPreTiles = 2;  // before Q: each tile is 2 * 64/B TMA issues, which delay the Q gather
    for (; t < min(n_tiles, kPreTiles); ++t) {
      if (key_begin + (t + 1) * kKT > cached_end) break;
      issue_kv(t);
    }
    pdl_wait();  // q and this step's fresh K/V rows come from the kernels before
    pdl_trigger();
    // Q: the 32 lanes gather the 128 GQA-packed rows (4 each) with cp.async into the swizzled layout
    for (int p = lane; p < kQT; p += 32) {
      const bool valid = p < rows_here;
      const int pr = qt * kQT + p;
      const __nv_bfloat16* src = a.q + (int64_t)(row0 + (valid ? pr / G : 0)) * a.ld_q + (kvh * G + (valid ? pr % G : 0)) * D;
#pragma unroll
      for (int c = 0; c < CH; ++c) cp_async16(sm + L::kQ + sw_off(p, c, kQT), valid ? src + c * 8 : a.q, valid);
    }
    cp_async_commit();
    cp_async_wait<0>();
    sm100::fence_proxy_async_smem();
    sm100::mbar_arrive(q_full);
    for (; t < n_tiles; ++t) {
      const int st = t % kNS<D>;
      if (t >= kNS<D>) sm100::mbar_wait(&kv_empty[st], ((t / kNS<D>) - 1) & 1);
      issue_kv(t);
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------------ MMA issuer
    pdl_wait();
    constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(kQT, kKT);
    constexpr uint32_t idesc_o = sm100::idesc_bf16_f32_bmn(kQT, D);
    sm100::mbar_wait(q_full, 0);
    if (lane == 0) ATTN_TRACE(1);
    sm100::tc_fence_after();
    // Event-driven issue (no head-of-line blocking): S_ts needs its K tile and a free S buffer (ts%3 was read by
    // softmax_{ts-3}, observed as p_full when PV_{ts-3} was issued: ts <= tp + 2); PV_tp needs P_tp.
    int ts = 0, tp = 0;
    while (tp < n_tiles) {
      bool did = false;
      if (ts < n_tiles && ts <= tp + 2) {
        const int st = ts % kNS<D>;
        uint32_t ready = 0;
        // S_ts overwrites the TMEM columns PV_{ts-3} reads its P from: wait for that PV to COMPLETE (issue
        // order alone does not order a later MMA's accumulator writes after an earlier MMA's operand reads)
        if (lane == 0)
          ready = sm100::mbar_test(&kv_full[st], (ts / kNS<D>) & 1) &&
                          (ts < kSBuf || sm100::mbar_test(&s_free[ts % kSBuf], ((ts / kSBuf) - 1) & 1))
                      ? 1u : 0u;
        ready = __shfl_sync(0xffffffffu, ready, 0);
        if (ready) {
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            const uint8_t* qb = sm + L::kQ;
            const uint8_t* kb = sm + L::kK + st * L::kKVBytes;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {  // K = D in 16-wide steps; sub-tile every 4 steps
              const uint64_t da = sm100::umma_desc_sw128(qb + (ks >> 2) * kQT * 128 + (ks & 3) * 32);
              const uint64_t db = sm100::umma_desc_sw128(kb + (ks >> 2) * kKT * 128 + (ks & 3) * 32);
              if (!(a.exp & 64)) sm100::mma_bf16_ss(tS[ts % kSBuf], da, db, idesc_s, ks > 0 ? 1u : 0u);
            }
            sm100::mma_commit(&s_full[ts % kSBuf]);
          }
          __syncwarp();
          ++ts;
          did = true;
        }
      }
      if (tp < ts) {
        uint32_t ready = 0;
        if (lane == 0) ready = sm100::mbar_test(&p_full[tp % kSBuf], (tp / kSBuf) & 1) ? 1u : 0u;
        ready = __shfl_sync(0xffffffffu, ready, 0);
        if (ready) {
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
            const uint32_t tp_a = tS[tp % kSBuf];  // P_tp: bf16 pairs in the first 32 columns of its S buffer
            const uint8_t* vb = sm + L::kV + (tp % kNS<D>) * L::kKVBytes;
#pragma unroll
            for (int kk = 0; kk < kKT / 16; ++kk) {  // K = 64 keys, 16 per step = 8 TMEM columns
              const uint64_t db = sm100::umma_desc_sw128_mn(vb + kk * 16 * 128, kKT * 128);
              if (!(a.exp & 64)) sm100::mma_bf16_ts(tO, tp_a + kk * 8, db, idesc_o, (tp > 0 || kk > 0) ? 1u : 0u);
            }
            sm100::mma_commit(&kv_empty[tp % kNS<D>]);
            sm100::mma_commit(&s_free[tp % kSBuf]);
          }
          __syncwarp();
          ++tp;
          did = true;
        }
      }
      if (!did) __nanosleep(32);
    }
  } else if (warp < live_warps) {
    // ------------------------------------------------------------------ softmax (live warps of 0-3)
    // Scores stay raw (unscaled): the max commutes with the positive scale, and each probability is one
    // FFMA + ex2: p = 2^(s * scale_log2 - m * scale_log2). m_run is kept raw; partials store it scaled.
    pdl_wait();
    const int r = tid;  // TMEM lane == packed row
    const bool live = r < rows_here;
    const int pos = live ? start + (qt * kQT + r) / G : -1;
    const int lim = min(pos, key_end - 1);
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const float sc = a.scale_log2;
    const float thr = kRescaleLog2 / sc;  // rescale threshold in raw score units
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = 0; t < n_tiles; ++t) {
      const int k0 = key_begin + t * kKT;
      sm100::mbar_wait(&s_full[t % kSBuf], (t / kSBuf) & 1);
      sm100::tc_fence_after();
      if (a.exp & 16) {  // timing experiment: no softmax work at all
        sm100::tc_fence_before();
        sm100::mbar_arrive(&p_full[t % kSBuf]);
        continue;
      }
      if (t == 0 && tid == 0) ATTN_TRACE(2);
      float sv[kKT];
      {
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(tS[t % kSBuf] + lane_base, r0);
        sm100::tmem_ld_32x32b_x32(tS[t % kSBuf] + lane_base + 32, r1);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sv[j] = __uint_as_float(r0[j]);
          sv[j + 32] = __uint_as_float(r1[j]);
        }
      }
      if (__any_sync(0xffffffffu, k0 + kKT - 1 > lim)) {  // causal / partition-end mask: warp-uniform branch
#pragma unroll
        for (int j = 0; j < kKT; ++j)
          if (k0 + j > lim) sv[j] = -INFINITY;
      }
      float mx[8];  // 8 independent max chains, then a tree
#pragma unroll
      for (int q = 0; q < 8; ++q) mx[q] = fmaxf(sv[q], sv[q + 8]);
#pragma unroll
      for (int j = 16; j < kKT; j += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) mx[q] = fmaxf(mx[q], sv[j + q]);
      }
      const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      const float m_new = fmaxf(m_run, mt);
      // lazy rescale: only when the max grew by more than 2^8 (or on the first finite max)
      const bool grow = m_new > m_run + thr || (m_run == -INFINITY && m_new != -INFINITY);
      if (t > 0 && __any_sync(0xffffffffu, grow && m_run != -INFINITY)) {
        const float corr = grow && m_run != -INFINITY ? fast_exp2((m_run - m_new) * sc) : 1.f;
        sm100::mbar_wait(&s_free[(t - 1) % kSBuf], ((t - 1) / kSBuf) & 1);  // O holds PV_{t-1}
        sm100::tc_fence_after();
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t ov[32];
          sm100::tmem_ld_32x32b_x32(tO + lane_base + c, ov);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
          sm100::tmem_st_32x32b_x32(tO + lane_base + c, ov);
        }
        sm100::tmem_st_wait();
        l_run *= corr;
      }
      if (grow) m_run = m_new;
      const float nb = m_run == -INFINITY ? 0.f : -m_run * sc;
      float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // P as bf16 pairs (key 2j in the low half of column j), 16 columns at a time
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float p0 = fast_exp2(fmaf(sv[h * 32 + 2 * j], sc, nb));
          const float p1 = fast_exp2(fmaf(sv[h * 32 + 2 * j + 1], sc, nb));
          rs4[j & 3] += p0 + p1;
          pk[j] = pack_bf16(p0, p1);
        }
        sm100::tmem_st_32x32b_x16(tS[t % kSBuf] + lane_base + h * 16, pk);
      }
      sm100::tmem_st_wait();
      l_run += (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[t % kSBuf]);
    }
    if (tid == 0) ATTN_TRACE(3);
    // final O
    sm100::mbar_wait(&s_free[(n_tiles - 1) % kSBuf], ((n_tiles - 1) / kSBuf) & 1);
    sm100::tc_fence_after();
    {
      const int pr = qt * kQT + r;
      const int tok = live ? pr / G : 0, head = kvh * G + (live ? pr % G : 0);
      const int64_t grow_ = row0 + tok;
      const bool emit = live && pos >= key_begin;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t ov[32];
        sm100::tmem_ld_32x32b_x32(tO + lane_base + c, ov);
        sm100::tmem_ld_wait();
        if (!emit) continue;
        if (parts_here == 1) {
          __nv_bfloat16* dst = a.out + grow_ * a.ld_out + head * D + c;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            __align__(16) __nv_bfloat162 o2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              o2[e] = __floats2bfloat162_rn(__uint_as_float(ov[q * 8 + e * 2]) * inv,
                                            __uint_as_float(ov[q * 8 + e * 2 + 1]) * inv);
            *reinterpret_cast<int4*>(dst + q * 8) = *reinterpret_cast<int4*>(o2);
          }
        } else {
          const int64_t slot = ((int64_t)part * a.M + grow_) * a.H + head;
          float* dst = a.ws_o + slot * D + c;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(reinterpret_cast<float4*>(dst + q * 4),
                   make_float4(__uint_as_float(ov[q * 4]), __uint_as_float(ov[q * 4 + 1]),
                               __uint_as_float(ov[q * 4 + 2]), __uint_as_float(ov[q * 4 + 3])));
          if (c == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml + slot * 2), make_float2(m_run * sc, l_run));
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 5) sm100::tmem_dealloc<(D == 64 ? 256 : 512)>(tmem);
  if (tid == 0) ATTN_TRACE(4);
  if (parts_here > 1) merge_partials<D>(a, s, kvh, qt, row0, start, rows_here, parts_here, G, &s_last);
  if (tid == 0) ATTN_TRACE(5);
}


// ============================================================================================================
// Shared-prefix attention over a host-built work list (attn_plan.cpp). The eval turn of a multi-adapter
// pipeline puts 8 requests on the SAME physical prefix blocks (base-aligned hashing, kv_cache.py:72-96); the
// per-span kernel above streams that prefix once per request with 64 live rows in each 128-row tile. Here a
// work item is (query set, 128-row M-tile, KV partition) x kv head: the set packs the rows of every request
// of a group, so one K/V stream feeds full tiles, and the item's segments (the shared prefix through the
// group's table, then each request's own keys through its own table, other rows masked) run through one
// online softmax. Decode steps of the same group share the prefix the same way.
// Pipeline: producer warp (TMA page boxes, segment by segment), MMA warp on a STATIC schedule with blocking
// mbarrier waits (the event loop of attn_tc_kernel spent ~150 cycles per mbar_test and bounded its tile rate),
// S running kSB-1 tiles ahead of PV, 4 softmax warps (one TMEM lane quadrant each).
// ============================================================================================================
template <int D>
constexpr int kSB = D == 128 ? 4 : 3;  // S buffers in TMEM (D=128: 4 x 64 + O 128 of 512; D=64: 3 x 64 + O 64 of 256)

struct GrpArgs {
  const __nv_bfloat16* q;
  int64_t ld_q;
  const int32_t* positions;  // [M] absolute position of each row
  const int32_t* row_seq;    // [M] span of each row
  const int32_t* block_table;
  int max_blocks;
  const int32_t* items;      // [n_items][8]
  const int32_t* segs;       // [n_segs][4]
  const int32_t* sets;       // [n_sets][2]
  const int32_t* set_tok;    // [M]
  const int32_t* sp_np;      // [S]
  const __nv_bfloat16* kv;
  int n_layers, layer, B, H, Hkv;
  float scale_log2;
  __nv_bfloat16* out;
  int64_t ld_out;
  float* ws_o;   // [max_np][M][H][D]
  float* ws_ml;  // [max_np][M][H][2]
  int M;
  unsigned long long* trace;
  int exp;
  long long* tl;  // ALORA_ATTN_TL=1: clock64 timeline of CTA (0, 0): [9 events][2 query tiles][256 tiles]
};

// walks an item's segments tile by tile (64 keys per tile)
struct SegCursor {
  const int32_t* segs;
  int j, end, t_in, nt, tab, lo, hi, filter;
  __device__ void load() {
    tab = segs[4 * j];
    lo = segs[4 * j + 1];
    hi = segs[4 * j + 2];
    filter = segs[4 * j + 3];
    nt = (hi - lo + kKT - 1) / kKT;
    t_in = 0;
  }
  __device__ void init(const int32_t* s, int b, int e) {
    segs = s;
    j = b;
    end = e;
    if (j < end) load();
    skip_empty();
  }
  __device__ void skip_empty() {
    while (j < end && t_in >= nt) {
      ++j;
      if (j < end) load();
    }
  }
  __device__ void next() {
    ++t_in;
    skip_empty();
  }
  __device__ int k0() const { return lo + t_in * kKT; }
};

// Producer: PW = 0 -> one warp issuing TMA page boxes [B keys x 64 dims]; PW > 0 -> PW warps loading whole
// tiles with cp.async (16-byte chunks written straight into the SW128 layout from per-lane precomputed offsets),
// warp w owning tiles w, w+PW, ..., each lane arriving on the tile's barrier when its copies land
// (cp.async.mbarrier.arrive), so every free ring stage is in flight. Per-box TMA processing (~70 ns per 2 KB page
// box) capped a CTA's K/V supply at ~30 GB/s; the first cp.async version (generic per-chunk address arithmetic,
// wait_group publishing) was issue-bound at about the same rate.
// MT = M-tiles per CTA. With MT = 2 (the default) a CTA runs two 128-row query tiles of a set against every
// K/V tile it loads, halving the per-row K/V ingest. Softmax warps 4X..4X+3 serve tile X (TMEM lane quadrant =
// warp % 4). Q sits in TMEM (the A operand of S = Q K^T), P goes to smem (the A operand of O += P V), so an S
// buffer is free again as soon as the softmax has read it: S_{t+NB} does not wait for PV_t, and two issuer warps
// (S and PV) keep either MMA from queueing behind the other's wait.
// Warps: 4 x MT softmax, PW producers, the S-MMA issuer, the PV-MMA issuer.
template <int PW, int MT>
constexpr int kGrpThreads = (4 * MT + (PW > 0 ? PW : 1) + 2) * 32;
// TMEM (512 columns; 256 for D=64 with one query tile, two CTAs per SM) per query tile x: O (D fp32 columns),
// Q (D/2 columns of bf16 pairs: the A operand of S = Q K^T comes from TMEM, which keeps the smem for the K/V
// ring) and NB S buffers of 64 columns
template <int D, int MT>
constexpr int kGrpNB = MT == 2 ? (D == 128 ? 1 : 2) : (D == 128 ? 3 : 2);
template <int D, int MT>
constexpr int kGrpTmemUsed = MT * (D + D / 2 + kGrpNB<D, MT> * 64);
template <int D, int MT>
constexpr int kGrpTmem = kGrpTmemUsed<D, MT> <= 256 ? 256 : 512;
// P buffers per query tile (bf16 [128 rows][64 keys] in smem, the A operand of O += P V); at D=128 one buffer
// (the softmax of tile t+1 rarely waits for PV_t) buys the sixth K/V stage
#ifndef ALORA_GRP_NP
#define ALORA_GRP_NP 1
#endif
template <int D, int MT>
constexpr int kGrpNP = (D == 64 && MT == 2) ? 2 : ALORA_GRP_NP;
// K/V ring stages: what the 227 KB of smem leaves after the P buffers (D=64 with one query tile keeps two CTAs
// per SM)
template <int D, int MT>
constexpr int kGrpNS = D == 128 ? (kGrpNP<D, MT> == 1 ? 6 : 5) : (MT == 2 ? 9 : 4);
template <int D, int MT>
struct SmemG {
  static constexpr int kKVBytes = kKT * D * 2;
  static constexpr int kPBytes = kQT * kKT * 2;
  static constexpr int kP = 0;
  static constexpr int kK = kP + MT * kGrpNP<D, MT> * kPBytes;
  static constexpr int kV = kK + kGrpNS<D, MT> * kKVBytes;
  static constexpr int kBar = kV + kGrpNS<D, MT> * kKVBytes;
  static constexpr int kTotal = kBar + 512 + 1024;
};
static_assert(SmemG<128, 2>::kTotal <= 232448 && SmemG<64, 2>::kTotal <= 232448 &&
              SmemG<128, 1>::kTotal <= 232448 && 2 * SmemG<64, 1>::kTotal <= 232448, "attn_grp smem");
static_assert(kGrpTmemUsed<128, 2> <= 512 && kGrpTmemUsed<64, 2> <= 512 && kGrpTmemUsed<128, 1> <= 512 &&
              kGrpTmemUsed<64, 1> <= 256, "attn_grp tmem");

template <int D, int PW, int MT>
__global__ void __launch_bounds__(kGrpThreads<PW, MT>, (D == 64 && MT == 1) ? 2 : 1)
    attn_grp_kernel(const GrpArgs a, const __grid_constant__ CUtensorMap tm_kv) {
  using L = SmemG<D, MT>;
  constexpr int NB = kGrpNB<D, MT>;
  constexpr int NS = kGrpNS<D, MT>;
  constexpr int NP = kGrpNP<D, MT>;
  static_assert(NS > NB, "the S look-ahead needs its K tiles in the ring");
  constexpr int kSoftWarps = 4 * MT;
  constexpr int kMmaWarp = kSoftWarps + (PW > 0 ? PW : 1);  // S = Q K^T issuer (and TMEM owner)
  constexpr int kPvWarp = kMmaWarp + 1;                       // O += P V issuer
  constexpr int kTmemCols = kGrpTmem<D, MT>;
  extern __shared__ uint8_t smem_raw_grp[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_grp) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kBar);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = kv_full + NS;
  uint64_t* s_full = kv_empty + NS;     // [MT][NB] S MMA committed
  uint64_t* s_free = s_full + MT * NB;  // [MT][NB] the softmax has read S into registers (one phase per use)
  uint64_t* p_full = s_free + MT * NB;  // [MT][NP] P stored to smem (and proxy-fenced)
  uint64_t* p_free = p_full + MT * NP;  // [MT][NP] the PV reading that P completed (one phase per use)
  uint64_t* q_full = p_free + MT * NP;  // [MT] Q rows stored to TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + MT);

  const int* it = a.items + (int64_t)blockIdx.x * 8;
  const int set = it[0], mtile = it[1], seg_b = it[2], seg_e = it[3], p_index = it[4], cached = it[5];
  const int n_tiles = it[6];
  const int kvh = blockIdx.y;
  const int G = a.H / a.Hkv;
  const int tok_off = a.sets[2 * set], n_tok = a.sets[2 * set + 1];
  int rows_t[MT];
#pragma unroll
  for (int x = 0; x < MT; ++x) rows_t[x] = max(0, min(kQT, n_tok * G - (mtile * MT + x) * kQT));
  // Decode-like sets (at most 32 GQA-packed rows, e.g. 8 adapters x 4 heads decoding on one conversation): one
  // softmax warp would carry every row through all 64 keys of each tile (~1 us per tile). Instead the rows are
  // replicated into the 4 TMEM lane quadrants of query tile 0 and quadrant q takes only keys [16q, 16q + 16) of
  // every tile (its P row is zero elsewhere), so the 4 warps split the exponentials; the 4 copies' (m, l, O)
  // combine in the epilogue like KV partitions.
  const int set_rows = n_tok * G;
  const bool rep4 = MT == 2 && set_rows <= 32;
  if (rep4) {
    rows_t[0] = kQT;
    rows_t[1] = 0;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) ATTN_TRACE(0);
  long long* tl = (a.tl && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0) ? a.tl : nullptr;
#define GRP_TL(ev, x, t) \
  if (tl && (t) < 256) tl[((ev) * 2 + (x)) * 256 + (t)] = clock64()
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      sm100::mbar_init(&kv_full[i], PW > 0 ? 32 : 1);  // cp.async: every lane of the loading warp arrives
      sm100::mbar_init(&kv_empty[i], 1);
    }
    for (int x = 0; x < MT; ++x) {
      const int live_threads = 32 * max(1, (rows_t[x] + 31) / 32);
      for (int i = 0; i < NB; ++i) {
        sm100::mbar_init(&s_full[x * NB + i], 1);
        sm100::mbar_init(&s_free[x * NB + i], live_threads);
      }
      for (int i = 0; i < NP; ++i) {
        sm100::mbar_init(&p_full[x * NP + i], live_threads);
        sm100::mbar_init(&p_free[x * NP + i], 1);
      }
      sm100::mbar_init(&q_full[x], live_threads);
    }
    sm100::fence_barrier_init();
  }
  if (warp == kMmaWarp) sm100::tmem_alloc<kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // O of tile x at x*D, its Q at MT*D + x*D/2, then the S buffers: tile x buffer i at MT*3D/2 + (x*NB + i)*64
  auto tOx = [&](int x) { return tmem + (uint32_t)(x * D); };
  auto tQx = [&](int x) { return tmem + (uint32_t)(MT * D + x * (D / 2)); };
  auto tSx = [&](int x, int i) { return tmem + (uint32_t)(MT * D + MT * (D / 2) + (x * NB + i) * 64); };

  if (PW > 0 && warp >= kSoftWarps && warp < kSoftWarps + PW) {
    // ------------------------------------------------------------------ cp.async producer warps
    const int pw = warp - kSoftWarps;
    SegCursor cur;
    cur.init(a.segs, seg_b, seg_e);
    int w0 = -(1 << 30), wseg = -1;
    int32_t win = 0;
    bool waited = false;
    const int kvw = a.Hkv * D;
    const int per_tile = kKT / a.B;
    const int r0 = lane >> 3, c0 = lane & 7;
    const int64_t g_lane = ((int64_t)r0 * kvw + c0 * 8) * 2;  // bytes
    const int64_t row4 = (int64_t)4 * kvw * 2, vstep = (int64_t)a.B * kvw * 2;
    const uint32_t s_lane0 = (uint32_t)(r0 * 128 + ((c0 ^ r0) << 4));
    const uint32_t s_lane1 = (uint32_t)((r0 + 4) * 128 + ((c0 ^ (r0 + 4)) << 4));
    constexpr uint32_t kVOff = L::kV - L::kK;  // V stage st sits at a fixed distance from K stage st
    for (int t = 0; t < n_tiles; ++t, cur.next()) {
      if (t % (PW > 0 ? PW : 1) != pw) continue;
      const int st = t % NS;
      const int k0 = cur.k0();
      if (!waited && !(k0 + kKT <= cached || (cur.filter < 0 && cur.hi <= cached))) {
        pdl_wait();  // this tile may hold keys the kernels before wrote
        waited = true;
      }
      if (t >= NS) sm100::mbar_wait(&kv_empty[st], ((t / NS) - 1) & 1);
      const int32_t* bt = a.block_table + (int64_t)cur.tab * a.max_blocks;
      const int last_blk = (cur.hi - 1) / a.B;
      const int b0 = k0 / a.B;
      if (cur.j != wseg) {
        wseg = cur.j;
        w0 = -(1 << 30);
      }
      if (b0 + per_tile - 1 >= w0 + 32 || b0 < w0) {
        w0 = b0;
        win = bt[min(w0 + lane, last_blk)];
      }
      // lane = (row r0 = lane / 8 of each 4-row group, 16-byte chunk c = lane % 8): every address below is a
      // per-lane base plus a per-(page, row group) step, so the loop is a run of cp.async with few address ops
      // (the generic per-chunk address arithmetic made this warp issue-bound at ~30 GB/s per SM)
      const uint32_t sk = smem_addr(sm + L::kK + st * L::kKVBytes);
      for (int j = 0; j < per_tile; ++j) {
        const int idx = min(b0 + j, last_blk);  // past the end: a valid duplicate, masked by the softmax
        const int64_t blk = __shfl_sync(0xffffffffu, win, idx - w0);
        const char* kp = reinterpret_cast<const char*>(
                             a.kv + ((blk * a.n_layers + a.layer) * 2) * a.B * (int64_t)kvw + kvh * D) + g_lane;
        const uint32_t sj = sk + (uint32_t)(j * a.B * 128);
#pragma unroll 4
        for (int i = 0; i < a.B / 4; ++i) {
          const char* kg = kp + (int64_t)i * row4;
          const uint32_t so = sj + (uint32_t)((i >> 1) * 1024) + ((i & 1) ? s_lane1 : s_lane0);
#pragma unroll
          for (int sub = 0; sub < D / 64; ++sub) {
            cp_async16_s(so + sub * kKT * 128, kg + sub * 128);
            cp_async16_s(so + sub * kKT * 128 + kVOff, kg + vstep + sub * 128);
          }
        }
      }
      // each lane's arrive fires when its copies (and all its earlier ones) have landed, so the warp never
      // blocks on its own loads: every free ring stage can be in flight. The MMA warp issues the proxy fence
      // after its wait (generic-proxy smem writes read by tcgen05.mma).
      cp_async_mbar_arrive_noinc(&kv_full[st]);
    }
    cp_async_wait<0>();
    if (!waited) pdl_wait();
  } else if (PW == 0 && warp == kSoftWarps) {
    // ------------------------------------------------------------------ TMA producer warp
    const uint64_t pol = sm100::policy_evict_first();
    SegCursor cur;
    cur.init(a.segs, seg_b, seg_e);
    int w0 = -(1 << 30), wtab = -1;
    int32_t win = 0;
    auto issue_kv = [&](int t) {  // warp-wide: K/V tile t (the cursor's tile), TMA page boxes [B keys x 64 dims]
      const int st = t % NS;
      const int per_tile = (a.exp & 32) ? 1 : kKT / a.B;  // timing experiment 32: one page per tile (wrong results)
      if (sm100::elect_one()) sm100::mbar_arrive_expect_tx(&kv_full[st], 2 * L::kKVBytes / (kKT / a.B) * per_tile);
      uint8_t* dk = sm + L::kK + st * L::kKVBytes;
      uint8_t* dv = sm + L::kV + st * L::kKVBytes;
      const int32_t* bt = a.block_table + (int64_t)cur.tab * a.max_blocks;
      const int last_blk = (cur.hi - 1) / a.B;
      const int b0 = cur.k0() / a.B;
      if (cur.j != wtab) {  // a new segment: its table row and its clamp bound differ, refill the window
        wtab = cur.j;
        w0 = -(1 << 30);
      }
      for (int j = 0; j < per_tile; ++j) {
        const int idx = min(b0 + j, last_blk);  // past the end: a valid duplicate, masked by the softmax
        if (idx >= w0 + 32 || idx < w0) {
          w0 = idx;
          win = bt[min(w0 + lane, last_blk)];
        }
        const int64_t blk = __shfl_sync(0xffffffffu, win, idx - w0);
        const int rowk = (int)(((blk * a.n_layers + a.layer) * 2) * a.B);
        if (sm100::elect_one()) {
#pragma unroll
          for (int sub = 0; sub < D / 64; ++sub) {
            sm100::tma_load_2d(dk + sub * kKT * 128 + j * a.B * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64, rowk,
                               pol);
            sm100::tma_load_2d(dv + sub * kKT * 128 + j * a.B * 128, &tm_kv, &kv_full[st], kvh * D + sub * 64,
                               rowk + a.B, pol);
          }
        }
        __syncwarp();
      }
    };
    int t = 0;
    // tiles wholly below every row's first computed position hold KV no kernel of this step writes: they stream
    // in before the dependency wait (at most kNS of them, the ring depth)
    for (; t < min(n_tiles, NS); ++t) {
      if (cur.k0() + kKT > cached && !(cur.filter < 0 && cur.hi <= cached)) break;
      issue_kv(t);
      cur.next();
    }
    pdl_wait();
    for (; t < n_tiles; ++t) {
      const int st = t % NS;
      if (t >= NS) sm100::mbar_wait(&kv_empty[st], ((t / NS) - 1) & 1);
      issue_kv(t);
      cur.next();
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------------ S-MMA issuer
    // Two issuer warps: S_{t+NB} needs only the softmax's read of S_t and the K tile, PV_t only P_t, so neither
    // waits behind the other (one in-order issuer left the PV ~800 cycles behind its P and S_{t+1} behind it)
    pdl_wait();
    pdl_trigger();
    constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(kQT, kKT);
    if (lane == 0) ATTN_TRACE(1);
    sm100::tc_fence_after();
    // S of tile ts for query tile x (A = Q from TMEM), into the buffer the softmax of tile ts - NB has read
    auto issue_s = [&](int ts) {
      const int st = ts % NS;
      sm100::mbar_wait(&kv_full[st], (ts / NS) & 1);
      if (PW > 0) sm100::fence_proxy_async_smem();  // cp.async (generic proxy) data -> tcgen05.mma operands
#pragma unroll
      for (int x = 0; x < MT; ++x) {
        if (rows_t[x] == 0) continue;
        if (ts == 0) sm100::mbar_wait(&q_full[x], 0);
        if (ts >= NB) sm100::mbar_wait(&s_free[x * NB + ts % NB], ((ts / NB) - 1) & 1);
        sm100::tc_fence_after();
        GRP_TL(2, x, ts);
        if (sm100::elect_one()) {
          const uint8_t* kb = sm + L::kK + st * L::kKVBytes;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint64_t db = sm100::umma_desc_sw128(kb + (ks >> 2) * kKT * 128 + (ks & 3) * 32);
            if (!(a.exp & 64)) sm100::mma_bf16_ts(tSx(x, ts % NB), tQx(x) + ks * 8, db, idesc_s, ks > 0 ? 1u : 0u);
          }
          sm100::mma_commit(&s_full[x * NB + ts % NB]);
        }
        __syncwarp();
      }
    };
    // S_{ts} reuses the buffer the softmax released as soon as it had read S_{ts-NB} into registers (P goes to
    // smem, not back into TMEM)
    for (int ts = 0; ts < n_tiles; ++ts) issue_s(ts);
  } else if (warp == kPvWarp) {
    // ------------------------------------------------------------------ PV-MMA issuer
    constexpr uint32_t idesc_o = sm100::idesc_bf16_f32_bmn(kQT, D);
    sm100::tc_fence_after();
    for (int tp = 0; tp < n_tiles; ++tp) {
#pragma unroll
      for (int x = 0; x < MT; ++x) {
        if (rows_t[x] == 0) continue;
        sm100::mbar_wait(&p_full[x * NP + tp % NP], (tp / NP) & 1);
        sm100::tc_fence_after();
        GRP_TL(3, x, tp);
        if (sm100::elect_one()) {
          const uint8_t* pb = sm + L::kP + (x * NP + tp % NP) * L::kPBytes;
          const uint8_t* vb = sm + L::kV + (tp % NS) * L::kKVBytes;
#pragma unroll
          for (int kk = 0; kk < kKT / 16; ++kk) {
            const uint64_t da = sm100::umma_desc_sw128(pb + kk * 32);
            const uint64_t db = sm100::umma_desc_sw128_mn(vb + kk * 16 * 128, kKT * 128);
            if (!(a.exp & 64)) sm100::mma_bf16_ss(tOx(x), da, db, idesc_o, (tp > 0 || kk > 0) ? 1u : 0u);
          }
          sm100::mma_commit(&p_free[x * NP + tp % NP]);
        }
        __syncwarp();
      }
      // every PV of tile tp read its V; S_tp (issued by the other warp) completed before the softmax published P_tp
      if (sm100::elect_one()) sm100::mma_commit(&kv_empty[tp % NS]);
      __syncwarp();
    }
  } else if (warp < kSoftWarps && (warp & 3) < (rows_t[warp >> 2] + 31) / 32) {
    // ------------------------------------------------------------------ softmax (live warps; 4 per query tile)
    pdl_wait();
    const int xt = warp >> 2;  // query tile
    const int r = (warp & 3) * 32 + lane;
    const int copy = rep4 ? (warp & 3) : 0;  // key quarter of this row copy (rep4)
    const int lr = rep4 ? lane : r;          // row within the tile's packed rows
    const bool live = rep4 ? lr < set_rows : r < rows_t[xt];
    const int pr = (mtile * MT + xt) * kQT + lr;
    const int row = live ? a.set_tok[tok_off + pr / G] : 0;
    const int head = kvh * G + pr % G;
    const int pos = live ? a.positions[row] : -1;
    const int span = live ? a.row_seq[row] : -2;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // this tile's barriers as 32-bit shared addresses (buffer i at + 8 i)
    const uint32_t s_full_x = smem_addr(s_full + xt * NB), s_free_x = smem_addr(s_free + xt * NB);
    const uint32_t p_full_x = smem_addr(p_full + xt * NP), p_free_x = smem_addr(p_free + xt * NP);
    const uint32_t tS0 = tSx(xt, 0) + lane_base;  // S buffer i at tS0 + 64 i
    const uint32_t tO = tOx(xt);
    // this thread's P row (K-major SW128: 16-byte chunk c of row r at chunk c ^ (r & 7))
    const uint32_t p_row = smem_addr(sm + L::kP + xt * NP * L::kPBytes) + (uint32_t)(r * 128);
    {  // this row's Q (D bf16 = D/2 columns of pairs, the layout of a TMEM A operand) into TMEM lane r
      const uint4* src = reinterpret_cast<const uint4*>(a.q + (int64_t)row * a.ld_q + head * D);
#pragma unroll
      for (int c = 0; c < D / 2; c += 32) {
        uint32_t qv[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 w = live ? __ldg(src + c / 4 + v) : make_uint4(0u, 0u, 0u, 0u);
          qv[4 * v] = w.x; qv[4 * v + 1] = w.y; qv[4 * v + 2] = w.z; qv[4 * v + 3] = w.w;
        }
        sm100::tmem_st_32x32b_x32(tQx(xt) + lane_base + c, qv);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&q_full[xt]);
    }
    const float sc = a.scale_log2;
    const float thr = kRescaleLog2 / sc;
    float m_run = -INFINITY, l_run = 0.f;
    SegCursor cur;
    cur.init(a.segs, seg_b, seg_e);
    int lim = -1, lim_seg = -1;
    if (rep4) {  // this row's P columns outside its key quarter stay zero for the whole kernel
#pragma unroll
      for (int b2 = 0; b2 < NP; ++b2)
#pragma unroll
        for (int c = 0; c < 8; ++c) st_shared_v4(p_row + (uint32_t)(b2 * L::kPBytes + (c << 4)), 0u, 0u, 0u, 0u);
    }
    // O *= corr once the previous PV has landed (lazy rescale: the row max grew by more than 2^8)
    auto rescale_o = [&](int t, float corr) {
      sm100::mbar_wait_a(p_free_x + 8 * ((t - 1) % NP), ((t - 1) / NP) & 1);  // O holds PV_{t-1}
      sm100::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < D; c += 16) {  // 16 columns at a time: the scores stay in registers
        uint32_t ov[16];
        sm100::tmem_ld_32x32b_x16(tO + lane_base + c, ov);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
        sm100::tmem_st_32x32b_x16(tO + lane_base + c, ov);
      }
      sm100::tmem_st_wait();
    };
    for (int t = 0; t < n_tiles; ++t) {
      if (cur.j != lim_seg) {
        lim_seg = cur.j;
        lim = (live && (cur.filter < 0 || cur.filter == span)) ? min(pos, cur.hi - 1) : -1;
      }
      const int k0 = cur.k0();
      cur.next();
      sm100::mbar_wait_a(s_full_x + 8 * (t % NB), (t / NB) & 1);
      sm100::tc_fence_after();
      if ((warp & 3) == 0) GRP_TL(0, xt, t);
      if (rep4) {  // ---- this copy's 16 keys of the tile
        float sq[16];
        {
          uint32_t rv[16];
          sm100::tmem_ld_32x32b_x16(tS0 + (uint32_t)((t % NB) * 64 + 16 * copy), rv);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) sq[j] = __uint_as_float(rv[j]);
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive_a(s_free_x + 8 * (t % NB));
        const int kq = k0 + 16 * copy;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (kq + j > lim) sq[j] = -INFINITY;
        float mt = sq[0];
#pragma unroll
        for (int j = 1; j < 16; ++j) mt = fmaxf(mt, sq[j]);
        const float m_new = fmaxf(m_run, mt);
        const bool grow = m_new > m_run + thr || (m_run == -INFINITY && m_new != -INFINITY);
        if (t > 0 && __any_sync(0xffffffffu, grow && m_run != -INFINITY)) {
          const float corr = grow && m_run != -INFINITY ? fast_exp2((m_run - m_new) * sc) : 1.f;
          rescale_o(t, corr);
          l_run *= corr;
        }
        if (grow) m_run = m_new;
        const float nb = m_run == -INFINITY ? 0.f : -m_run * sc;
        uint32_t pk[8];
        float ls = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float p0 = fast_exp2(fmaf(sq[2 * j], sc, nb)), p1 = fast_exp2(fmaf(sq[2 * j + 1], sc, nb));
          ls += p0 + p1;
          pk[j] = pack_bf16(p0, p1);
        }
        l_run += ls;
        if (t >= NP) sm100::mbar_wait_a(p_free_x + 8 * (t % NP), ((t / NP) - 1) & 1);
        const uint32_t pb = p_row + (uint32_t)((t % NP) * L::kPBytes);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          st_shared_v4(pb + (uint32_t)(((2 * copy + c) ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                       pk[4 * c + 3]);
        sm100::fence_proxy_async_smem();
        sm100::mbar_arrive_a(p_full_x + 8 * (t % NP));
        continue;
      }
      float sv[kKT];
      {
        const uint32_t ts = tS0 + (uint32_t)((t % NB) * 64);
        uint32_t rv0[32], rv1[32];  // both loads in flight before the one wait
        sm100::tmem_ld_32x32b_x32(ts, rv0);
        sm100::tmem_ld_32x32b_x32(ts + 32, rv1);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sv[j] = __uint_as_float(rv0[j]);
          sv[32 + j] = __uint_as_float(rv1[j]);
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive_a(s_free_x + 8 * (t % NB));  // S_{t+NB} may overwrite the buffer
      if ((warp & 3) == 0) GRP_TL(6, xt, t);
      if (__any_sync(0xffffffffu, k0 + kKT - 1 > lim)) {
#pragma unroll
        for (int j = 0; j < kKT; ++j)
          if (k0 + j > lim) sv[j] = -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) mx[q] = fmaxf(sv[q], sv[q + 8]);
#pragma unroll
      for (int j = 16; j < kKT; j += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) mx[q] = fmaxf(mx[q], sv[j + q]);
      }
      const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      const float m_new = fmaxf(m_run, mt);
      const bool grow = m_new > m_run + thr || (m_run == -INFINITY && m_new != -INFINITY);
      if (t > 0 && __any_sync(0xffffffffu, grow && m_run != -INFINITY)) {
        const float corr = grow && m_run != -INFINITY ? fast_exp2((m_run - m_new) * sc) : 1.f;
        rescale_o(t, corr);
        l_run *= corr;
      }
      if (grow) m_run = m_new;
      const float nb = m_run == -INFINITY ? 0.f : -m_run * sc;
      // paired fp32 (FFMA2 / FADD2): half the FMA-pipe instructions of the scale and the row sum
      const uint64_t sc2 = f2_pack(sc, sc), nb2 = f2_pack(nb, nb);
      if ((warp & 3) == 0) GRP_TL(7, xt, t);
      uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
      uint32_t pk[kKT / 2];
#pragma unroll
      for (int j = 0; j < kKT / 2; ++j) {
        float x0, x1;
        f2_unpack(ffma2(f2_pack(sv[2 * j], sv[2 * j + 1]), sc2, nb2), x0, x1);
        const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
        acc2[j & 3] = fadd2(acc2[j & 3], f2_pack(p0, p1));
        pk[j] = pack_bf16(p0, p1);
      }
      {
        const uint64_t s2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float l0, l1;
        f2_unpack(s2, l0, l1);
        l_run += l0 + l1;
      }
      if ((warp & 3) == 0) GRP_TL(4, xt, t);
      if (t >= NP) sm100::mbar_wait_a(p_free_x + 8 * (t % NP), ((t / NP) - 1) & 1);  // PV_{t-NP} read this buffer
      if ((warp & 3) == 0) GRP_TL(5, xt, t);
      {
        const uint32_t pb = p_row + (uint32_t)((t % NP) * L::kPBytes);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(pb + (uint32_t)((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      if ((warp & 3) == 0) GRP_TL(8, xt, t);
      sm100::fence_proxy_async_smem();  // generic-proxy P stores -> tcgen05.mma operand reads
      sm100::mbar_arrive_a(p_full_x + 8 * (t % NP));
      if ((warp & 3) == 0) GRP_TL(1, xt, t);
    }
    if (tid == 0) ATTN_TRACE(3);
    sm100::mbar_wait_a(p_free_x + 8 * ((n_tiles - 1) % NP), ((n_tiles - 1) / NP) & 1);  // O holds the last PV
    sm100::tc_fence_after();
    if (rep4) {
      // combine the 4 row copies through smem (the K/V ring is free: every MMA has completed): [copy][32][D] O,
      // [copy][32] (m, l); copy 0's warp writes the row
      float* xo = reinterpret_cast<float*>(sm + L::kK);
      float* xml = xo + 4 * 32 * D;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t ov[32];
        sm100::tmem_ld_32x32b_x32(tO + lane_base + c, ov);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(xo + ((copy * 32 + lane) * D + c + 4 * q)) =
              make_float4(__uint_as_float(ov[4 * q]), __uint_as_float(ov[4 * q + 1]), __uint_as_float(ov[4 * q + 2]),
                          __uint_as_float(ov[4 * q + 3]));
      }
      xml[(copy * 32 + lane) * 2] = m_run == -INFINITY ? -INFINITY : m_run * sc;
      xml[(copy * 32 + lane) * 2 + 1] = l_run;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 softmax warps of query tile 0
      if (copy == 0 && live) {
        float mc[4], wc[4], mx = -INFINITY, l = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          mc[q] = xml[(q * 32 + lane) * 2];
          if (xml[(q * 32 + lane) * 2 + 1] > 0.f) mx = fmaxf(mx, mc[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float lq = xml[(q * 32 + lane) * 2 + 1];
          wc[q] = lq > 0.f ? fast_exp2(mc[q] - mx) : 0.f;
          l += wc[q] * lq;
        }
        const float inv4 = l > 0.f ? 1.f / l : 0.f;
        for (int c = 0; c < D; c += 8) {
          float o8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float acc = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc += wc[q] * xo[(q * 32 + lane) * D + c + e];
            o8[e] = acc;
          }
          if (p_index < 0) {
            __align__(16) __nv_bfloat162 o2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) o2[e] = __floats2bfloat162_rn(o8[2 * e] * inv4, o8[2 * e + 1] * inv4);
            *reinterpret_cast<int4*>(a.out + (int64_t)row * a.ld_out + head * D + c) = *reinterpret_cast<int4*>(o2);
          } else {
            const int64_t slot = ((int64_t)p_index * a.M + row) * a.H + head;
            __stcg(reinterpret_cast<float4*>(a.ws_o + slot * D + c), make_float4(o8[0], o8[1], o8[2], o8[3]));
            __stcg(reinterpret_cast<float4*>(a.ws_o + slot * D + c + 4), make_float4(o8[4], o8[5], o8[6], o8[7]));
            if (c == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml + slot * 2), make_float2(mx, l));
          }
        }
      }
    } else {
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t ov[32];
      sm100::tmem_ld_32x32b_x32(tO + lane_base + c, ov);
      sm100::tmem_ld_wait();
      if (!live) continue;
      const int oc = c;  // O column
      if (p_index < 0) {
        __nv_bfloat16* dst = a.out + (int64_t)row * a.ld_out + head * D + oc;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __align__(16) __nv_bfloat162 o2[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            o2[e] = __floats2bfloat162_rn(__uint_as_float(ov[q * 8 + e * 2]) * inv,
                                          __uint_as_float(ov[q * 8 + e * 2 + 1]) * inv);
          *reinterpret_cast<int4*>(dst + q * 8) = *reinterpret_cast<int4*>(o2);
        }
      } else {
        const int64_t slot = ((int64_t)p_index * a.M + row) * a.H + head;
        float* dst = a.ws_o + slot * D + oc;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          __stcg(reinterpret_cast<float4*>(dst + q * 4),
                 make_float4(__uint_as_float(ov[q * 4]), __uint_as_float(ov[q * 4 + 1]),
                             __uint_as_float(ov[q * 4 + 2]), __uint_as_float(ov[q * 4 + 3])));
        if (oc == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml + slot * 2), make_float2(m_run * sc, l_run));
      }
    }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) sm100::tmem_dealloc<kTmemCols>(tmem);
  if (tid == 0) ATTN_TRACE(4);
}

// Combines the KV-partition partials of the rows whose span was split (sp_np > 1), in partition order.
template <int D>
__global__ void __launch_bounds__(256) attn_grp_merge_kernel(const GrpArgs a) {
  const int row = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  const int np = a.sp_np[a.row_seq[row]];
  if (np <= 1) return;
  constexpr int G8 = D / 8;
  const int n = a.H * G8;
  const int64_t pstride = (int64_t)a.M * a.H;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int head = i / G8, c8 = (i % G8) * 8;
    const int64_t slot0 = (int64_t)row * a.H + head;
    float mx = -INFINITY;
    for (int p = 0; p < np; ++p) mx = fmaxf(mx, __ldcg(a.ws_ml + (slot0 + p * pstride) * 2));
    float l = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int p = 0; p < np; ++p) {
      const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.ws_ml + (slot0 + p * pstride) * 2));
      const float w = ml.y > 0.f ? fast_exp2(ml.x - mx) : 0.f;
      const float4 x0 = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8));
      const float4 x1 = __ldcg(reinterpret_cast<const float4*>(a.ws_o + (slot0 + p * pstride) * D + c8 + 4));
      l += w * ml.y;
      acc[0] += w * x0.x; acc[1] += w * x0.y; acc[2] += w * x0.z; acc[3] += w * x0.w;
      acc[4] += w * x1.x; acc[5] += w * x1.y; acc[6] += w * x1.z; acc[7] += w * x1.w;
    }
    const float inv = l > 0.f ? __fdividef(1.f, l) : 0.f;
    __align__(16) __nv_bfloat162 ov[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) ov[e] = __floats2bfloat162_rn(acc[2 * e] * inv, acc[2 * e + 1] * inv);
    *reinterpret_cast<int4*>(a.out + (int64_t)row * a.ld_out + head * D + c8) = *reinterpret_cast<int4*>(ov);
  }
}

}  // namespace tc

// Query tiles per CTA of the grouped kernel; the planner sizes its items to match (ALORA_ATTN_MT=1 for A/B).
int grp_query_tiles() {
  static const int mt = getenv("ALORA_ATTN_MT") ? std::max(1, std::min(2, atoi(getenv("ALORA_ATTN_MT")))) : 2;
  return mt;
}

template <int D, int MT>
int launch_grp(const tc::GrpArgs& a, int n_items, bool merge, int64_t kv_rows, cudaStream_t st) {
  CUtensorMap tm{};
  if (!make_tmap_2d(&tm, a.kv, (uint64_t)kv_rows, (uint64_t)a.Hkv * D, (uint64_t)a.Hkv * D, a.B, 64))
    return ALORA_ECUDA;
  const int smem = tc::SmemG<D, MT>::kTotal;
  // cp.async producer warps: 2 with two query tiles per CTA, 4 with one at D=128; D=64 with one query tile runs
  // two CTAs per SM (register bound) with the TMA producer. ALORA_ATTN_TMA=1 forces the TMA producer (A/B).
  static const bool force_tma = getenv("ALORA_ATTN_TMA") != nullptr;
  // cp.async producer warps with two query tiles per CTA; one query tile (A/B only) uses the TMA producer
  constexpr int PW = MT == 2 ? 2 : 0;
  const bool use_pw = PW > 0 && !force_tma && a.B % 8 == 0;  // producer lanes assume 8-row swizzle groups per page
  auto kern = use_pw ? tc::attn_grp_kernel<D, PW, MT> : tc::attn_grp_kernel<D, 0, MT>;
  const int threads = use_pw ? tc::kGrpThreads<PW, MT> : tc::kGrpThreads<0, MT>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(tc::attn_grp_kernel<D, PW, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(tc::attn_grp_kernel<D, 0, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
            cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  tc::GrpArgs ta = a;
  static const bool timeline = getenv("ALORA_ATTN_TL") != nullptr;
  static long long* tlbuf = nullptr;
  if (timeline) {
    if (!tlbuf) cudaMalloc(&tlbuf, sizeof(long long) * 9 * 2 * 256);
    cudaMemsetAsync(tlbuf, 0, sizeof(long long) * 9 * 2 * 256, st);
    ta.tl = tlbuf;
  }
  static const bool tracing = getenv("ALORA_ATTN_TRACE") != nullptr;
  static unsigned long long* tbuf = nullptr;
  const dim3 grid(n_items, a.Hkv);
  const int n_ctas = n_items * a.Hkv;
  if (tracing) {
    if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * 6 * 65536);
    cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * 6 * std::min(n_ctas, 65536), st);
    ta.trace = n_ctas <= 65536 ? tbuf : nullptr;
  }
  ALORA_CUDA_CHECK(launch_pdl(kern, grid, dim3(threads), smem, st, nullptr, 0, ta, tm));
  ALORA_LAUNCH_CHECK();
  if (tracing && ta.trace) {
    std::vector<unsigned long long> h(6 * n_ctas);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0, longest = 0;
    double ph[4] = {0, 0, 0, 0};
    int live = 0;
    for (int c = 0; c < n_ctas; ++c) {
      if (!h[6 * c] || !h[6 * c + 4]) continue;
      ++live;
      t0 = std::min(t0, h[6 * c]);
      t1 = std::max(t1, h[6 * c + 4]);
      longest = std::max(longest, h[6 * c + 4] - h[6 * c]);
      for (int p = 0; p < 4; ++p)
        if (h[6 * c + p + 1] && h[6 * c + p]) ph[p] += double(h[6 * c + p + 1] - h[6 * c + p]);
    }
    if (live)
      fprintf(stderr, "[attn grp trace] ctas %d/%d span %.2f us (longest CTA %.2f); mean start->Q %.2f, Q->S0 %.2f, "
              "S0->last P %.2f, ->end %.2f us\n", live, n_ctas, (t1 - t0) / 1e3, longest / 1e3, ph[0] / live / 1e3,
              ph[1] / live / 1e3, ph[2] / live / 1e3, ph[3] / live / 1e3);
  }
  if (timeline) {  // per-tile means over CTA (0, 0), SM cycles
    std::vector<long long> h(9 * 2 * 256);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), tlbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    auto at = [&](int ev, int x, int t) { return h[(ev * 2 + x) * 256 + t]; };
    for (int x = 0; x < MT; ++x) {
      double soft = 0, wait_s = 0, s_lat = 0, pv_lag = 0, pwait = 0, ph_ld = 0, ph_max = 0, ph_exp = 0, ph_st = 0,
             ph_fence = 0;
      int n = 0;
      for (int t = 2; t < 250; ++t) {
        if (!at(0, x, t) || !at(1, x, t) || !at(2, x, t) || !at(3, x, t) || !at(1, x, t - 1)) break;
        soft += at(1, x, t) - at(0, x, t);        // softmax: S in hand -> P published
        wait_s += at(0, x, t) - at(1, x, t - 1);  // softmax idle before S_t
        s_lat += at(0, x, t) - at(2, x, t);       // S_t issued -> softmax has it
        pv_lag += at(3, x, t) - at(1, x, t);      // P_t published -> PV_t issued
        pwait += at(5, x, t) - at(4, x, t);       // softmax waiting for PV_{t-NP} before writing P_t
        ph_ld += at(6, x, t) - at(0, x, t);       // S -> registers
        ph_max += at(7, x, t) - at(6, x, t);      // mask, row max, lazy rescale
        ph_exp += at(4, x, t) - at(7, x, t);      // exponentials, row sum, P packing
        ph_st += at(8, x, t) - at(5, x, t);       // P stores
        ph_fence += at(1, x, t) - at(8, x, t);    // proxy fence + arrive
        ++n;
      }
      if (n)
        fprintf(stderr, "[attn grp timeline] tile %d: %d tiles, per tile (cycles): softmax %.0f, softmax idle %.0f, "
                "S issue->softmax %.0f, P->PV issue %.0f, P-buffer wait %.0f, period %.0f\n", x, n, soft / n,
                wait_s / n, s_lat / n, pv_lag / n, pwait / n, double(at(1, x, n + 1) - at(1, x, 1)) / n);
      if (n)
        fprintf(stderr, "[attn grp timeline] tile %d softmax phases (cycles): S->regs %.0f, max/rescale %.0f, exp %.0f, "
                "P stores %.0f, fence+arrive %.0f\n", x, ph_ld / n, ph_max / n, ph_exp / n, ph_st / n, ph_fence / n);
    }
  }
  if (merge) {
    ALORA_CUDA_CHECK(launch_pdl(tc::attn_grp_merge_kernel<D>, dim3(a.M), dim3(256), 0, st, nullptr, 0, ta));
    ALORA_LAUNCH_CHECK();
  }
  return ALORA_OK;
}

// ============================================================================================================
// Decode attention (every sequence of the step has ONE query row): G = H/Hkv query heads share a kv head, so
// a work item is G rows -- far below a 128-row tcgen05 tile (4 live rows of 128 at G=4, one live softmax
// warp whose per-tile chain bounded the tcgen05 kernel at ~20 us per layer for 12 x 2k contexts). Here:
//   the keys are split into more partitions (~3 CTAs per SM); each of the 4 warps of a CTA owns every 4th
//   32-key chunk of the partition and its own 2-stage smem ring filled by TMA page boxes [B keys x 64 dims]
//   (SW128-swizzled, as in the tcgen05 kernel), so warps never synchronise until the end;
//   S = Q K^T and O += P V run as warp-level mma.sync m16n8k16 (rows = the G heads, zero-padded to 16;
//   K/V fragments by ldmatrix from the swizzled chunk), P stays in registers (S accumulator -> A fragment);
//   online softmax per head in fp32 with exp2, scale applied to the fp32 scores.
// Warp-level MMA is the right unit here: 16-row fragments waste 12 of 16 rows instead of 124 of 128, and the
// kernel is bound by HBM and per-chunk latency, not by tensor throughput.
// ============================================================================================================
constexpr int kDecWarpsSplit = 4;  // warps per CTA when the keys are split into partitions
// warps per CTA when one CTA covers a (sequence, kv head): each warp's 2-stage ring is 8 KB x D/64, so D=128
// stays at 4 warps (128 KB) -- 8 would need 256 KB of shared memory
template <int D>
constexpr int kDecWarpsWhole = D == 64 ? 8 : 4;
// resident split-mode CTAs per SM (shared memory bound): 3 at D=64 (66 KB), 1 at D=128 (130 KB)
template <int D>
constexpr int kDecSplitCtasPerSm = D == 64 ? 3 : 1;
constexpr int kDecMaxG = 8;
constexpr int kDecKeys = 32;  // keys per chunk (one per lane)

template <int D, int W>
struct DecSmem {
  static constexpr int kTile = kDecKeys * D * 2;           // one K (or V) chunk: [D/64][32][64] bf16
  static constexpr int kStage = 2 * kTile;                 // K | V
  // ring stages per warp: 3 for the 8-warp whole-sequence CTA at D=64 (one CTA per SM, 192 KB in flight)
  static constexpr int kNS = (D == 64 && W == 8) ? 3 : 2;
  static constexpr int kWarp = kNS * kStage;
  static constexpr int kRing = W * kWarp;
  static constexpr int kTotal = kRing + 1024 + 256;        // + alignment slack + barriers
};

template <int D, int G, int W>
__global__ void __launch_bounds__(32 * W) attn_decode_kernel(const AttnArgs a,
                                                                   const __grid_constant__ CUtensorMap tm_kv) {
  using L = DecSmem<D, W>;
  constexpr int DL = D / 32;  // dims per lane in the PV accumulation (2 for D=64)
  extern __shared__ uint8_t smem_dec_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dec_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + L::kRing);  // [warps][NS]
  __shared__ float sm_m[W][G], sm_l[W][G];
  __shared__ float so[W][G][D];
  __shared__ int s_last;
  const int s = blockIdx.z / a.Hkv, kvh = blockIdx.z % a.Hkv;
  const int part = blockIdx.y;
  const int row = a.cu_q[s];
  const int start = a.start_pos[s];
  const int key_begin = part * a.part_size;
  const int key_end = min(start + 1, key_begin + a.part_size);
  if (key_begin >= key_end) return;
  const int parts_here = min(a.n_parts, (start + a.part_size) / a.part_size);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* bt = a.block_table + (int64_t)s * a.max_blocks;
  const int last_blk = (key_end - 1) / a.B;
  const int per_chunk = kDecKeys / a.B;  // pages per chunk (B divides 32)
  const int n_chunks = (key_end - key_begin + kDecKeys - 1) / kDecKeys;
  uint8_t* wring = ring + warp * L::kWarp;
  uint64_t* wfull = full + warp * L::kNS;
  if (lane == 0) {
    sm100::prefetch_tmap(&tm_kv);
    for (int i = 0; i < L::kNS; ++i) sm100::mbar_init(&wfull[i], 1);
    sm100::fence_barrier_init();
  }
  __syncwarp();
  const uint64_t pol = sm100::policy_evict_first();
  auto issue = [&](int c, int st) {  // chunk c (partition-relative) of this warp into stage st
    uint8_t* dk = wring + st * L::kStage;
    uint8_t* dv = dk + L::kTile;
    sm100::mbar_arrive_expect_tx(&wfull[st], L::kStage);
    const int b0 = (key_begin + c * kDecKeys) / a.B;
    for (int j = 0; j < per_chunk; ++j) {
      const int64_t blk = bt[min(b0 + j, last_blk)];  // past the end: a valid duplicate, masked below
      const int rowk = (int)(((blk * a.n_layers + a.layer) * 2) * a.B);
#pragma unroll
      for (int sub = 0; sub < D / 64; ++sub) {
        sm100::tma_load_2d(dk + sub * kDecKeys * 128 + j * a.B * 128, &tm_kv, &wfull[st], kvh * D + sub * 64, rowk, pol);
        sm100::tma_load_2d(dv + sub * kDecKeys * 128 + j * a.B * 128, &tm_kv, &wfull[st], kvh * D + sub * 64,
                           rowk + a.B, pol);
      }
    }
  };
  // chunks of this warp: c = warp, warp + 4, ...; the cached prefix streams in before the dependency wait
  // (only the step's last key -- the row being decoded -- is written by the kernel before this one)
  const int cached_end = (start / a.B) * a.B;
  int issued = 0;
  if (lane == 0)
    for (int c = warp; issued < L::kNS && c < n_chunks; c += W, ++issued) {
      if (key_begin + (c + 1) * kDecKeys > cached_end) break;
      issue(c, issued);
    }
  issued = __shfl_sync(0xffffffffu, issued, 0);
  pdl_wait();  // q and this step's K/V row come from the kernels before
  pdl_trigger();
  if (lane == 0)
    for (int k = issued, c = warp + issued * W; k < L::kNS && c < n_chunks; ++k, c += W) issue(c, k);
  // Q as mma.sync A fragments: row = lane/4 is query head g (rows >= G and the upper 8 rows are zero)
  const int qg = lane >> 2, qt4 = lane & 3;
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const uint32_t* qr = reinterpret_cast<const uint32_t*>(a.q + (int64_t)row * a.ld_q + (kvh * G + qg) * D + kk * 16);
    qf[kk][0] = qg < G ? qr[qt4] : 0u;
    qf[kk][1] = 0u;
    qf[kk][2] = qg < G ? qr[4 + qt4] : 0u;
    qf[kk][3] = 0u;
  }
  // swizzled element offset of (row, 16-byte unit u) in a [D/64][32][64] chunk tile (TMA SW128 boxes)
  auto sw = [](int r, int u) { return (u >> 3) * kDecKeys * 64 + r * 64 + (((u & 7) ^ (r & 7)) << 3); };
  int koff[2][D / 16], voff[D / 16];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
    for (int jn = 0; jn < 2; ++jn)
      koff[jn][kk] = sw(jn * 16 + (lane & 7) + (lane >> 4) * 8, kk * 2 + ((lane >> 3) & 1));
    voff[kk] = sw(lane & 15, kk * 2 + (lane >> 4)) - (lane & 15) * 64;  // + row term added per key block
  }
  const float scl = a.scale_log2;
  float m_run = -INFINITY, l_run = 0.f;  // row qg
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  int it = 0;
  for (int c = warp; c < n_chunks; c += W, ++it) {
    const int st = it % L::kNS;
    sm100::mbar_wait(&wfull[st], (it / L::kNS) & 1);
    const __nv_bfloat16* sk = reinterpret_cast<const __nv_bfloat16*>(wring + st * L::kStage);
    const __nv_bfloat16* sv = sk + kDecKeys * D;
    const int c0 = key_begin + c * kDecKeys;
    float sc4[4][4];  // S = Q K^T: 16 rows x 32 keys (n-tiles of 8 keys)
#pragma unroll
    for (int j = 0; j < 4; ++j) sc4[j][0] = sc4[j][1] = sc4[j][2] = sc4[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) {
        uint32_t bfr[4];
        ldsm_x4(bfr, sk + koff[jn][kk]);
        mma16816(sc4[2 * jn], qf[kk], bfr[0], bfr[1]);
        mma16816(sc4[2 * jn + 1], qf[kk], bfr[2], bfr[3]);
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float v = sc4[j][e] * scl;
        if (c0 + j * 8 + 2 * qt4 + e >= key_end) v = -INFINITY;
        sc4[j][e] = v;
        mx = fmaxf(mx, v);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);  // finite: every chunk holds at least one valid key
    const float corr = fast_exp2(m_run - m_new);
    m_run = m_new;
    float rs = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sc4[j][0] = fast_exp2(sc4[j][0] - m_new);
      sc4[j][1] = fast_exp2(sc4[j][1] - m_new);
      rs += sc4[j][0] + sc4[j][1];
    }
    l_run = l_run * corr + rs;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) { o[j][0] *= corr; o[j][1] *= corr; }
    // O += P V (P from the S accumulators; the dead upper 8 rows stay zero)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(sc4[2 * kk][0], sc4[2 * kk][1]);
      pa[1] = 0u;
      pa[2] = pack_bf16(sc4[2 * kk + 1][0], sc4[2 * kk + 1][1]);
      pa[3] = 0u;
#pragma unroll
      for (int jd = 0; jd < D / 16; ++jd) {
        uint32_t bfr[4];
        ldsm_x4_t(bfr, sv + (kk * 16 + (lane & 15)) * 64 + voff[jd]);
        mma16816(o[2 * jd], pa, bfr[0], bfr[1]);
        mma16816(o[2 * jd + 1], pa, bfr[2], bfr[3]);
      }
    }
    // this stage is consumed: refill it with chunk c + NS*4 (generic reads -> async-proxy writes)
    __syncwarp();
    if (lane == 0 && c + L::kNS * W < n_chunks) {
      sm100::fence_proxy_async_smem();
      issue(c + L::kNS * W, st);
    }
    __syncwarp();
  }
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  if (qg < G) {
    if (qt4 == 0) {
      sm_m[warp][qg] = m_run;
      sm_l[warp][qg] = l_run;
    }
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      so[warp][qg][j * 8 + 2 * qt4] = o[j][0];
      so[warp][qg][j * 8 + 2 * qt4 + 1] = o[j][1];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += blockDim.x) {
    const int g = i / D, d = i % D;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < W; ++w) mx = fmaxf(mx, sm_m[w][g]);
    float l = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float f = sm_m[w][g] == -INFINITY ? 0.f : fast_exp2(sm_m[w][g] - mx);
      l += f * sm_l[w][g];
      acc += f * so[w][g][d];
    }
    const int head = kvh * G + g;
    if (parts_here == 1) {
      a.out[(int64_t)row * a.ld_out + head * D + d] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
    } else {
      const int64_t slot = ((int64_t)part * a.M + row) * a.H + head;
      __stcg(a.ws_o + slot * D + d, acc);
      if (d == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml + slot * 2), make_float2(mx, l));
    }
  }
  if (parts_here > 1) merge_partials<D>(a, s, kvh, 0, row, start, G, parts_here, G, &s_last);
}

template <int D, int G, int W>
int launch_decode_g(const AttnArgs& a, dim3 grid, const CUtensorMap& tm, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_decode_kernel<D, G, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DecSmem<D, W>::kTotal) != cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  ALORA_CUDA_CHECK(launch_pdl(attn_decode_kernel<D, G, W>, grid, dim3(32 * W), DecSmem<D, W>::kTotal, st, nullptr,
                              0, a, tm));
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

template <int D>
int launch_decode(const AttnArgs& a, dim3 grid, int G, int64_t kv_rows, cudaStream_t st) {
  CUtensorMap tm{};
  if (!make_tmap_2d(&tm, a.kv, (uint64_t)kv_rows, (uint64_t)a.Hkv * D, (uint64_t)a.Hkv * D, a.B, 64))
    return ALORA_ECUDA;
  // one CTA per (sequence, kv head) with 8 warps when that alone fills most SMs (no partition merge),
  // otherwise 4-warp CTAs over key partitions
  const bool whole = a.n_parts == 1;
  switch (G) {
    case 1: return whole ? launch_decode_g<D, 1, kDecWarpsWhole<D>>(a, grid, tm, st)
                         : launch_decode_g<D, 1, kDecWarpsSplit>(a, grid, tm, st);
    case 2: return whole ? launch_decode_g<D, 2, kDecWarpsWhole<D>>(a, grid, tm, st)
                         : launch_decode_g<D, 2, kDecWarpsSplit>(a, grid, tm, st);
    case 4: return whole ? launch_decode_g<D, 4, kDecWarpsWhole<D>>(a, grid, tm, st)
                         : launch_decode_g<D, 4, kDecWarpsSplit>(a, grid, tm, st);
    case 8: return whole ? launch_decode_g<D, 8, kDecWarpsWhole<D>>(a, grid, tm, st)
                         : launch_decode_g<D, 8, kDecWarpsSplit>(a, grid, tm, st);
    default: return ALORA_EINVAL;
  }
}

// Decode plan: with at least ~half an SM-count of (sequence, kv head) units, one 8-warp CTA per unit
// covers all its keys (no partition merge); below that, 4-warp CTAs over key partitions (~3 per SM).
void plan_decode(int n_seqs, int max_ctx, int Hkv, int D, int& part_size, int& n_parts) {
  const int units = std::max(1, n_seqs * Hkv);
  static const int whole_min = getenv("ALORA_DEC_WHOLE_MIN") ? atoi(getenv("ALORA_DEC_WHOLE_MIN")) : kNumSMs / 2;
  if (units >= whole_min) {
    n_parts = 1;
    part_size = (max_ctx + 31) / 32 * 32;
    return;
  }
  const int slots = (D == 64 ? kDecSplitCtasPerSm<64> : kDecSplitCtasPerSm<128>) * kNumSMs;
  int np = std::max(1, std::min({kMaxParts, slots / units, (max_ctx + kMinPartKeys - 1) / kMinPartKeys}));
  int ps = (max_ctx + np - 1) / np;
  ps = (ps + 31) / 32 * 32;
  n_parts = (max_ctx + ps - 1) / ps;
  part_size = ps;
}

// Partition plan shared by the workspace query and the launch. When the step has fewer work items than
// resident CTA slots (aLoRA suffix turns, decode) the keys are split so that all partitions run in ONE wave:
// a second wave would double the per-CTA fixed cost (setup, Q load, merge) on the critical path.
void plan(int n_seqs, int max_q, int max_ctx, int H, int Hkv, int D, int& part_size, int& n_parts, int& n_qtiles) {
  const int G = H / Hkv;
  n_qtiles = (max_q * G + kQT - 1) / kQT;
  const int64_t items = (int64_t)n_qtiles * n_seqs * Hkv;
  const int slots = D == 64 ? kTargetCtas : kNumSMs;  // resident tcgen05 CTAs (smem/TMEM bound)
  const int max_parts = (max_ctx + kMinPartKeys - 1) / kMinPartKeys;
  int np = 1;
  if (items < slots && items <= kMaxCounters) np = (int)(slots / items);
  np = std::max(1, std::min({np, max_parts, kMaxParts}));
  int ps = (max_ctx + np - 1) / np;
  ps = (ps + kKT - 1) / kKT * kKT;
  n_parts = (max_ctx + ps - 1) / ps;
  part_size = ps;
}

template <int D>
int launch_attn(const AttnArgs& a, int n_seqs, int64_t kv_rows, cudaStream_t st) {
  dim3 grid(a.n_qtiles, a.n_parts, n_seqs * a.Hkv);
  static const bool force_mma = getenv("ALORA_ATTN_MMA") != nullptr;  // A/B switch to the mma.sync kernel
  // the tcgen05 kernel loads pages with TMA boxes of [B x 64]: B must tile the 64-key KV tile
  // the tcgen05 kernel loads pages with TMA boxes of [B x 64]: B must tile the 64-key KV tile
  const bool use_tc = !force_mma && a.B <= kKT && kKT % a.B == 0 && kv_rows > 0 && kv_rows < (1ll << 31);
  CUtensorMap tm{};
  if (use_tc && !make_tmap_2d(&tm, a.kv, (uint64_t)kv_rows, (uint64_t)a.Hkv * D, (uint64_t)a.Hkv * D, a.B, 64))
    return ALORA_ECUDA;
  if (!use_tc) {
    const int smem = (kQT + 2 * kStagesA * kKT) * D * 2;
    static bool configured = false;
    if (!configured) {
      if (cudaFuncSetAttribute(attn_bf16_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return ALORA_ECUDA;
      configured = true;
    }
    attn_bf16_kernel<D><<<grid, kThreadsA, smem, st>>>(a);
  } else {
    const int smem = tc::Smem<D>::kTotal;
    static bool configured = false;
    if (!configured) {
      if (cudaFuncSetAttribute(tc::attn_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return ALORA_ECUDA;
      configured = true;
    }
    static const bool tracing = getenv("ALORA_ATTN_TRACE") != nullptr;
    static unsigned long long* tbuf = nullptr;
    const int n_ctas = grid.x * grid.y * grid.z;
    AttnArgs ta = a;
    static const int exp_mode = getenv("ALORA_ATTN_EXP") ? atoi(getenv("ALORA_ATTN_EXP")) : 0;
    ta.exp = exp_mode;
    if (tracing) {
      if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * 6 * 65536);
      cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * 6 * n_ctas, st);
      ta.trace = tbuf;
    }
    ALORA_CUDA_CHECK(launch_pdl(tc::attn_tc_kernel<D>, grid, dim3(tc::kThreads), smem, st, nullptr, 0, ta, tm));
    if (tracing) {  // debug: per-phase means over the CTAs that ran (early-exit CTAs have no stamps)
      std::vector<unsigned long long> h(6 * n_ctas);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, t1 = 0;
      double ph[5] = {0, 0, 0, 0, 0};
      int live = 0;
      for (int c = 0; c < n_ctas; ++c) {
        if (!h[6 * c] || !h[6 * c + 5]) continue;
        ++live;
        t0 = std::min(t0, h[6 * c]);
        t1 = std::max(t1, h[6 * c + 5]);
        for (int p = 0; p < 5; ++p)
          if (h[6 * c + p + 1] && h[6 * c + p]) ph[p] += double(h[6 * c + p + 1] - h[6 * c + p]);
      }
      unsigned long long last_start = 0, max_dur = 0;
      for (int c = 0; c < n_ctas; ++c) {
        if (!h[6 * c] || !h[6 * c + 5]) continue;
        last_start = std::max(last_start, h[6 * c] - t0);
        max_dur = std::max(max_dur, h[6 * c + 5] - h[6 * c]);
      }
      fprintf(stderr, "[attn trace] ctas %d/%d span %.2f us (last CTA start +%.2f, longest CTA %.2f); mean start->Q "
              "%.2f, Q->S0 %.2f, S0->last P %.2f, ->epilogue %.2f, merge %.2f us (parts %d, part keys %d)\n", live,
              n_ctas, (t1 - t0) / 1e3, last_start / 1e3, max_dur / 1e3, ph[0] / live / 1e3, ph[1] / live / 1e3,
              ph[2] / live / 1e3, ph[3] / live / 1e3, ph[4] / live / 1e3, a.n_parts, a.part_size);
    }
  }
  ALORA_LAUNCH_CHECK();
  return ALORA_OK;
}

}  // namespace

void configure_attention() {
  prefer_max_smem(attn_bf16_kernel<64>);
  prefer_max_smem(attn_bf16_kernel<128>);
  prefer_max_smem(tc::attn_tc_kernel<64>);
  prefer_max_smem(tc::attn_tc_kernel<128>);
}

// Upper bound over all steps: a split happens only when items < kTargetCtas; then every item covers <= kQT
// packed rows, so n_parts * M * H <= kQT * (kTargetCtas + items) < 2 * kQT * kTargetCtas.
int64_t attn_bf16_workspace_bound(int H, int D) {
  (void)H;
  return (int64_t)2 * kTargetCtas * kQT * (D + 2) * 4 + (int64_t)kMaxCounters * 4;
}

int64_t attn_bf16_workspace(int M, int n_seqs, int max_q, int max_ctx, int H, int Hkv, int D) {
  int ps, np, nq;
  plan(n_seqs, max_q, max_ctx, H, Hkv, D, ps, np, nq);
  if (max_q == 1 && H / Hkv <= kDecMaxG) {
    int dps, dnp;
    plan_decode(n_seqs, max_ctx, Hkv, D, dps, dnp);
    np = std::max(np, dnp);
  }
  if (np <= 1) return 0;
  return (int64_t)np * M * H * (D + 2) * 4 + (int64_t)kMaxCounters * 4;
}

int attn_bf16(const __nv_bfloat16* q, int64_t ld_q, int M, int n_seqs, const int32_t* cu_q, const int32_t* start_pos,
              const int32_t* block_table, int max_blocks, int max_q, int max_ctx, const __nv_bfloat16* kv,
              int n_layers, int layer, int B, int H, int Hkv, int D, __nv_bfloat16* out, int64_t ld_out, void* ws,
              int64_t ws_bytes, cudaStream_t st, int total_blocks) {
  if (M == 0 || n_seqs == 0) return ALORA_OK;
  if (H % Hkv || (D != 64 && D != 128) || ld_q % 8 || ld_out % 8 || max_q < 1 || max_ctx < 1) return ALORA_EINVAL;
  AttnArgs a{};
  a.q = q; a.ld_q = ld_q; a.cu_q = cu_q; a.start_pos = start_pos; a.block_table = block_table;
  a.max_blocks = max_blocks; a.kv = kv; a.n_layers = n_layers; a.layer = layer; a.B = B; a.H = H; a.Hkv = Hkv;
  a.D = D; a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  a.out = out; a.ld_out = ld_out; a.M = M;
  static const bool no_dec = getenv("ALORA_ATTN_NO_DECODE") != nullptr;  // A/B switch
  const int Gq = H / Hkv;
  const int64_t kv_rows_all = (int64_t)total_blocks * n_layers * 2 * B;
  const bool decode = !no_dec && !g_batch_invariant && max_q == 1 && (Gq == 1 || Gq == 2 || Gq == 4 || Gq == 8) &&
                      total_blocks > 0 &&
                      B <= kDecKeys && kDecKeys % B == 0 && kv_rows_all < (1ll << 31);
  if (decode) {
    plan_decode(n_seqs, max_ctx, Hkv, D, a.part_size, a.n_parts);
    a.n_qtiles = 1;
    // fewer partitions when the caller's workspace cannot hold them (it is sized by attn_bf16_workspace_bound)
    while (a.n_parts > 1 && (ws == nullptr || ws_bytes < (int64_t)a.n_parts * M * H * (D + 2) * 4 +
                                                             (int64_t)kMaxCounters * 4)) {
      a.part_size = ((max_ctx + a.n_parts - 2) / (a.n_parts - 1) + 31) / 32 * 32;
      a.n_parts = (max_ctx + a.part_size - 1) / a.part_size;
    }
  } else {
    plan(n_seqs, max_q, max_ctx, H, Hkv, D, a.part_size, a.n_parts, a.n_qtiles);
    if (g_batch_invariant) {  // one partition: a row's key tiles and softmax order never depend on the step
      a.n_parts = 1;
      a.part_size = (max_ctx + kKT - 1) / kKT * kKT;
    }
  }
  if (a.n_parts > 1) {
    const int64_t need = (int64_t)a.n_parts * M * H * (D + 2) * 4 + (int64_t)kMaxCounters * 4;
    if (ws == nullptr || ws_bytes < need) return ALORA_EINVAL;
    // counters live at the END of the caller's buffer so their position does not depend on the step shape
    a.counters = reinterpret_cast<int*>(static_cast<char*>(ws) + ws_bytes - (int64_t)kMaxCounters * 4);
    a.ws_o = static_cast<float*>(ws);
    a.ws_ml = a.ws_o + (int64_t)a.n_parts * M * H * D;
  }
  if (decode) {
    const dim3 grid(1, a.n_parts, n_seqs * Hkv);
    return D == 64 ? launch_decode<64>(a, grid, Gq, kv_rows_all, st) : launch_decode<128>(a, grid, Gq, kv_rows_all, st);
  }
  const int64_t kv_rows = (int64_t)total_blocks * n_layers * 2 * B;
  return D == 64 ? launch_attn<64>(a, n_seqs, kv_rows, st) : launch_attn<128>(a, n_seqs, kv_rows, st);
}

int attn_grouped(const __nv_bfloat16* q, int64_t ld_q, int M, int S, const int32_t* positions, const int32_t* row_seq,
                 const int32_t* block_table, int max_blocks, const int32_t* plan, int n_items, int n_segs, int n_sets,
                 int max_np, bool merge, const __nv_bfloat16* kv, int total_blocks, int n_layers, int layer, int B,
                 int H, int Hkv, int D, __nv_bfloat16* out, int64_t ld_out, void* ws, int64_t ws_bytes,
                 cudaStream_t st) {
  if (M == 0 || n_items == 0) return ALORA_OK;
  if (H % Hkv || (D != 64 && D != 128) || ld_q % 8 || ld_out % 8 || !plan || !positions || !row_seq ||
      B > kKT || kKT % B || total_blocks < 1)
    return ALORA_EINVAL;
  const int64_t kv_rows = (int64_t)total_blocks * n_layers * 2 * B;
  if (kv_rows >= (1ll << 31)) return ALORA_EINVAL;
  tc::GrpArgs a{};
  a.q = q; a.ld_q = ld_q; a.positions = positions; a.row_seq = row_seq; a.block_table = block_table;
  a.max_blocks = max_blocks;
  a.items = plan + 8;
  a.segs = a.items + 8LL * n_items;
  a.sets = a.segs + 4LL * n_segs;
  a.set_tok = a.sets + 2LL * n_sets;
  a.sp_np = a.set_tok + M;
  a.kv = kv; a.n_layers = n_layers; a.layer = layer; a.B = B; a.H = H; a.Hkv = Hkv;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  a.out = out; a.ld_out = ld_out; a.M = M;
  if (max_np > 1) {
    const int64_t need = (int64_t)max_np * M * H * (D + 2) * 4;
    if (!ws || ws_bytes < need) return ALORA_EINVAL;
    a.ws_o = static_cast<float*>(ws);
    a.ws_ml = a.ws_o + (int64_t)max_np * M * H * D;
  }
  static const int exp_mode = getenv("ALORA_ATTN_EXP") ? atoi(getenv("ALORA_ATTN_EXP")) : 0;
  a.exp = exp_mode;
  (void)S;
  const bool mg = merge && max_np > 1;
  if (grp_query_tiles() == 2)
    return D == 64 ? launch_grp<64, 2>(a, n_items, mg, kv_rows, st) : launch_grp<128, 2>(a, n_items, mg, kv_rows, st);
  return D == 64 ? launch_grp<64, 1>(a, n_items, mg, kv_rows, st) : launch_grp<128, 1>(a, n_items, mg, kv_rows, st);
}

}  // namespace alora
