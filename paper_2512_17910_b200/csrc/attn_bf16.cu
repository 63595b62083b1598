// Paged causal prefill attention, bf16 tier (model.py:149-187 generalised to GQA).
//
// Work item = (sequence, kv head, 64-row query tile, KV partition). Query rows
// are GQA-packed: row r of a sequence's tile space is (token r / G, q head
// kvh*G + r % G), so one K/V tile read from HBM serves all G query heads that
// share it. K/V tiles of 64 keys are gathered page by page through the block
// table with cp.async (16-byte chunks, XOR-swizzled smem rows, double
// buffered); QK^T and PV use mma.sync m16n8k16 bf16 with fp32 accumulation and
// an fp32 online softmax (exp2). When a step has too few work items to fill
// the 148 SMs (the aLoRA suffix turn: few query rows, long cached prefix) the
// key range is split into partitions whose partial (m, l, O) are merged by a
// second kernel in a fixed partition order.

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace alora {

namespace {

constexpr int kQT = 64;       // packed query rows per CTA
constexpr int kKT = 64;       // keys per KV tile
constexpr int kThreadsA = 128;
constexpr int kTargetCtas = 2 * kNumSMs;

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
  int part_size;     // keys per partition (multiple of kKT); >= max_ctx when not split
  int n_parts;
  __nv_bfloat16* out;
  int64_t ld_out;
  float* ws_o;  // [n_parts][M*H][D] when split
  float* ws_ml; // [n_parts][M*H][2]
  int M;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
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
__global__ void __launch_bounds__(kThreadsA) attn_bf16_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_attn[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sK = sQ + kQT * D;       // [2][kKT][D]
  __nv_bfloat16* sV = sK + 2 * kKT * D;   // [2][kKT][D]

  const int G = a.H / a.Hkv;
  const int s = blockIdx.z / a.Hkv, kvh = blockIdx.z % a.Hkv;
  const int qt = blockIdx.x, part = blockIdx.y;
  const int row0 = a.cu_q[s];
  const int n_tok = a.cu_q[s + 1] - row0;
  const int R = n_tok * G;
  if (qt * kQT >= R) return;
  const int start = a.start_pos[s];
  const int last_tok = min(n_tok - 1, (qt * kQT + kQT - 1) / G);
  const int key_end = min(start + last_tok + 1, (part + 1) * a.part_size);  // exclusive
  const int key_begin = part * a.part_size;
  if (key_begin >= key_end) return;  // nothing visible in this partition for any row of the tile

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kvw = a.Hkv * D;
  const int32_t* bt = a.block_table + (int64_t)s * a.max_blocks;
  constexpr int CH = D / 8;  // 16-byte chunks per row

  // ---- Q tile (packed rows) -> smem
  for (int i = tid; i < kQT * CH; i += kThreadsA) {
    const int r = i / CH, c = i % CH;
    const int pr = qt * kQT + r;
    const bool valid = pr < R;
    const int tok = valid ? pr / G : 0, g = valid ? pr % G : 0;
    const __nv_bfloat16* src = a.q + (int64_t)(row0 + tok) * a.ld_q + (kvh * G + g) * D + c * 8;
    cp_async16(tile_ptr<D>(sQ, r, c * 8), valid ? src : a.q, valid);
  }
  auto load_kv = [&](int buf, int k0) {
    __nv_bfloat16* dk = sK + buf * kKT * D;
    __nv_bfloat16* dv = sV + buf * kKT * D;
    for (int i = tid; i < kKT * CH; i += kThreadsA) {
      const int r = i / CH, c = i % CH;
      const int t = k0 + r;
      const bool valid = t < key_end;
      const __nv_bfloat16* ksrc = a.kv;
      if (valid) {
        const int64_t blk = bt[t / a.B];
        ksrc = a.kv + ((((blk * a.n_layers + a.layer) * 2) * a.B + (t % a.B)) * (int64_t)kvw) + kvh * D + c * 8;
      }
      cp_async16(tile_ptr<D>(dk, r, c * 8), ksrc, valid);
      cp_async16(tile_ptr<D>(dv, r, c * 8), valid ? ksrc + (int64_t)a.B * kvw : a.kv, valid);
    }
  };
  load_kv(0, key_begin);
  cp_async_commit();

  // per-thread rows: lane/4 and lane/4 + 8 of this warp's 16-row slice
  const int wr = warp * 16;
  int pos_r[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int pr = qt * kQT + wr + (lane >> 2) + h * 8;
    pos_r[h] = pr < R ? start + pr / G : -1;
  }
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  uint32_t qf[D / 16][4];

  const int n_tiles = (key_end - key_begin + kKT - 1) / kKT;
  for (int it = 0; it < n_tiles; ++it) {
    const int k0 = key_begin + it * kKT;
    if (it + 1 < n_tiles) load_kv((it + 1) & 1, k0 + kKT);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (it == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ldsm_x4(qf[kk], tile_ptr<D>(sQ, wr + (lane & 15), kk * 16 + (lane >> 4) * 8));
    }
    const __nv_bfloat16* cK = sK + (it & 1) * kKT * D;
    const __nv_bfloat16* cV = sV + (it & 1) * kKT * D;
    // S = Q K^T  (16 x 64 per warp)
    float sc[kKT / 8][4];
#pragma unroll
    for (int j = 0; j < kKT / 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int jn = 0; jn < kKT / 16; ++jn) {
        uint32_t b[4];
        const int key = jn * 16 + (lane & 7) + (lane >> 4) * 8;
        ldsm_x4(b, tile_ptr<D>(const_cast<__nv_bfloat16*>(cK), key, kk * 16 + ((lane >> 3) & 1) * 8));
        mma16816(sc[2 * jn], qf[kk], b[0], b[1]);
        mma16816(sc[2 * jn + 1], qf[kk], b[2], b[3]);
      }
    }
    // mask + online softmax (log2 domain)
    float mnew[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float mx = m_r[h];
#pragma unroll
      for (int j = 0; j < kKT / 8; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = k0 + j * 8 + 2 * (lane & 3) + e;
          float v = sc[j][h * 2 + e] * a.scale_log2;
          if (key > pos_r[h] || key >= key_end) v = -INFINITY;
          sc[j][h * 2 + e] = v;
          mx = fmaxf(mx, v);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[h] = mx;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float base = mnew[h] == -INFINITY ? 0.f : mnew[h];
      const float corr = exp2f(m_r[h] - base);
#pragma unroll
      for (int j = 0; j < D / 8; ++j) { o[j][h * 2] *= corr; o[j][h * 2 + 1] *= corr; }
      l_r[h] *= corr;
      m_r[h] = mnew[h];
#pragma unroll
      for (int j = 0; j < kKT / 8; ++j) {
        sc[j][h * 2] = exp2f(sc[j][h * 2] - base);
        sc[j][h * 2 + 1] = exp2f(sc[j][h * 2 + 1] - base);
        rs[h] += sc[j][h * 2] + sc[j][h * 2 + 1];
      }
    }
    l_r[0] += rs[0];
    l_r[1] += rs[1];
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
        ldsm_x4_t(b, tile_ptr<D>(const_cast<__nv_bfloat16*>(cV), kk * 16 + (lane & 15), jd * 16 + (lane >> 4) * 8));
        mma16816(o[2 * jd], pa, b[0], b[1]);
        mma16816(o[2 * jd + 1], pa, b[2], b[3]);
      }
    }
    __syncthreads();
  }
  // finalize: full row sums across the 4 lanes of a quad
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int pr = qt * kQT + wr + (lane >> 2) + h * 8;
    if (pr >= R || pos_r[h] < key_begin) continue;
    const int tok = pr / G, head = kvh * G + pr % G;
    const int64_t grow = row0 + tok;
    if (a.n_parts == 1) {
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
        *reinterpret_cast<float2*>(dst + j * 8 + 2 * (lane & 3)) = make_float2(o[j][h * 2], o[j][h * 2 + 1]);
      if ((lane & 3) == 0) {
        a.ws_ml[slot * 2] = m_r[h];
        a.ws_ml[slot * 2 + 1] = l_r[h];
      }
    }
  }
}

// Merge partitions in fixed order: one warp per (row, head).
__global__ void attn_combine_kernel(const AttnArgs a, int n_seqs) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= a.M * a.H) return;
  const int row = w / a.H, head = w % a.H;
  const int s = seq_of_row(a.cu_q, n_seqs, row);
  const int pos = a.start_pos[s] + (row - a.cu_q[s]);
  const int np = min(a.n_parts, pos / a.part_size + 1);
  float m = -INFINITY;
  for (int p = 0; p < np; ++p) m = fmaxf(m, a.ws_ml[(((int64_t)p * a.M + row) * a.H + head) * 2]);
  float l = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int p = 0; p < np; ++p) {
    const int64_t slot = ((int64_t)p * a.M + row) * a.H + head;
    const float wgt = exp2f(a.ws_ml[slot * 2] - m);
    l += wgt * a.ws_ml[slot * 2 + 1];
    for (int i = 0; i < a.D / 32; ++i) acc[i] += wgt * a.ws_o[slot * a.D + lane + 32 * i];
  }
  const float inv = 1.f / l;
  for (int i = 0; i < a.D / 32; ++i)
    a.out[(int64_t)row * a.ld_out + head * a.D + lane + 32 * i] = __float2bfloat16_rn(acc[i] * inv);
}

// Partition plan shared by the workspace query and the launch.
void plan(int M, int n_seqs, int max_q, int max_ctx, int H, int Hkv, int& part_size, int& n_parts) {
  const int G = H / Hkv;
  const int qtiles = (max_q * G + kQT - 1) / kQT;
  const int64_t items = (int64_t)qtiles * n_seqs * Hkv;
  const int max_parts = (max_ctx + 255) / 256;  // at least 256 keys per partition
  int np = 1;
  if (items < kTargetCtas) np = (int)((kTargetCtas + items - 1) / items);
  np = std::max(1, std::min(np, max_parts));
  int ps = (max_ctx + np - 1) / np;
  ps = (ps + kKT - 1) / kKT * kKT;
  n_parts = (max_ctx + ps - 1) / ps;
  part_size = ps;
  (void)M;
}

template <int D>
int launch_attn(const AttnArgs& a, int n_seqs, int max_q, cudaStream_t st) {
  const int G = a.H / a.Hkv;
  const int smem = (kQT + 4 * kKT) * D * 2;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bf16_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return ALORA_ECUDA;
    configured = true;
  }
  dim3 grid((max_q * G + kQT - 1) / kQT, a.n_parts, n_seqs * a.Hkv);
  attn_bf16_kernel<D><<<grid, kThreadsA, smem, st>>>(a);
  ALORA_LAUNCH_CHECK();
  if (a.n_parts > 1) {
    const int warps = a.M * a.H;
    attn_combine_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(a, n_seqs);
    ALORA_LAUNCH_CHECK();
  }
  return ALORA_OK;
}

}  // namespace

// Upper bound over all steps: a split happens only when items < kTargetCtas, and then
// n_parts * M * H <= 2 * kTargetCtas * kQT (see plan()).
int64_t attn_bf16_workspace_bound(int H, int D) {
  (void)H;
  return (int64_t)2 * kTargetCtas * kQT * (D + 2) * 4;
}

int64_t attn_bf16_workspace(int M, int n_seqs, int max_q, int max_ctx, int H, int Hkv, int D) {
  int ps, np;
  plan(M, n_seqs, max_q, max_ctx, H, Hkv, ps, np);
  if (np <= 1) return 0;
  return (int64_t)np * M * H * (D + 2) * 4;
}

int attn_bf16(const __nv_bfloat16* q, int64_t ld_q, int M, int n_seqs, const int32_t* cu_q, const int32_t* start_pos,
              const int32_t* block_table, int max_blocks, int max_q, int max_ctx, const __nv_bfloat16* kv,
              int n_layers, int layer, int B, int H, int Hkv, int D, __nv_bfloat16* out, int64_t ld_out, void* ws,
              int64_t ws_bytes, cudaStream_t st) {
  if (M == 0 || n_seqs == 0) return ALORA_OK;
  if (H % Hkv || (D != 64 && D != 128) || ld_q % 8 || max_q < 1 || max_ctx < 1) return ALORA_EINVAL;
  AttnArgs a{};
  a.q = q; a.ld_q = ld_q; a.cu_q = cu_q; a.start_pos = start_pos; a.block_table = block_table;
  a.max_blocks = max_blocks; a.kv = kv; a.n_layers = n_layers; a.layer = layer; a.B = B; a.H = H; a.Hkv = Hkv;
  a.D = D; a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  a.out = out; a.ld_out = ld_out; a.M = M;
  plan(M, n_seqs, max_q, max_ctx, H, Hkv, a.part_size, a.n_parts);
  if (a.n_parts > 1) {
    const int64_t need = (int64_t)a.n_parts * M * H * (D + 2) * 4;
    if (ws == nullptr || ws_bytes < need) return ALORA_EINVAL;
    a.ws_o = static_cast<float*>(ws);
    a.ws_ml = a.ws_o + (int64_t)a.n_parts * M * H * D;
  }
  return D == 64 ? launch_attn<64>(a, n_seqs, max_q, st) : launch_attn<128>(a, n_seqs, max_q, st);
}

}  // namespace alora
