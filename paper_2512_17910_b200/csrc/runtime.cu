// C ABI entry points and the native step executor.
//
// alora_model_forward replaces Model.forward_step / _forward_one
// (model.py:233-272): instead of a Python loop per span and per layer, all
// spans of an engine step are packed into one varlen batch and every layer's
// kernels are launched from here, on the caller's stream, with no host sync.

#include <algorithm>
#include <cxxabi.h>
#include <string>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace alora;

namespace alora {
void configure_kernels() {
  static std::once_flag once;
  std::call_once(once, [] {
    configure_bf16_ops();
    configure_kv_ops();
    configure_attention();
    configure_gemm();
    configure_tp();
  });
}
}  // namespace alora

namespace {

// Event-bracketed launch records (alora_model_set_profiling).
struct ProfRec {
  const char* kind;
  int ev0, ev1;
  double bytes, flops;
  std::vector<LaunchNote> kernels;  // what the launcher actually launched (function, grid size)
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> events;
  int used = 0;
  std::vector<ProfRec> recs;
  int event(cudaStream_t st) {
    if (used == (int)events.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      events.push_back(e);
    }
    cudaEventRecord(events[used], st);
    return used++;
  }
  ~Profiler() {
    for (auto e : events) cudaEventDestroy(e);
  }
};

// A captured forward: valid for steps with the same shape and the same staged device buffers.
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  AloraStepDesc step{};
  int32_t launches = 0;
  uint64_t last_use = 0;
  bool uploaded = false;
};
// n_tokens, n_seqs, max_blocks, max_q, max_ctx, attention items, attention partitions (the grids a capture bakes in)
using GraphKey = std::tuple<int, int, int, int, int, int, int>;

struct Model {
  AloraModelDesc d;
  std::vector<const void*> w_qkv_t, w_o_t, w_in_t, w_out_t, lora_down, lora_up_t;
  // O / MLP adapter targets (empty = untargeted)
  std::vector<const void*> lora_o_down, lora_o_up_t, lora_in_down, lora_in_up_t, lora_out_down, lora_out_up_t;
  std::vector<const float*> attn_norm, mlp_norm;
  std::vector<void*> tp_peers;  // fused TP all-reduce: every rank's symmetric buffer (empty = hook path)
  int32_t last_launches = 0;
  Profiler prof;
  std::map<GraphKey, GraphEntry> graphs;
  uint64_t graph_clock = 0;
  ~Model() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  }
};

// Runs one launcher; counts it and, when profiling, brackets it with events and tags its algorithmic cost.
struct Launcher {
  Model& m;
  cudaStream_t st;
  int n = 0;
  // Debug only (timing attribution): ALORA_SKIP="attention,gemm_o" drops those launches (results are wrong).
  static bool skipped(const char* kind) {
    static const char* env = getenv("ALORA_SKIP");
    if (!env) return false;
    const size_t n = strlen(kind);
    for (const char* p = strstr(env, kind); p; p = strstr(p + 1, kind))
      if ((p == env || p[-1] == ',') && (p[n] == ',' || p[n] == 0)) return true;
    return false;
  }
  template <typename F>
  int operator()(const char* kind, double bytes, double flops, F&& fn) {
    if (skipped(kind)) return ALORA_OK;
    int e0 = m.prof.on ? m.prof.event(st) : -1;
    std::vector<LaunchNote> log;
    if (m.prof.on) g_launch_log = &log;
    const int rc = fn();
    g_launch_log = nullptr;
    if (rc != ALORA_OK) return rc;
    ++n;
    if (m.prof.on) {
      const int e1 = m.prof.event(st);
      if (e0 >= 0 && e1 >= 0) m.prof.recs.push_back({kind, e0, e1, bytes, flops, std::move(log)});
    }
    return ALORA_OK;
  }
};

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Workspace carve-up shared by alora_model_workspace_bytes and the executor.
struct Ws {
  int64_t x, h, qkv, attn, gu, act, s, masks, hf, attn_ws, gemm_ws, part, amax, tpd, total;
  int64_t part_bytes;
  int64_t attn_ws_bytes, gemm_ws_bytes;
};

Ws plan_ws(const AloraModelDesc& d) {
  const int64_t T = d.max_tokens, S = d.max_seqs;
  const int64_t e = d.dtype == ALORA_BF16 ? 2 : 4;
  const int64_t nq = (int64_t)d.n_heads * d.head_dim, nkv = (int64_t)d.n_kv_heads * d.head_dim;
  const int64_t F = d.ffn_dim;
  const int64_t ks = (int64_t)d.n_slots * d.lora_rank;
  Ws w{};
  int64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = off; off = align_up(off + bytes, 256); return o; };
  w.x = take(T * d.d_model * 4);
  w.h = take(T * d.d_model * e);
  w.qkv = take(T * (nq + 2 * nkv) * e);
  w.attn = take(T * nq * e);
  w.gu = take(d.arch == ALORA_ARCH_LLAMA && d.dtype == ALORA_F32 ? T * 2 * F * 4 : 0);
  w.act = take(T * F * e);
  w.s = take(d.dtype == ALORA_BF16 ? 3 * T * ks * 2 : 3 * T * d.lora_rank * 4);
  w.masks = take((T / 128 + 2) * 4);
  w.hf = take(S * d.d_model * e);
  w.attn_ws_bytes = d.dtype == ALORA_BF16
                        ? attn_bf16_workspace_bound(d.n_heads, d.head_dim)
                        : 0;
  w.attn_ws = take(w.attn_ws_bytes);
  w.gemm_ws_bytes = d.dtype == ALORA_BF16 ? gemm_bf16_workspace_bytes() : 0;
  w.gemm_ws = take(w.gemm_ws_bytes);  // split-K counters must start zeroed: the caller zero-fills the workspace
  // deferred split-K partials of the weight-streaming GEMMs (M <= 256): [<= 8 splits][M][max(Nqkv, d)] fp32
  w.part_bytes = d.dtype == ALORA_BF16 ? 8LL * std::min<int64_t>(T, 256) * std::max<int64_t>(nq + 2 * nkv, d.d_model) * 4 : 0;
  w.part = take(w.part_bytes);
  w.amax = take(S * 8);  // packed greedy argmax per span (fused into the lm_head epilogue)
  // TP through the hook: this rank's residual delta, all-reduced in place (the fused path uses the peer buffers)
  w.tpd = take(d.tp_size > 1 && d.tp_peers == nullptr ? T * d.d_model * 4 : 0);
  w.total = off;
  return w;
}

int validate(const AloraModelDesc* d) {
  if (!d) return ALORA_EINVAL;
  if (d->arch != ALORA_ARCH_REF && d->arch != ALORA_ARCH_LLAMA) return ALORA_EINVAL;
  if (d->dtype != ALORA_F32 && d->dtype != ALORA_BF16) return ALORA_EINVAL;
  if (d->n_layers < 1 || d->d_model < 1 || d->n_heads < 1 || d->n_kv_heads < 1 || d->head_dim < 2 ||
      d->ffn_dim < 1 || d->vocab < 1 || d->max_tokens < 1 || d->max_seqs < 1)
    return ALORA_EINVAL;
  if (d->n_heads % d->n_kv_heads != 0 || d->head_dim % 2 != 0) return ALORA_EINVAL;
  if (d->arch == ALORA_ARCH_REF && (d->n_kv_heads != d->n_heads || d->n_heads * d->head_dim != d->d_model))
    return ALORA_EINVAL;
  if (d->n_slots < 0 || d->lora_rank < 0 || (d->n_slots > 0 && d->lora_rank < 1)) return ALORA_EINVAL;
  if (d->dtype == ALORA_BF16 && d->n_slots > 32) return ALORA_EINVAL;  // tile slot masks are 32-bit
  if (d->tp_size > 1 && (d->dtype != ALORA_BF16 || (d->tp_allreduce == nullptr && d->tp_peers == nullptr)))
    return ALORA_EINVAL;
  if (d->tp_size > 1 && d->tp_peers != nullptr && (d->tp_size > 8 || d->tp_rank < 0 || d->tp_rank >= d->tp_size))
    return ALORA_EINVAL;
  return ALORA_OK;
}

// LoRA shrink for every row against all adapters' stacked down rows [3*SR, K] on the tensor cores, with the
// per-row slot/target select in the epilogue; the SIMT segmented kernel covers SR that is not a multiple of 64.
// With a deferral buffer, a weight-streaming shrink may split K; its select epilogue then runs in
// lora_select_finalize_bf16 (one extra small launch, counted in *extra_launches).
int shrink(const __nv_bfloat16* h, int M, int K, const int32_t* row_slot, const uint8_t* row_apply,
           const __nv_bfloat16* down, int n_slots, int R, const uint8_t* targets, __nv_bfloat16* s, cudaStream_t st,
           const GemmWs* gw, float* part = nullptr, int64_t part_bytes = 0, int* extra_launches = nullptr,
           int n_planes = 3, int tbit0 = 0) {
  const int SR = n_slots * R;
  if (SR % 64 != 0)
    return lora_shrink_bf16(h, M, K, row_slot, row_apply, down, n_slots, R, targets, s, st, n_planes, tbit0);
  GemmLora g;
  g.sel_row_slot = row_slot;
  g.sel_row_apply = row_apply;
  g.sel_targets = targets;
  g.sel_sr = SR;
  g.sel_rank = R;
  g.sel_planes = n_planes;
  g.sel_tbit0 = tbit0;
  GemmDefer df;
  df.partial = part;
  df.capacity = part_bytes;
  const int rc =
      gemm_bf16(kEpiLoraSelect, h, K, down, K, s, SR, M, n_planes * SR, K, &g, st, gw, 8, part ? &df : nullptr);
  if (rc != ALORA_OK || !df.deferred) return rc;
  if (extra_launches) ++*extra_launches;
  return lora_select_finalize_bf16(part, df.splits_out, M, SR, R, row_slot, row_apply, targets, s, st, n_planes,
                                   tbit0);
}

int forward_f32(Model& mdl, const AloraStepDesc& s, cudaStream_t st) {
  const AloraModelDesc& d = mdl.d;
  const Ws w = plan_ws(d);
  char* base = static_cast<char*>(d.workspace);
  float* x = reinterpret_cast<float*>(base + w.x);
  float* h = reinterpret_cast<float*>(base + w.h);
  float* qkv = reinterpret_cast<float*>(base + w.qkv);
  float* attn = reinterpret_cast<float*>(base + w.attn);
  float* gu = reinterpret_cast<float*>(base + w.gu);
  float* act = reinterpret_cast<float*>(base + w.act);
  float* sws = reinterpret_cast<float*>(base + w.s);
  float* hf = reinterpret_cast<float*>(base + w.hf);
  const int M = s.n_tokens, S = s.n_seqs, dm = d.d_model, F = d.ffn_dim;
  const int H = d.n_heads, Hkv = d.n_kv_heads, D = d.head_dim;
  const int Nq = H * D, Nkv = Hkv * D, Nqkv = Nq + 2 * Nkv;
  const bool llama = d.arch == ALORA_ARCH_LLAMA;
  int n = 0;
  int rc;
#define RUN(call)                      \
  do {                                 \
    rc = (call);                       \
    if (rc != ALORA_OK) return rc;     \
    ++n;                               \
  } while (0)
  RUN(embed_f32(s.tokens, s.positions, static_cast<const float*>(d.embed), llama ? nullptr : d.pos_table, M, dm, x,
                st, s.next_ids));
  for (int l = 0; l < d.n_layers; ++l) {
    RUN(rmsnorm_f64(x, nullptr, M, dm, mdl.attn_norm[l], d.rms_eps, h, st));
    RUN(gemm_f64(kEpiStore, h, dm, static_cast<const float*>(mdl.w_qkv_t[l]), dm, qkv, Nqkv, M, Nqkv, dm, st));
    if (d.n_slots > 0) {
      RUN(lora_f64(h, M, dm, s.row_slot, s.row_apply, static_cast<const float*>(mdl.lora_down[l]),
                   static_cast<const float*>(mdl.lora_up_t[l]), d.n_slots, d.lora_rank, d.slot_targets, sws, Nq, Nkv,
                   qkv, Nqkv, st));
      ++n;  // shrink + expand
    }
    if (llama) RUN(rope_f64(qkv, Nqkv, s.positions, M, H, Hkv, D, d.rope_cos, d.rope_sin, st));
    RUN(kv_write(ALORA_F32, qkv + Nq, qkv + Nq + Nkv, Nqkv, s.slot_mapping, M, Nkv, d.kv_pool, d.n_layers, l,
                 d.block_size, st));
    RUN(attn_f64(qkv, Nqkv, M, S, s.cu_q, s.start_pos, s.block_table, s.max_blocks,
                 static_cast<const float*>(d.kv_pool), d.n_layers, l, d.block_size, H, Hkv, D, 0.f, attn, Nq, st));
    RUN(gemm_f64(kEpiAdd, attn, Nq, static_cast<const float*>(mdl.w_o_t[l]), Nq, x, dm, M, dm, Nq, st));
    RUN(rmsnorm_f64(x, nullptr, M, dm, mdl.mlp_norm[l], d.rms_eps, h, st));
    if (llama) {
      RUN(gemm_f64(kEpiStore, h, dm, static_cast<const float*>(mdl.w_in_t[l]), dm, gu, 2 * F, M, 2 * F, dm, st));
      RUN(silu_mul_f64(gu, M, F, act, st));
    } else {
      RUN(gemm_f64(kEpiRelu, h, dm, static_cast<const float*>(mdl.w_in_t[l]), dm, act, F, M, F, dm, st));
    }
    RUN(gemm_f64(kEpiAdd, act, F, static_cast<const float*>(mdl.w_out_t[l]), F, x, dm, M, dm, F, st));
  }
  RUN(rmsnorm_f64(x, s.last_row, S, dm, d.final_norm, d.rms_eps, hf, st));
  RUN(gemm_f64(kEpiStore, hf, dm, static_cast<const float*>(d.unembed_t), dm, s.logits, d.vocab, S, d.vocab, dm,
               st));
  RUN(argmax_rows(s.logits, S, d.vocab, s.next_ids, st));
#undef RUN
  mdl.last_launches = n;
  return ALORA_OK;
}

int forward_bf16(Model& mdl, const AloraStepDesc& s, cudaStream_t st) {
  const AloraModelDesc& d = mdl.d;
  const Ws w = plan_ws(d);
  char* base = static_cast<char*>(d.workspace);
  float* x = reinterpret_cast<float*>(base + w.x);
  auto* h = reinterpret_cast<__nv_bfloat16*>(base + w.h);
  auto* qkv = reinterpret_cast<__nv_bfloat16*>(base + w.qkv);
  auto* attn = reinterpret_cast<__nv_bfloat16*>(base + w.attn);
  auto* act = reinterpret_cast<__nv_bfloat16*>(base + w.act);
  auto* sws = reinterpret_cast<__nv_bfloat16*>(base + w.s);
  auto* masks = reinterpret_cast<uint32_t*>(base + w.masks);
  auto* hf = reinterpret_cast<__nv_bfloat16*>(base + w.hf);
  void* aws = base + w.attn_ws;
  const GemmWs gws = gemm_ws_from(base + w.gemm_ws, w.gemm_ws_bytes);
  const GemmWs* gw = &gws;  // split-K scratch of the per-tile GEMM (M > 256)
  float* part = reinterpret_cast<float*>(base + w.part);  // deferred split-K partials (M <= 256)
  int pend = 0;  // splits of the residual update still pending in `pend_buf` (applied by the next RMSNorm)
  const float* pend_buf = part;

  const int M = s.n_tokens, S = s.n_seqs, dm = d.d_model, F = d.ffn_dim;
  const int H = d.n_heads, Hkv = d.n_kv_heads, D = d.head_dim;
  const int Nq = H * D, Nkv = Hkv * D, Nqkv = Nq + 2 * Nkv;
  const bool llama = d.arch == ALORA_ARCH_LLAMA;
  const bool lora = d.n_slots > 0;
  const int rk = d.lora_rank;
  // batch-invariant mode pins every per-row choice to the model, never to the step: the segmented shrink for
  // any row count (else the per-row SIMT shrink), one GEMM kernel and K range, one attention partition
  struct InvariantScope {
    bool prev;
    explicit InvariantScope(bool on) : prev(g_batch_invariant) { g_batch_invariant = on; }
    ~InvariantScope() { g_batch_invariant = prev; }
  } inv_scope(d.batch_invariant != 0);
  const bool inv = d.batch_invariant != 0;
  const bool seg_ok = lora && d.d_model % 128 == 0 && (rk == 8 || rk == 16 || rk == 32 || rk == 64);
  const bool seg_shrink = seg_ok && (s.lora_rows_max <= kSegMaxRows || inv);
  // row chunks of the segmented shrink: a function of the step's graph key (n_tokens and this switch), never of
  // the exact per-slot counts, so a captured decode / prefill graph stays correct on replay
  const int seg_rows = s.lora_rows_max <= kSegMaxRows ? kSegMaxRows : M;
  const bool lora_o = lora && !mdl.lora_o_down.empty(), lora_in = lora && !mdl.lora_in_down.empty();
  const bool lora_out = lora && !mdl.lora_out_down.empty();
  const int in_planes = llama ? 2 : 1;
  Launcher run{mdl, st};
  const bool tp = d.tp_size > 1;
  const bool tp_fused = tp && !mdl.tp_peers.empty();
  float* tpd = reinterpret_cast<float*>(base + w.tpd);
  int ar_i = 0;          // fused all-reduces issued so far in this forward (partial slot = parity)
  bool h_ready = false;  // the fused all-reduce already produced the next RMSNorm's output in h
  // Residual-producing GEMM (O-projection, MLP-down). Unsharded: x += A.W^T fused in the epilogue, or the
  // split-K partials are left for the next RMSNorm. Tensor parallel: this rank's partial product is
  // materialised in tpd (split-K summed in order), all-reduced by the caller's hook, then applied by the
  // RMSNorm as a single pending partial (row-parallel linear layer + all-reduce).
  auto residual_gemm = [&](const __nv_bfloat16* A, int K, const void* W, int ldw,
                           const GemmLora* gla = nullptr) -> int {
    GemmDefer df;
    df.partial = part;
    df.capacity = w.part_bytes;
    if (!tp) {
      const int rc = gemm_bf16(kEpiAdd, A, K, static_cast<const __nv_bfloat16*>(W), ldw, x, dm, M, dm, K, gla,
                               st, gw, 8, &df);
      pend = df.deferred ? df.splits_out : 0;
      pend_buf = part;
      return rc;
    }
    if (tp_fused) {  // this rank's partial -> its symmetric buffer slot, reduced by tp_allreduce_norm
      float* slot = tp_partial_slot(mdl.tp_peers[d.tp_rank], d.max_tokens, dm, ar_i);
      pend = 0;
      return gemm_bf16(kEpiStore | 16, A, K, static_cast<const __nv_bfloat16*>(W), ldw, slot, dm, M, dm, K, gla,
                       st, gw, 8, nullptr);
    }
    int rc = gemm_bf16(kEpiStore | 16, A, K, static_cast<const __nv_bfloat16*>(W), ldw, tpd, dm, M, dm, K, gla,
                       st, gw, 8, nullptr);
    pend = 1;
    pend_buf = tpd;
    return rc;
  };
  int rc;
  const double m_ = M, dm_ = dm, F_ = F, Nqkv_ = Nqkv, Nq_ = Nq, V_ = d.vocab, S_ = S, ks_ = (double)d.n_slots * d.lora_rank;
  // algorithmic bytes of a bf16 GEMM: A + B read once, C written (and read for +=)
  auto gemm_bytes = [](double m, double n, double k, double out_b, bool rmw) {
    return 2.0 * (m * k + n * k) + m * n * out_b * (rmw ? 2.0 : 1.0);
  };
#define RUN(kind, bytes, flops, call)                                           \
  do {                                                                          \
    rc = run(kind, bytes, flops, [&]() { return (call); });                     \
    if (rc != ALORA_OK) return rc;                                              \
  } while (0)
  RUN("embed", m_ * dm_ * 6, 0, embed_bf16(s.tokens, s.positions, static_cast<const __nv_bfloat16*>(d.embed),
                                           llama ? nullptr : d.pos_table, M, dm, x, st, s.next_ids));
  if (lora) RUN("lora_masks", m_ * 5, 0, lora_tile_masks(s.row_slot, s.row_apply, M, masks, st));
  // fused TP: sum of every rank's partial (rank order) + residual + the next RMSNorm (norm_w) in one kernel
  auto tp_reduce = [&](const float* norm_w, bool norm) -> int {
    const int rc = tp_allreduce_norm(mdl.tp_peers.data(), d.tp_size, d.tp_rank, d.tp_colocated, d.max_tokens, ar_i,
                                     M, dm, x, norm_w, d.rms_eps, norm ? h : nullptr, st);
    ++ar_i;
    h_ready = norm;
    return rc;
  };
  const double tp_bytes = m_ * dm_ * 4.0 * (d.tp_size + 2) + m_ * dm_ * 2;
  for (int l = 0; l < d.n_layers; ++l) {
    if (!h_ready)
      RUN("rmsnorm", m_ * dm_ * (pend ? 10.0 + 4.0 * pend : 6.0), 0,
          residual_rmsnorm_bf16(x, pend_buf, pend, M, nullptr, M, dm, mdl.attn_norm[l], d.rms_eps, h, st));
    h_ready = false;
    pend = 0;
    GemmLora gl;
    if (lora && seg_shrink) {
      // few delta rows per adapter: stream each adapter's down rows once against its rows (+ the zero fill)
      const double act = s.lora_rows_max;
      RUN("lora_shrink", 3.0 * d.n_slots * d.lora_rank * dm_ * 2 + d.n_slots * act * dm_ * 2 + 3.0 * m_ * ks_ * 2,
          2.0 * 3 * d.n_slots * act * d.lora_rank * dm_,
          lora_shrink_seg_bf16(h, M, dm, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(mdl.lora_down[l]),
                               d.n_slots, d.lora_rank, d.slot_targets, sws, st, 3, 0, seg_rows));
    } else if (lora && inv) {
      RUN("lora_shrink", m_ * dm_ * 2 + 3.0 * ks_ * dm_ * 2 + 3.0 * m_ * ks_ * 2, 2.0 * 3 * m_ * ks_ * dm_,
          lora_shrink_bf16(h, M, dm, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(mdl.lora_down[l]),
                           d.n_slots, d.lora_rank, d.slot_targets, sws, st));
    } else if (lora) {
      RUN("lora_shrink", m_ * dm_ * 2 + 3.0 * ks_ * dm_ * 2 + 3.0 * m_ * ks_ * 2, 2.0 * 3 * m_ * ks_ * dm_,
          shrink(h, M, dm, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(mdl.lora_down[l]), d.n_slots,
                 d.lora_rank, d.slot_targets, sws, st, gw, part, w.part_bytes, &run.n));
    }
    if (lora) {
      gl.s = sws;
      gl.up_t = static_cast<const __nv_bfloat16*>(mdl.lora_up_t[l]);
      gl.ks = d.n_slots * d.lora_rank;
      gl.n_q = Nq;
      gl.n_kv = Nkv;
      gl.tile_slot_mask = masks;
      gl.rank = d.lora_rank;
    }
    if (llama) {  // RoPE fused into the QKV epilogue: fp32 rotate of the accumulator, one bf16 rounding
      gl.positions = s.positions;
      gl.rope_cos = d.rope_cos;
      gl.rope_sin = d.rope_sin;
      gl.rope_cols = Nq + Nkv;
      gl.head_dim = D;
      // large-M steps: the epilogue also scatters K / V into the paged pool (no separate kv_write pass)
      gl.kv_pool = static_cast<__nv_bfloat16*>(d.kv_pool);
      gl.kv_slots = s.slot_mapping;
      gl.kv_q = Nq;
      gl.kv_w = Nkv;
      gl.kv_layer = l;
      gl.kv_layers = d.n_layers;
      gl.kv_block = d.block_size;
    }
    GemmDefer dq;
    dq.partial = part;
    dq.capacity = w.part_bytes;
    RUN("gemm_qkv", gemm_bytes(m_, Nqkv_, dm_, 2, false) + (lora ? 2.0 * Nqkv_ * ks_ : 0.0), 2.0 * m_ * Nqkv_ * dm_,
        gemm_bf16(llama ? kEpiRope : kEpiStore, h, dm, static_cast<const __nv_bfloat16*>(mdl.w_qkv_t[l]), dm, qkv,
                  Nqkv, M, Nqkv, dm, (lora || llama) ? &gl : nullptr, st, gw, 8, llama ? &dq : nullptr));
    if (dq.deferred) {  // split-K / decode QKV: RoPE + bf16 + the paged KV scatter run in the finalize kernel
      RUN("qkv_finalize", m_ * Nqkv_ * 4.0 * dq.splits_out + 2.0 * m_ * Nqkv_ + 2.0 * 2 * m_ * Nkv * 2, 0,
          qkv_finalize_bf16(part, dq.splits_out, M, Nq, Nkv, D, s.positions, d.rope_cos, d.rope_sin, qkv, Nqkv,
                            s.slot_mapping, static_cast<__nv_bfloat16*>(d.kv_pool), d.n_layers, l, d.block_size, st));
    } else if (!dq.kv_written) {
      RUN("kv_write", 2.0 * 2 * m_ * Nkv * 2, 0,
          kv_write(ALORA_BF16, qkv + Nq, qkv + Nq + Nkv, Nqkv, s.slot_mapping, M, Nkv, d.kv_pool, d.n_layers, l,
                   d.block_size, st));
    }
    if (s.attn_plan != nullptr && !inv) {  // shared-prefix plan: each group's prefix KV streamed once for all its rows
      RUN("attention", s.attn_kv_tokens * 2.0 * Nkv * 2 + 2.0 * m_ * Nq_ * 2, 4.0 * H * D * s.attn_qk_pairs,
          attn_grouped(qkv, Nqkv, M, S, s.positions, s.row_seq, s.block_table, s.max_blocks, s.attn_plan,
                       s.attn_items, s.attn_segs, s.attn_sets, s.attn_max_parts, true,
                       static_cast<const __nv_bfloat16*>(d.kv_pool), d.total_blocks, d.n_layers, l, d.block_size, H,
                       Hkv, D, attn, Nq, aws, w.attn_ws_bytes, st));
    } else {
      RUN("attention", s.attn_kv_tokens * 2.0 * Nkv * 2 + 2.0 * m_ * Nq_ * 2, 4.0 * H * D * s.attn_qk_pairs,
          attn_bf16(qkv, Nqkv, M, S, s.cu_q, s.start_pos, s.block_table, s.max_blocks, s.max_q, s.max_ctx,
                    static_cast<const __nv_bfloat16*>(d.kv_pool), d.n_layers, l, d.block_size, H, Hkv, D, attn, Nq,
                    aws, w.attn_ws_bytes, st, d.total_blocks));
    }
    // O / MLP adapter targets (extension): the masked shrink of the projection's input into the shrink
    // workspace (its q|k|v planes were consumed by gemm_qkv), then the expand as extra K of the GEMM
    auto target_shrink = [&](const __nv_bfloat16* in, int K, const void* down, int planes, int tbit0) -> int {
      if (seg_shrink && lora_shrink_seg_fits(K))
        return lora_shrink_seg_bf16(in, M, K, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(down),
                                    d.n_slots, rk, d.slot_targets, sws, st, planes, tbit0, seg_rows);
      if (inv)
        return lora_shrink_bf16(in, M, K, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(down),
                                d.n_slots, rk, d.slot_targets, sws, st, planes, tbit0);
      return shrink(in, M, K, s.row_slot, s.row_apply, static_cast<const __nv_bfloat16*>(down), d.n_slots, rk,
                    d.slot_targets, sws, st, gw, part, w.part_bytes, &run.n, planes, tbit0);
    };
    auto target_lora = [&](const void* up_t, int N, int planes) {
      GemmLora g;
      g.s = sws;
      g.up_t = static_cast<const __nv_bfloat16*>(up_t);
      g.ks = d.n_slots * rk;
      g.rank = rk;
      g.tile_slot_mask = masks;
      g.planes = planes > 1 ? planes : 0;
      g.s_planes = planes;
      g.n_q = N;  // select mode: every column reads plane 0
      g.n_kv = 0;
      return g;
    };
    const double shrink_bytes_o = m_ * Nq_ * 2 + (double)ks_ * Nq_ * 2 + m_ * ks_ * 2;
    if (lora_o)
      RUN("lora_shrink", shrink_bytes_o, 2.0 * m_ * ks_ * Nq_,
          target_shrink(attn, Nq, mdl.lora_o_down[l], 1, 3));
    const GemmLora glo = lora_o ? target_lora(mdl.lora_o_up_t[l], dm, 1) : GemmLora{};
    RUN("gemm_o", gemm_bytes(m_, dm_, Nq_, 4, true) + (lora_o ? 2.0 * dm_ * ks_ : 0.0), 2.0 * m_ * dm_ * Nq_,
        residual_gemm(attn, Nq, mdl.w_o_t[l], Nq, lora_o ? &glo : nullptr));
    if (tp_fused) RUN("tp_allreduce", tp_bytes, 0, tp_reduce(mdl.mlp_norm[l], true));
    else if (tp) RUN("tp_allreduce", m_ * dm_ * 4.0, 0, d.tp_allreduce(d.tp_ctx, tpd, (int64_t)M * dm, st));
    if (!h_ready)
      RUN("rmsnorm", m_ * dm_ * (pend ? 10.0 + 4.0 * pend : 6.0), 0,
          residual_rmsnorm_bf16(x, pend_buf, pend, M, nullptr, M, dm, mdl.mlp_norm[l], d.rms_eps, h, st));
    h_ready = false;
    pend = 0;
    const double n_in = llama ? 2 * F_ : F_;
    if (lora_in)
      RUN("lora_shrink", m_ * dm_ * 2 + in_planes * ks_ * dm_ * 2 + in_planes * m_ * ks_ * 2,
          2.0 * in_planes * m_ * ks_ * dm_, target_shrink(h, dm, mdl.lora_in_down[l], in_planes, 4 + (llama ? 0 : 1)));
    const GemmLora gli = lora_in ? target_lora(mdl.lora_in_up_t[l], llama ? 2 * F : F, in_planes) : GemmLora{};
    RUN("gemm_mlp_in", 2.0 * (m_ * dm_ + n_in * dm_) + m_ * F_ * 2 + (lora_in ? 2.0 * n_in * in_planes * ks_ : 0.0),
        2.0 * m_ * n_in * dm_,
        gemm_bf16(llama ? kEpiSwiglu : kEpiRelu, h, dm, static_cast<const __nv_bfloat16*>(mdl.w_in_t[l]), dm, act, F,
                  M, llama ? 2 * F : F, dm, lora_in ? &gli : nullptr, st, gw));
    if (lora_out)
      RUN("lora_shrink", m_ * F_ * 2 + ks_ * F_ * 2 + m_ * ks_ * 2, 2.0 * m_ * ks_ * F_,
          target_shrink(act, F, mdl.lora_out_down[l], 1, 6));
    const GemmLora glw = lora_out ? target_lora(mdl.lora_out_up_t[l], dm, 1) : GemmLora{};
    RUN("gemm_mlp_out", gemm_bytes(m_, dm_, F_, 4, true) + (lora_out ? 2.0 * dm_ * ks_ : 0.0), 2.0 * m_ * dm_ * F_,
        residual_gemm(act, F, mdl.w_out_t[l], F, lora_out ? &glw : nullptr));
    if (tp_fused) {
      const bool last = l + 1 == d.n_layers;  // the final norm runs on the last rows only (below)
      RUN("tp_allreduce", tp_bytes, 0, tp_reduce(last ? nullptr : mdl.attn_norm[l + 1], !last));
    } else if (tp) {
      RUN("tp_allreduce", m_ * dm_ * 4.0, 0, d.tp_allreduce(d.tp_ctx, tpd, (int64_t)M * dm, st));
    }
  }
  // greedy argmax fused into the lm_head epilogue (weight-streaming path: S <= 256 spans, vocab % 32 == 0)
  auto* amax = reinterpret_cast<unsigned long long*>(base + w.amax);
  const bool fused_argmax = S <= 256 && d.vocab % 32 == 0;
  RUN("rmsnorm", S_ * dm_ * (pend ? 10.0 + 4.0 * pend : 6.0), 0,
      residual_rmsnorm_bf16(x, pend_buf, pend, M, s.last_row, S, dm, d.final_norm, d.rms_eps, hf, st,
                            fused_argmax ? amax : nullptr));
  GemmLora glm;
  glm.argmax = fused_argmax ? amax : nullptr;
  RUN("gemm_lm_head", gemm_bytes(S_, V_, dm_, 4, false), 2.0 * S_ * V_ * dm_,
      gemm_bf16(kEpiStore + 16 /* fp32 out */, hf, dm, static_cast<const __nv_bfloat16*>(d.unembed_t), dm, s.logits,
                d.vocab, S, d.vocab, dm, fused_argmax ? &glm : nullptr, st, gw));
  if (fused_argmax)
    RUN("argmax", S_ * 12.0, 0, argmax_unpack(amax, S, s.next_ids, st));
  else
    RUN("argmax", S_ * V_ * 4, 0, argmax_rows(s.logits, S, d.vocab, s.next_ids, st));
#undef RUN
  mdl.last_launches = run.n;
  return ALORA_OK;
}

}  // namespace

extern "C" {

const char* alora_version(void) {
  return "libalora_sm100a 0.1 (sm_100a, tcgen05/TMA; fp64-acc parity tier + bf16 tensor-core tier)";
}

int alora_qkv_proj(int32_t dtype, const void* x, int32_t M, int32_t K, const void* w_qkv_t, int32_t Nq,
                   int32_t Nkv, const int32_t* row_slot, const uint8_t* row_apply, const void* lora_down,
                   const void* lora_up_t, int32_t n_slots, int32_t rank, const uint8_t* slot_targets, void* s_ws,
                   void* out, int32_t ld_out, void* stream) {
  if (M < 0 || K < 1 || Nq < 1 || Nkv < 1 || ld_out < Nq + 2 * Nkv) return ALORA_EINVAL;
  if (M == 0) return ALORA_OK;
  if (!x || !w_qkv_t || !out) return ALORA_EINVAL;
  const bool lora = n_slots > 0 && rank > 0 && lora_down && lora_up_t && row_slot && row_apply && slot_targets && s_ws;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  configure_kernels();
  const int N = Nq + 2 * Nkv;
  int rc;
  if (dtype == ALORA_F32) {
    rc = gemm_f64(kEpiStore, static_cast<const float*>(x), K, static_cast<const float*>(w_qkv_t), K,
                  static_cast<float*>(out), ld_out, M, N, K, st);
    if (rc != ALORA_OK || !lora) return rc;
    return lora_f64(static_cast<const float*>(x), M, K, row_slot, row_apply, static_cast<const float*>(lora_down),
                    static_cast<const float*>(lora_up_t), n_slots, rank, slot_targets, static_cast<float*>(s_ws), Nq,
                    Nkv, static_cast<float*>(out), ld_out, st);
  }
  if (dtype != ALORA_BF16) return ALORA_EINVAL;
  GemmLora gl;
  if (lora) {
    if (n_slots > 32) return ALORA_EINVAL;
    // masks live after the shrink output in the caller's workspace
    auto* sws = static_cast<__nv_bfloat16*>(s_ws);
    auto* masks = reinterpret_cast<uint32_t*>(sws + align_up(3LL * M * n_slots * rank, 128));
    rc = lora_tile_masks(row_slot, row_apply, M, masks, st);
    if (rc != ALORA_OK) return rc;
    rc = shrink(static_cast<const __nv_bfloat16*>(x), M, K, row_slot, row_apply,
                static_cast<const __nv_bfloat16*>(lora_down), n_slots, rank, slot_targets, sws, st, nullptr);
    if (rc != ALORA_OK) return rc;
    gl.s = sws;
    gl.up_t = static_cast<const __nv_bfloat16*>(lora_up_t);
    gl.ks = n_slots * rank;
    gl.n_q = Nq;
    gl.n_kv = Nkv;
    gl.tile_slot_mask = masks;
    gl.rank = rank;
  }
  return gemm_bf16(kEpiStore, static_cast<const __nv_bfloat16*>(x), K, static_cast<const __nv_bfloat16*>(w_qkv_t),
                   K, out, ld_out, M, N, K, lora ? &gl : nullptr, st);
}

int alora_kv_write(int32_t dtype, const void* k, const void* v, int64_t ld_src, const int32_t* slot_mapping,
                   int32_t M, int32_t kv_width, void* kv_pool, int32_t n_layers, int32_t layer, int32_t block_size,
                   void* stream) {
  if (dtype != ALORA_F32 && dtype != ALORA_BF16) return ALORA_EINVAL;
  if (M > 0 && (!k || !v || !slot_mapping || !kv_pool)) return ALORA_EINVAL;
  configure_kernels();
  return kv_write(dtype, k, v, ld_src, slot_mapping, M, kv_width, kv_pool, n_layers, layer, block_size,
                  static_cast<cudaStream_t>(stream));
}

int alora_paged_prefill_attn(int32_t dtype, const void* q, int64_t ld_q, int32_t n_rows, int32_t n_seqs,
                             const int32_t* cu_q, const int32_t* start_pos, const int32_t* block_table,
                             int32_t max_blocks, int32_t max_q, int32_t max_ctx, const void* kv_pool,
                             int32_t total_blocks, int32_t n_layers, int32_t layer, int32_t block_size,
                             int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, void* out, int64_t ld_out,
                             void* workspace, int64_t workspace_bytes, void* stream) {
  if (n_seqs < 0 || n_rows < 0 || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads || head_dim < 1 ||
      block_size < 1 || layer < 0 || layer >= n_layers || max_blocks < 1)
    return ALORA_EINVAL;
  if (n_seqs == 0 || n_rows == 0) return ALORA_OK;
  if (!q || !cu_q || !start_pos || !block_table || !kv_pool || !out) return ALORA_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  configure_kernels();
  if (dtype == ALORA_F32)
    return attn_f64(static_cast<const float*>(q), ld_q, n_rows, n_seqs, cu_q, start_pos, block_table, max_blocks,
                    static_cast<const float*>(kv_pool), n_layers, layer, block_size, n_heads, n_kv_heads, head_dim,
                    0.f, static_cast<float*>(out), ld_out, st);
  if (dtype != ALORA_BF16) return ALORA_EINVAL;
  const int64_t need = attn_bf16_workspace(n_rows, n_seqs, max_q, max_ctx, n_heads, n_kv_heads, head_dim);
  if (need > 0 && (workspace == nullptr || workspace_bytes < need)) return ALORA_EINVAL;
  return attn_bf16(static_cast<const __nv_bfloat16*>(q), ld_q, n_rows, n_seqs, cu_q, start_pos, block_table,
                   max_blocks, max_q, max_ctx, static_cast<const __nv_bfloat16*>(kv_pool), n_layers, layer,
                   block_size, n_heads, n_kv_heads, head_dim, static_cast<__nv_bfloat16*>(out), ld_out, workspace,
                   workspace_bytes, st, total_blocks);
}

int64_t alora_attn_partial_capacity(int32_t n_heads, int32_t head_dim) {
  if (n_heads < 1 || head_dim < 1) return ALORA_EINVAL;
  return attn_bf16_workspace_bound(n_heads, head_dim) - 4096 * 4;  // the executor's buffer minus merge counters
}

int alora_paged_prefix_attn(const void* q, int64_t ld_q, int32_t n_rows, int32_t n_seqs, const int32_t* positions,
                            const int32_t* row_seq, const int32_t* block_table, int32_t max_blocks,
                            const int32_t* plan, int32_t n_items, int32_t n_segs, int32_t n_sets, int32_t max_parts,
                            const void* kv_pool, int32_t total_blocks, int32_t n_layers, int32_t layer,
                            int32_t block_size, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, void* out,
                            int64_t ld_out, void* workspace, int64_t workspace_bytes, void* stream) {
  if (n_rows < 0 || n_seqs < 0 || n_items < 0 || n_segs < 0 || n_sets < 0 || max_parts < 1 || n_heads < 1 ||
      n_kv_heads < 1 || n_heads % n_kv_heads || layer < 0 || layer >= n_layers || max_blocks < 1)
    return ALORA_EINVAL;
  if (n_rows == 0 || n_items == 0) return ALORA_OK;
  if (!q || !positions || !row_seq || !block_table || !plan || !kv_pool || !out) return ALORA_EINVAL;
  configure_kernels();
  return attn_grouped(static_cast<const __nv_bfloat16*>(q), ld_q, n_rows, n_seqs, positions, row_seq, block_table,
                      max_blocks, plan, n_items, n_segs, n_sets, max_parts, true,
                      static_cast<const __nv_bfloat16*>(kv_pool), total_blocks, n_layers, layer, block_size, n_heads,
                      n_kv_heads, head_dim, static_cast<__nv_bfloat16*>(out), ld_out, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream));
}

int64_t alora_attn_workspace_bytes(int32_t dtype, int32_t n_rows, int32_t n_seqs, int32_t max_q, int32_t max_ctx,
                                   int32_t n_heads, int32_t n_kv_heads, int32_t head_dim) {
  if (dtype != ALORA_BF16) return 0;
  return attn_bf16_workspace(n_rows, n_seqs, max_q, max_ctx, n_heads, n_kv_heads, head_dim);
}

int alora_gemm_bf16(int32_t epi, const void* A, int32_t lda, const void* Bt, int32_t ldb, void* C, int32_t ldc,
                    int32_t M, int32_t N, int32_t K, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!A || !Bt || !C) return ALORA_EINVAL;
  if (epi != kEpiStore && epi != kEpiAdd && epi != kEpiRelu && epi != kEpiSwiglu && epi != 16) return ALORA_EINVAL;
  configure_kernels();
  const GemmWs ws = gemm_ws_from(workspace, workspace_bytes);
  return gemm_bf16(epi, static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(Bt), ldb, C,
                   ldc, M, N, K, nullptr, static_cast<cudaStream_t>(stream), ws.partial ? &ws : nullptr);
}

int64_t alora_gemm_workspace_bytes(void) { return gemm_bf16_workspace_bytes(); }

int alora_argmax(const float* logits, int32_t rows, int32_t vocab, int32_t* out_ids, void* stream) {
  if (rows < 0) return ALORA_EINVAL;
  configure_kernels();
  return argmax_rows(logits, rows, vocab, out_ids, static_cast<cudaStream_t>(stream));
}

int64_t alora_model_workspace_bytes(const AloraModelDesc* desc) {
  if (validate(desc) != ALORA_OK) return -1;
  return plan_ws(*desc).total;
}

int alora_model_create(const AloraModelDesc* desc, void** out_handle) {
  int rc = validate(desc);
  if (rc != ALORA_OK || !out_handle) return ALORA_EINVAL;
  configure_kernels();
  Model* m = new (std::nothrow) Model();
  if (!m) return ALORA_ECUDA;
  m->d = *desc;
  const int L = desc->n_layers;
  auto copy_ptrs = [L](const void* const* src, std::vector<const void*>& dst) {
    dst.assign(L, nullptr);
    if (src) for (int i = 0; i < L; ++i) dst[i] = src[i];
  };
  copy_ptrs(desc->w_qkv_t, m->w_qkv_t);
  copy_ptrs(desc->w_o_t, m->w_o_t);
  copy_ptrs(desc->w_in_t, m->w_in_t);
  copy_ptrs(desc->w_out_t, m->w_out_t);
  copy_ptrs(desc->lora_down, m->lora_down);
  copy_ptrs(desc->lora_up_t, m->lora_up_t);
  auto copy_opt = [&](const void* const* src, std::vector<const void*>& dst) {
    if (src && desc->n_slots > 0) copy_ptrs(src, dst);
  };
  copy_opt(desc->lora_o_down, m->lora_o_down);
  copy_opt(desc->lora_o_up_t, m->lora_o_up_t);
  copy_opt(desc->lora_in_down, m->lora_in_down);
  copy_opt(desc->lora_in_up_t, m->lora_in_up_t);
  copy_opt(desc->lora_out_down, m->lora_out_down);
  copy_opt(desc->lora_out_up_t, m->lora_out_up_t);
  m->attn_norm.assign(L, nullptr);
  m->mlp_norm.assign(L, nullptr);
  for (int i = 0; i < L; ++i) {
    if (desc->attn_norm) m->attn_norm[i] = desc->attn_norm[i];
    if (desc->mlp_norm) m->mlp_norm[i] = desc->mlp_norm[i];
  }
  // host arrays are not retained
  m->d.w_qkv_t = m->d.w_o_t = m->d.w_in_t = m->d.w_out_t = m->d.lora_down = m->d.lora_up_t = nullptr;
  m->d.attn_norm = m->d.mlp_norm = nullptr;
  m->d.lora_o_down = m->d.lora_o_up_t = m->d.lora_in_down = m->d.lora_in_up_t = nullptr;
  m->d.lora_out_down = m->d.lora_out_up_t = nullptr;
  auto pair_ok = [&](const std::vector<const void*>& a, const std::vector<const void*>& b) {
    if (a.empty() != b.empty()) return false;
    for (size_t i = 0; i < a.size(); ++i)
      if (!a[i] || !b[i]) return false;
    return true;
  };
  const bool extra_targets = !m->lora_o_down.empty() || !m->lora_in_down.empty() || !m->lora_out_down.empty();
  if (!pair_ok(m->lora_o_down, m->lora_o_up_t) || !pair_ok(m->lora_in_down, m->lora_in_up_t) ||
      !pair_ok(m->lora_out_down, m->lora_out_up_t) || (extra_targets && desc->dtype != ALORA_BF16)) {
    delete m;
    return ALORA_EINVAL;
  }
  for (int i = 0; i < L; ++i)
    if (!m->w_qkv_t[i] || !m->w_o_t[i] || !m->w_in_t[i] || !m->w_out_t[i] ||
        (desc->n_slots > 0 && (!m->lora_down[i] || !m->lora_up_t[i]))) {
      delete m;
      return ALORA_EINVAL;
    }
  if (!desc->embed || !desc->unembed_t || !desc->kv_pool || !desc->workspace ||
      desc->workspace_bytes < plan_ws(*desc).total) {
    delete m;
    return ALORA_EINVAL;
  }
  if (desc->tp_size > 1 && desc->tp_peers) {
    m->tp_peers.assign(desc->tp_peers, desc->tp_peers + desc->tp_size);
    for (void* p : m->tp_peers)
      if (!p) {
        delete m;
        return ALORA_EINVAL;
      }
  }
  m->d.tp_peers = nullptr;
  *out_handle = m;
  return ALORA_OK;
}

int alora_model_destroy(void* handle) {
  delete static_cast<Model*>(handle);
  return ALORA_OK;
}

int alora_model_forward(void* handle, const AloraStepDesc* step, void* stream) {
  if (!handle || !step) return ALORA_EINVAL;
  Model& m = *static_cast<Model*>(handle);
  if (step->n_tokens < 1 || step->n_tokens > m.d.max_tokens || step->n_seqs < 1 || step->n_seqs > m.d.max_seqs)
    return ALORA_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return m.d.dtype == ALORA_F32 ? forward_f32(m, *step, st) : forward_bf16(m, *step, st);
}

static bool same_step_buffers(const AloraStepDesc& a, const AloraStepDesc& b) {
  return a.tokens == b.tokens && a.positions == b.positions && a.slot_mapping == b.slot_mapping &&
         a.row_slot == b.row_slot && a.row_apply == b.row_apply && a.cu_q == b.cu_q && a.start_pos == b.start_pos &&
         a.block_table == b.block_table && a.last_row == b.last_row && a.logits == b.logits && a.next_ids == b.next_ids &&
         a.row_seq == b.row_seq && a.attn_plan == b.attn_plan && a.attn_segs == b.attn_segs && a.attn_sets == b.attn_sets;
}

// The captured forward for this step shape (capturing on first sight); nullptr + rc on failure.
static GraphEntry* graph_for(Model& m, const AloraStepDesc* step, cudaStream_t st, int* rc_out) {
  *rc_out = ALORA_OK;
  const GraphKey key{step->n_tokens, step->n_seqs, step->max_blocks, step->max_q, step->max_ctx,
                     step->attn_plan ? step->attn_items : -1,
                     (step->attn_plan ? step->attn_max_parts : -1) * 2 + (step->lora_rows_max <= kSegMaxRows ? 1 : 0)};
  auto it = m.graphs.find(key);
  if (it != m.graphs.end() && !same_step_buffers(it->second.step, *step)) {
    cudaGraphExecDestroy(it->second.exec);
    m.graphs.erase(it);
    it = m.graphs.end();
  }
  if (it == m.graphs.end()) {
    if (m.graphs.size() >= 32) {  // evict the least recently used capture
      auto lru = m.graphs.begin();
      for (auto j = m.graphs.begin(); j != m.graphs.end(); ++j)
        if (j->second.last_use < lru->second.last_use) lru = j;
      cudaGraphExecDestroy(lru->second.exec);
      m.graphs.erase(lru);
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      *rc_out = ALORA_ECUDA;
      return nullptr;
    }
    const int rc = forward_bf16(m, *step, st);
    const cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (rc != ALORA_OK) {
      if (g) cudaGraphDestroy(g);
      *rc_out = rc;
      return nullptr;
    }
    if (ce != cudaSuccess || g == nullptr) {
      *rc_out = ALORA_ECUDA;
      return nullptr;
    }
    GraphEntry e;
    const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      *rc_out = ALORA_ECUDA;
      return nullptr;
    }
    e.step = *step;
    e.launches = m.last_launches;
    it = m.graphs.emplace(key, e).first;
  }
  return &it->second;
}

int alora_model_forward_graph(void* handle, const AloraStepDesc* step, void* stream) {
  if (!handle || !step) return ALORA_EINVAL;
  Model& m = *static_cast<Model*>(handle);
  if (m.d.dtype != ALORA_BF16 || m.prof.on) return alora_model_forward(handle, step, stream);
  if (step->n_tokens < 1 || step->n_tokens > m.d.max_tokens || step->n_seqs < 1 || step->n_seqs > m.d.max_seqs)
    return ALORA_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc;
  GraphEntry* e = graph_for(m, step, st, &rc);
  if (!e) return rc;
  e->last_use = ++m.graph_clock;
  m.last_launches = e->launches;
  return cudaGraphLaunch(e->exec, st) == cudaSuccess ? ALORA_OK : ALORA_ECUDA;
}

int alora_model_graph_prepare(void* handle, const AloraStepDesc* step, void* stream) {
  if (!handle || !step) return ALORA_EINVAL;
  Model& m = *static_cast<Model*>(handle);
  if (m.d.dtype != ALORA_BF16 || m.prof.on) return ALORA_OK;
  if (step->n_tokens < 1 || step->n_tokens > m.d.max_tokens || step->n_seqs < 1 || step->n_seqs > m.d.max_seqs)
    return ALORA_EINVAL;
  int rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GraphEntry* e = graph_for(m, step, st, &rc);
  if (!e) return rc;
  if (!e->uploaded) {  // the first launch would upload the executable graph: do it here, off the critical path
    if (cudaGraphUpload(e->exec, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) return ALORA_ECUDA;
    e->uploaded = true;
  }
  return ALORA_OK;
}

int32_t alora_model_last_launches(void* handle) {
  return handle ? static_cast<Model*>(handle)->last_launches : -1;
}

int alora_model_set_profiling(void* handle, int32_t enable) {
  if (!handle) return ALORA_EINVAL;
  Profiler& p = static_cast<Model*>(handle)->prof;
  p.on = enable != 0;
  p.recs.clear();
  p.used = 0;
  return ALORA_OK;
}

int alora_model_profile_read(void* handle, int32_t max_kinds, char* names, float* ms, int32_t* counts,
                             double* bytes, double* flops) {
  if (!handle || max_kinds < 1 || !names || !ms || !counts || !bytes || !flops) return ALORA_EINVAL;
  Profiler& p = static_cast<Model*>(handle)->prof;
  std::vector<const char*> kinds;
  for (const ProfRec& r : p.recs) {
    int k = 0;
    while (k < (int)kinds.size() && std::strcmp(kinds[k], r.kind) != 0) ++k;
    if (k == (int)kinds.size()) {
      if (k == max_kinds) continue;
      kinds.push_back(r.kind);
      std::strncpy(names + 32 * k, r.kind, 31);
      names[32 * k + 31] = 0;
      ms[k] = 0.f;
      counts[k] = 0;
      bytes[k] = flops[k] = 0.0;
    }
    float t = 0.f;
    if (cudaEventElapsedTime(&t, p.events[r.ev0], p.events[r.ev1]) != cudaSuccess) return ALORA_ECUDA;
    ms[k] += t;
    counts[k] += 1;
    bytes[k] += r.bytes;
    flops[k] += r.flops;
  }
  return (int)kinds.size();
}

int64_t alora_model_profile_kernels(void* handle, char* buf, int64_t cap) {
  if (!handle) return ALORA_EINVAL;
  Profiler& p = static_cast<Model*>(handle)->prof;
  // one line per distinct (kind, kernel, grid): "kind<TAB>demangled kernel<TAB>grid CTAs<TAB>launches"
  std::vector<std::tuple<std::string, std::string, unsigned, int>> rows;
  for (const ProfRec& r : p.recs)
    for (const LaunchNote& k : r.kernels) {
      const char* raw = nullptr;
      std::string name = "?";
      if (cudaFuncGetName(&raw, k.fn) == cudaSuccess && raw) {
        int status = 0;
        char* dm = abi::__cxa_demangle(raw, nullptr, nullptr, &status);
        name = (status == 0 && dm) ? dm : raw;
        free(dm);
      }
      bool found = false;
      for (auto& row : rows)
        if (std::get<0>(row) == r.kind && std::get<1>(row) == name && std::get<2>(row) == k.grid) {
          ++std::get<3>(row);
          found = true;
          break;
        }
      if (!found) rows.emplace_back(r.kind, name, k.grid, 1);
    }
  std::string out;
  for (auto& row : rows)
    out += std::get<0>(row) + "\t" + std::get<1>(row) + "\t" + std::to_string(std::get<2>(row)) + "\t" +
           std::to_string(std::get<3>(row)) + "\n";
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, (int64_t)out.size());
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size() + 1;
}

}  // extern "C"
