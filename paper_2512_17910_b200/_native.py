"""ctypes binding of libalora_sm100a.so (include/alora_sm100a.h).

The product path has no CPU fallback: if the library is missing this module
raises at import, and device entry points raise if CUDA is unavailable.
Statuses map like the reference's errors: ALORA_EINVAL -> ValueError,
everything else -> RuntimeError.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ALORA_LIB (developer A/B switch) loads another in-tree build of the same library
LIB_PATH = os.environ.get("ALORA_LIB") or os.path.join(_HERE, "libalora_sm100a.so")

ALORA_OK = 0
ALORA_EINVAL = -1
ALORA_ECUDA = -2
ALORA_EUNSUPPORTED = -3
ALORA_ENOSPC = -4
ALORA_ESTATE = -5
ALORA_F32 = 0
ALORA_BF16 = 1
ALORA_ARCH_REF = 0
ALORA_ARCH_LLAMA = 1

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_2512_17910_b200`). There is no CPU fallback."
    )

lib = ctypes.CDLL(LIB_PATH)

c_void_p = ctypes.c_void_p
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_u8p = ctypes.POINTER(ctypes.c_uint8)


class AloraModelDesc(ctypes.Structure):
    _fields_ = [
        ("arch", c_i32), ("dtype", c_i32),
        ("n_layers", c_i32), ("d_model", c_i32), ("n_heads", c_i32), ("n_kv_heads", c_i32),
        ("head_dim", c_i32), ("ffn_dim", c_i32), ("vocab", c_i32), ("max_seq_len", c_i32),
        ("rms_eps", c_f32), ("rope_theta", c_f32),
        ("max_tokens", c_i32), ("max_seqs", c_i32),
        ("embed", c_void_p), ("unembed_t", c_void_p), ("pos_table", c_void_p),
        ("rope_cos", c_void_p), ("rope_sin", c_void_p), ("final_norm", c_void_p),
        ("w_qkv_t", ctypes.POINTER(c_void_p)), ("w_o_t", ctypes.POINTER(c_void_p)),
        ("w_in_t", ctypes.POINTER(c_void_p)), ("w_out_t", ctypes.POINTER(c_void_p)),
        ("attn_norm", ctypes.POINTER(c_void_p)), ("mlp_norm", ctypes.POINTER(c_void_p)),
        ("n_slots", c_i32), ("lora_rank", c_i32),
        ("lora_down", ctypes.POINTER(c_void_p)), ("lora_up_t", ctypes.POINTER(c_void_p)),
        ("slot_targets", c_void_p),
        ("kv_pool", c_void_p), ("total_blocks", c_i32), ("block_size", c_i32),
        ("workspace", c_void_p), ("workspace_bytes", c_i64),
        ("tp_size", c_i32), ("tp_ctx", c_void_p), ("tp_allreduce", c_void_p),
        ("lora_o_down", ctypes.POINTER(c_void_p)), ("lora_o_up_t", ctypes.POINTER(c_void_p)),
        ("lora_in_down", ctypes.POINTER(c_void_p)), ("lora_in_up_t", ctypes.POINTER(c_void_p)),
        ("lora_out_down", ctypes.POINTER(c_void_p)), ("lora_out_up_t", ctypes.POINTER(c_void_p)),
        ("tp_rank", c_i32), ("tp_peers", ctypes.POINTER(c_void_p)), ("tp_colocated", c_i32),
        ("batch_invariant", c_i32),
    ]


# int32_t (*alora_allreduce_fn)(void* ctx, float* buf, int64_t count, void* stream)
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, c_void_p, c_void_p, c_i64, c_void_p)


class AloraStepDesc(ctypes.Structure):
    _fields_ = [
        ("n_tokens", c_i32), ("n_seqs", c_i32), ("max_blocks", c_i32), ("max_q", c_i32), ("max_ctx", c_i32),
        ("tokens", c_void_p), ("positions", c_void_p), ("slot_mapping", c_void_p), ("row_slot", c_void_p),
        ("row_apply", c_void_p), ("cu_q", c_void_p), ("start_pos", c_void_p), ("block_table", c_void_p),
        ("last_row", c_void_p), ("logits", c_void_p), ("next_ids", c_void_p),
        ("attn_kv_tokens", ctypes.c_double), ("attn_qk_pairs", ctypes.c_double),
        ("row_seq", c_void_p), ("attn_plan", c_void_p),
        ("attn_items", c_i32), ("attn_segs", c_i32), ("attn_sets", c_i32), ("attn_max_parts", c_i32),
        ("lora_rows_max", c_i32),
    ]


def _sig(name, restype, *argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


# Every symbol declared in include/alora_sm100a.h (tests check this list against the header).
EXPORTS = {
    "alora_version": _sig("alora_version", ctypes.c_char_p),
    "alora_hash_block": _sig("alora_hash_block", c_i32, c_void_p, c_void_p, c_i32, ctypes.c_char_p, c_i32, c_void_p),
    "alora_hash_chain": _sig("alora_hash_chain", c_i32, c_void_p, c_void_p, c_i64, c_i32, ctypes.c_char_p,
                             c_void_p, c_void_p),
    "alora_hash_chains": _sig("alora_hash_chains", c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_i32, c_void_p,
                              c_void_p, c_void_p, c_i32),
    "alora_hash_requests": _sig("alora_hash_requests", c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_i32, c_void_p, c_i32),
    "alora_pool_create": _sig("alora_pool_create", c_void_p, c_i32, c_i32),
    "alora_pool_destroy": _sig("alora_pool_destroy", None, c_void_p),
    "alora_pool_views": _sig("alora_pool_views", c_i32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p),
    "alora_pool_num_free": _sig("alora_pool_num_free", c_i32, c_void_p),
    "alora_pool_lookup": _sig("alora_pool_lookup", c_i64, c_void_p, c_void_p, c_i64, c_void_p),
    "alora_pool_allocate": _sig("alora_pool_allocate", c_i32, c_void_p, c_i64, c_void_p),
    "alora_pool_release": _sig("alora_pool_release", c_i32, c_void_p, c_void_p, c_i64),
    "alora_pool_publish": _sig("alora_pool_publish", c_i32, c_void_p, c_void_p, c_void_p, c_i64),
    "alora_pool_set_fill": _sig("alora_pool_set_fill", c_i32, c_void_p, c_void_p, c_i64, c_i64, c_i64),
    "alora_pool_free_list": _sig("alora_pool_free_list", c_i64, c_void_p, c_void_p, c_i64),
    "alora_pool_index_get": _sig("alora_pool_index_get", c_i32, c_void_p, c_void_p),
    "alora_pool_index_dump": _sig("alora_pool_index_dump", c_i64, c_void_p, c_void_p, c_void_p, c_i64),
    "alora_sched_create": _sig("alora_sched_create", c_void_p, c_void_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32),
    "alora_sched_destroy": _sig("alora_sched_destroy", None, c_void_p),
    "alora_sched_submit": _sig("alora_sched_submit", c_i32, c_void_p, c_void_p, c_i64, c_i32, c_i32, ctypes.c_char_p,
                               c_i32, c_i64),
    "alora_sched_has_work": _sig("alora_sched_has_work", c_i32, c_void_p),
    "alora_sched_step": _sig("alora_sched_step", c_i32, c_void_p, c_void_p, c_i32, c_void_p, c_i32, c_void_p, c_i32,
                             c_void_p, c_void_p, c_i64, c_void_p),
    "alora_sched_step_done": _sig("alora_sched_step_done", c_i32, c_void_p, c_i32, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p),
    "alora_sched_set_token": _sig("alora_sched_set_token", c_i32, c_void_p, c_i32, c_i64, c_i64),
    "alora_sched_retire": _sig("alora_sched_retire", c_i32, c_void_p, c_i32),
    "alora_sched_info": _sig("alora_sched_info", c_i32, c_void_p, c_i32, c_void_p),
    "alora_sched_blocks": _sig("alora_sched_blocks", c_i64, c_void_p, c_i32, c_void_p, c_i64),
    "alora_sched_owned_total": _sig("alora_sched_owned_total", c_i64, c_void_p),
    "alora_qkv_proj": _sig("alora_qkv_proj", c_i32, c_i32, c_void_p, c_i32, c_i32, c_void_p, c_i32, c_i32,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_void_p, c_void_p, c_void_p,
                           c_i32, c_void_p),
    "alora_kv_write": _sig("alora_kv_write", c_i32, c_i32, c_void_p, c_void_p, c_i64, c_void_p, c_i32, c_i32,
                           c_void_p, c_i32, c_i32, c_i32, c_void_p),
    "alora_paged_prefill_attn": _sig("alora_paged_prefill_attn", c_i32, c_i32, c_void_p, c_i64, c_i32, c_i32,
                                     c_void_p, c_void_p, c_void_p, c_i32, c_i32, c_i32, c_void_p, c_i32, c_i32,
                                     c_i32, c_i32, c_i32, c_i32, c_i32, c_void_p, c_i64, c_void_p, c_i64, c_void_p),
    "alora_attn_workspace_bytes": _sig("alora_attn_workspace_bytes", c_i64, c_i32, c_i32, c_i32, c_i32, c_i32,
                                       c_i32, c_i32, c_i32),
    "alora_plan_attention": _sig("alora_plan_attention", c_i64, c_i32, c_void_p, c_void_p, c_void_p, c_i32, c_i32,
                                 c_i32, c_i32, c_i32, c_i32, c_i64, c_void_p, c_i64),
    "alora_attn_partial_capacity": _sig("alora_attn_partial_capacity", c_i64, c_i32, c_i32),
    "alora_paged_prefix_attn": _sig("alora_paged_prefix_attn", c_i32, c_void_p, c_i64, c_i32, c_i32, c_void_p,
                                    c_void_p, c_void_p, c_i32, c_void_p, c_i32, c_i32, c_i32, c_i32, c_void_p,
                                    c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_void_p, c_i64, c_void_p,
                                    c_i64, c_void_p),
    "alora_gemm_bf16": _sig("alora_gemm_bf16", c_i32, c_i32, c_void_p, c_i32, c_void_p, c_i32, c_void_p, c_i32,
                            c_i32, c_i32, c_i32, c_void_p, c_i64, c_void_p),
    "alora_gemm_workspace_bytes": _sig("alora_gemm_workspace_bytes", c_i64),
    "alora_argmax": _sig("alora_argmax", c_i32, c_void_p, c_i32, c_i32, c_void_p, c_void_p),
    "alora_tp_buffer_bytes": _sig("alora_tp_buffer_bytes", c_i64, c_i32, c_i32),
    "alora_tp_partial_offset": _sig("alora_tp_partial_offset", c_i64, c_i32, c_i32, c_i32),
    "alora_device_alloc": _sig("alora_device_alloc", c_i32, c_i64, c_void_p),
    "alora_device_free": _sig("alora_device_free", c_i32, c_void_p),
    "alora_ipc_get_handle": _sig("alora_ipc_get_handle", c_i32, c_void_p, c_void_p),
    "alora_ipc_open": _sig("alora_ipc_open", c_i32, c_void_p, c_void_p),
    "alora_ipc_close": _sig("alora_ipc_close", c_i32, c_void_p),
    "alora_tp_allreduce_norm": _sig("alora_tp_allreduce_norm", c_i32, c_void_p, c_i32, c_i32, c_i32, c_i32, c_i32,
                                    c_i32, c_i32, c_void_p, c_void_p, c_f32, c_void_p, c_void_p),
    "alora_model_workspace_bytes": _sig("alora_model_workspace_bytes", c_i64, ctypes.POINTER(AloraModelDesc)),
    "alora_model_create": _sig("alora_model_create", c_i32, ctypes.POINTER(AloraModelDesc),
                               ctypes.POINTER(c_void_p)),
    "alora_model_destroy": _sig("alora_model_destroy", c_i32, c_void_p),
    "alora_model_forward": _sig("alora_model_forward", c_i32, c_void_p, ctypes.POINTER(AloraStepDesc), c_void_p),
    "alora_model_graph_prepare": _sig("alora_model_graph_prepare", c_i32, c_void_p, c_void_p, c_void_p),
    "alora_model_forward_graph": _sig("alora_model_forward_graph", c_i32, c_void_p, ctypes.POINTER(AloraStepDesc),
                                      c_void_p),
    "alora_model_last_launches": _sig("alora_model_last_launches", c_i32, c_void_p),
    "alora_model_set_profiling": _sig("alora_model_set_profiling", c_i32, c_void_p, c_i32),
    "alora_model_profile_read": _sig("alora_model_profile_read", c_i32, c_void_p, c_i32, c_void_p, c_void_p,
                                     c_void_p, c_void_p, c_void_p),
    "alora_model_profile_kernels": _sig("alora_model_profile_kernels", c_i64, c_void_p, c_void_p, c_i64),
}


def check(rc: int, what: str) -> None:
    if rc == ALORA_OK:
        return
    if rc == ALORA_EINVAL:
        raise ValueError(f"{what}: invalid argument (ALORA_EINVAL)")
    if rc == ALORA_ESTATE:
        raise AssertionError(f"{what}: block pool invariant violated (ALORA_ESTATE)")
    if rc == ALORA_EUNSUPPORTED:
        raise RuntimeError(f"{what}: unsupported configuration (ALORA_EUNSUPPORTED)")
    raise RuntimeError(f"{what}: CUDA error (status {rc})")


def require_cuda():
    """The device path is the only path: fail loudly without a GPU."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("libalora_sm100a needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch


def version() -> str:
    return lib.alora_version().decode()
