"""Tensor parallelism for the llama architecture (Llama-3-70B TP=8).

The reference has no parallelism (single process, engine.py). This module shards
a model across `size` ranks the Megatron way, so that each rank runs the same
native executor on a smaller "model":

  * q|k|v projections are column-parallel by head: rank r owns q heads
    [r*H/T, (r+1)*H/T) and kv heads [r*Hkv/T, (r+1)*Hkv/T);
  * gate|up are column-parallel over the FFN dimension, the O-projection and
    MLP-down are row-parallel (their input dimension is sharded), so each rank
    produces a partial residual update that is all-reduced before the residual
    add + RMSNorm (the `tp_allreduce` hook of alora_model_forward);
  * the aLoRA down factors (A, [d, r]) are replicated and the up factors (B)
    are column-sharded with the weights they correct, so the masked LoRA
    delta needs no collective of its own;
  * embeddings, norms and the lm_head are replicated; the paged KV pool of a
    rank holds its own kv heads ([NB, L, 2, B, Hkv/T * D]). Block ids, block
    tables and block hashes are identical on every rank because every rank
    runs the same deterministic scheduler on the same requests.

The all-reduce. By default (`fused=True`) it is the executor's own kernel
(csrc/tp_allreduce.cu): every rank maps every other rank's symmetric buffer
(alora_tp_buffer_bytes), the row-parallel GEMM writes its fp32 partial into its
own buffer, and one kernel per rank sums all ranks' partials in rank order over
peer memory (NVLink / NVSwitch), adds the residual and applies the next RMSNorm
-- no host round trip, so the whole TP forward is CUDA-graph capturable.
`fused=False` keeps the host hook (group.all_reduce through torch.distributed).

Groups: `TorchDistGroup` is one process per GPU: its peer buffers are exchanged
as CUDA IPC handles over the torch.distributed group (NCCL on B200s), and its
hook path all-reduces with NCCL. `ThreadGroup` runs the ranks as threads of one
process (each on its own CUDA stream, peer buffers are plain device memory of
the one GPU) -- the single-GPU harness the GPU tests use to check the sharded
forward against the unsharded one.
"""

import ctypes
import threading
from dataclasses import replace

import numpy as np

from . import _native
from .adapters import LoraAdapter
from .model import Model, ModelConfig
from .weights import BaseWeights, LayerWeights, generate_weights

__all__ = ["shard_config", "shard_weights", "shard_adapter", "TorchDistGroup", "ThreadGroup", "TPModel"]


def shard_config(cfg: ModelConfig, size: int) -> ModelConfig:
    """The per-rank model of a `size`-way tensor-parallel llama model."""
    if size < 1:
        raise ValueError("tp size must be >= 1")
    if size == 1:
        return cfg
    if cfg.arch != "llama":
        raise ValueError("tensor parallelism is implemented for the llama architecture")
    if cfg.n_heads % size or cfg.kv_heads % size or cfg.ffn % size:
        raise ValueError(f"heads ({cfg.n_heads}/{cfg.kv_heads}) and ffn ({cfg.ffn}) must divide by tp={size}")
    if (cfg.ffn // size) % 64:
        raise ValueError("the per-rank ffn must be a multiple of 64 (fused SwiGLU blocks)")
    return replace(cfg, n_heads=cfg.n_heads // size, n_kv_heads=cfg.kv_heads // size, ffn_dim=cfg.ffn // size)


def _cols(a, r, n):
    w = a.shape[-1] // n
    return np.ascontiguousarray(a[..., r * w:(r + 1) * w])


def _rows(a, r, n):
    h = a.shape[0] // n
    return np.ascontiguousarray(a[r * h:(r + 1) * h])


def shard_weights(w: BaseWeights, cfg: ModelConfig, size: int, rank: int) -> BaseWeights:
    """Rank `rank`'s slice of full host weights (weights are stored [in, out])."""
    if size == 1:
        return w
    shard_config(cfg, size)  # validates
    layers = []
    for lw in w.layers:
        layers.append(LayerWeights(
            wq=_cols(lw.wq, rank, size), wk=_cols(lw.wk, rank, size), wv=_cols(lw.wv, rank, size),
            wo=_rows(lw.wo, rank, size),
            w_in=_cols(lw.w_in, rank, size), w_up=None if lw.w_up is None else _cols(lw.w_up, rank, size),
            w_out=_rows(lw.w_out, rank, size),
            attn_norm=lw.attn_norm, mlp_norm=lw.mlp_norm))
    return BaseWeights(embed=w.embed, layers=layers, unembed=w.unembed, final_norm=w.final_norm)


def shard_adapter(ad: LoraAdapter, cfg: ModelConfig, size: int, rank: int) -> LoraAdapter:
    """Down factors replicated, up factors column-sharded like the projection they correct."""
    if size == 1:
        return ad
    up = {t: _cols(np.asarray(ad.up[t]), rank, size) for t in ad.targets}
    return replace(ad, up=up)


def _tensor_at(ptr: int, count: int):
    """Zero-copy fp32 torch view of `count` values at a device pointer (CUDA array interface)."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f4", "data": (int(ptr), False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device="cuda")


class TorchDistGroup:
    """One process per GPU: in-place sum all-reduce over a torch.distributed process group (NCCL)."""

    colocated = False

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._own = None
        self._opened = []

    def all_reduce(self, t) -> None:
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)

    def peer_buffers(self, nbytes: int) -> list:
        """Allocate this rank's symmetric buffer and map every peer's (CUDA IPC handles exchanged over the
        group); returns the device pointer of each rank's buffer in this process, in rank order."""
        lib = _native.lib
        own = ctypes.c_void_p()
        _native.check(lib.alora_device_alloc(int(nbytes), ctypes.byref(own)), "alora_device_alloc")
        self._own = own.value
        handle = (ctypes.c_uint8 * 64)()
        _native.check(lib.alora_ipc_get_handle(self._own, handle), "alora_ipc_get_handle")
        handles = [None] * self.size
        self._dist.all_gather_object(handles, (self.rank, bytes(handle)), group=self.group)
        ptrs = [0] * self.size
        for r, h in handles:
            if r == self.rank:
                ptrs[r] = self._own
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * 64).from_buffer_copy(h)
            _native.check(lib.alora_ipc_open(buf, ctypes.byref(p)), "alora_ipc_open")
            self._opened.append(p.value)
            ptrs[r] = p.value
        self._dist.barrier(group=self.group)
        return ptrs

    def close(self) -> None:
        for p in self._opened:
            _native.lib.alora_ipc_close(p)
        self._opened = []
        if self._own:
            self._dist.barrier(group=self.group)  # no peer still maps it
            _native.lib.alora_device_free(self._own)
            self._own = None


class ThreadGroup:
    """`size` ranks as threads of one process on one device: a host barrier orders the exchange and the
    sum runs on each rank's own stream (deterministic: ranks are added in rank order)."""

    def __init__(self, size: int):
        self.size = size
        self._barrier = threading.Barrier(size)
        self._slots = [None] * size
        self._buffers = None
        self._lock = threading.Lock()

    def rank_view(self, rank: int):
        return _ThreadRank(self, rank)

    def peer_buffers(self, nbytes: int) -> list:
        import torch

        with self._lock:
            if self._buffers is None or self._buffers[0].numel() < nbytes:
                self._buffers = [torch.zeros(int(nbytes), dtype=torch.uint8, device="cuda") for _ in range(self.size)]
                torch.cuda.synchronize()
            return [b.data_ptr() for b in self._buffers]


class _ThreadRank:
    colocated = True  # every rank on the same GPU

    def __init__(self, parent: ThreadGroup, rank: int):
        self.parent, self.rank, self.size = parent, rank, parent.size

    def peer_buffers(self, nbytes: int) -> list:
        return self.parent.peer_buffers(nbytes)

    def launch_barrier(self) -> None:
        """Every rank has finished its host-side step preparation before any rank enqueues the forward: a
        rank spinning in the fused all-reduce must not meet a peer still inside a device-synchronising
        CUDA call (an allocation or pageable copy while staging), which would wait for the spinner."""
        self.parent._barrier.wait()

    def all_reduce(self, t) -> None:
        import torch

        p = self.parent
        torch.cuda.current_stream().synchronize()
        p._slots[self.rank] = t
        p._barrier.wait()
        total = p._slots[0].clone()
        for r in range(1, p.size):
            total += p._slots[r]
        torch.cuda.current_stream().synchronize()
        p._barrier.wait()  # everyone has read every rank's buffer
        t.copy_(total)
        torch.cuda.current_stream().synchronize()
        p._barrier.wait()


class TPModel(Model):
    """Model drop-in for one tensor-parallel rank: `config` is the FULL model, the rank holds its shard.

    The engine on every rank is identical (same requests, same scheduler); the pool it builds must use
    `pool_kv_width` (this rank's kv heads), and adapters registered with full factors are sharded here.
    """

    def __init__(self, config: ModelConfig, group, weights: BaseWeights | None = None, init: str = "philox",
                 fused: bool = True, **kw):
        self.full_config = config
        self.tp_group = group
        scfg = shard_config(config, group.size)
        if weights is None and init == "philox":
            weights = generate_weights(config)
        if weights is not None:
            weights = shard_weights(weights, config, group.size, group.rank)
        self._tp_shards = {}
        self._tp_error = None

        def _cb(ctx, buf, count, stream):
            try:
                group.all_reduce(_tensor_at(buf, count))
                return 0
            except Exception as e:  # surfaced by forward(): the native call sees a failed hook
                self._tp_error = e
                return _native.ALORA_ECUDA

        self._tp_cb = _native.ALLREDUCE_FN(_cb)  # kept alive for the handle's lifetime
        fused = fused and group.size > 1 and hasattr(group, "peer_buffers")
        self._tp_fused = None
        if fused:
            # the peer-buffer layout is sized for a fixed step capacity: the workspace never grows past it
            self._tp_max_tokens = int(kw.get("max_tokens", 2048))
            nbytes = int(_native.lib.alora_tp_buffer_bytes(self._tp_max_tokens, config.d_model))
            peers = group.peer_buffers(nbytes)
            arr = (ctypes.c_void_p * group.size)(*peers)
            self._tp_peer_arr = arr
            self._tp_fused = (group.rank, ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), int(group.colocated))
            self._tp = (group.size, None)
            import os
            if os.environ.get("ALORA_TP_GRAPHS", "1") == "0":  # debug / A-B: eager decode steps
                kw["graphs"] = False
        else:
            self._tp = (group.size, ctypes.cast(self._tp_cb, ctypes.c_void_p).value) if group.size > 1 else None
            # the all-reduce hook is a host callback (stream syncs / host barriers): not capturable in a graph
            kw.setdefault("graphs", group.size <= 1)
        super().__init__(scfg, weights=weights, init=init, **kw)
        self.pool_kv_width = scfg.kv_width

    def _grow_workspace(self, tokens: int):
        if self._tp_fused is not None:
            if tokens > self._tp_max_tokens:
                raise ValueError(f"step of {tokens} rows exceeds the TP model's max_tokens {self._tp_max_tokens}")
            if self._ws is not None:
                return
            tokens = self._tp_max_tokens
        super()._grow_workspace(tokens)

    def _slot_for(self, adapter: LoraAdapter | None) -> int:
        if adapter is None:
            return -1
        sh = self._tp_shards.get(adapter.adapter_id)
        if sh is None or sh[0] is not adapter:
            sh = (adapter, shard_adapter(adapter, self.full_config, self.tp_group.size, self.tp_group.rank))
            self._tp_shards[adapter.adapter_id] = sh
        return super()._slot_for(sh[1])

    def launch(self, st) -> None:
        self._tp_error = None
        if self._tp_fused is not None and getattr(self.tp_group, "colocated", False):
            if self._staged_graphable and not getattr(self, "_profiling", False):  # capture before the barrier
                gs = self._graph_stream
                gs.wait_stream(self._torch.cuda.current_stream())
                _native.check(_native.lib.alora_model_graph_prepare(self._handle, ctypes.byref(st),
                                                                    ctypes.c_void_p(gs.cuda_stream)),
                              "alora_model_graph_prepare")
            self.tp_group.launch_barrier()
        try:
            super().launch(st)
        finally:
            if self._tp_error is not None:
                raise RuntimeError(f"tensor-parallel all-reduce failed: {self._tp_error}") from self._tp_error
