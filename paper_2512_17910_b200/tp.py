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

Groups: `TorchDistGroup` all-reduces with torch.distributed (NCCL on B200s,
one process per GPU); `ThreadGroup` runs the ranks as threads of one process
(each on its own CUDA stream) and reduces on the device -- the single-GPU
harness the GPU tests use to check the sharded forward against the unsharded
one.
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

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_reduce(self, t) -> None:
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)


class ThreadGroup:
    """`size` ranks as threads of one process on one device: a host barrier orders the exchange and the
    sum runs on each rank's own stream (deterministic: ranks are added in rank order)."""

    def __init__(self, size: int):
        self.size = size
        self._barrier = threading.Barrier(size)
        self._slots = [None] * size

    def rank_view(self, rank: int):
        return _ThreadRank(self, rank)


class _ThreadRank:
    def __init__(self, parent: ThreadGroup, rank: int):
        self.parent, self.rank, self.size = parent, rank, parent.size

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
                 **kw):
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
        self._tp = (group.size, ctypes.cast(self._tp_cb, ctypes.c_void_p).value) if group.size > 1 else None
        # the all-reduce hook is a host callback (stream syncs / host barriers): not capturable in a CUDA graph
        kw.setdefault("graphs", group.size <= 1)
        super().__init__(scfg, weights=weights, init=init, **kw)
        self.pool_kv_width = scfg.kv_width

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
        try:
            super().launch(st)
        finally:
            if self._tp_error is not None:
                raise RuntimeError(f"tensor-parallel all-reduce failed: {self._tp_error}") from self._tp_error
