"""Model drop-in: the reference's model API, computed by libalora_sm100a.so on a B200.

Same names and behaviour as aloraserve/model.py:
  ModelConfig (model.py:25-42), generate_weights (73-92), project_qkv_masked
  (117-146), paged_attention (149-187), greedy_next_token (190-195), SeqInput
  (198-214), Model.forward_step (233-245) and its validation (247-259).

What changes is where the work runs: `Model.forward_step` packs every span
of the step into one varlen batch (the reference loops per span,
model.py:243) and makes ONE native call, alora_model_forward, which launches
all layers' kernels on the current CUDA stream. dtype "fp32" reproduces the
reference numerics (fp32 storage, fp64 accumulation); dtype "bf16" is the
tcgen05 tensor-core tier. arch "llama" adds RoPE/GQA/SwiGLU/weighted RMSNorm
(no reference counterpart).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .adapters import MODE_ACTIVATED, TARGET_BITS, LoraAdapter, target_shapes
from .weights import BaseWeights, LayerWeights, generate_weights, position_table, rope_tables

__all__ = ["ModelConfig", "LayerWeights", "BaseWeights", "generate_weights", "SeqInput", "Model",
           "project_qkv_masked", "paged_attention", "greedy_next_token", "write_kv"]


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int = 2
    n_heads: int = 4
    head_dim: int = 16
    d_model: int = 64
    vocab_size: int = 256
    max_seq_len: int = 8192
    seed: int = 0
    arch: str = "ref"  # "ref" (aloraserve) | "llama"
    n_kv_heads: int | None = None
    ffn_dim: int | None = None
    rope_theta: float = 500000.0
    dtype: str = "fp32"  # "fp32" (reference numerics) | "bf16" (tensor cores)

    def __post_init__(self):
        if min(self.n_layers, self.n_heads, self.head_dim, self.d_model, self.vocab_size) < 1:
            raise ValueError("all model dimensions must be positive")
        if self.arch not in ("ref", "llama"):
            raise ValueError(f"unknown arch {self.arch!r}")
        if self.dtype not in ("fp32", "bf16"):
            raise ValueError(f"unknown dtype {self.dtype!r}")
        if self.arch == "ref" and self.d_model != self.n_heads * self.head_dim:
            raise ValueError(f"d_model ({self.d_model}) must equal n_heads*head_dim ({self.n_heads}*{self.head_dim})")
        if self.n_heads % self.kv_heads:
            raise ValueError("n_heads must be a multiple of n_kv_heads")

    @property
    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def q_width(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_width(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def ffn(self) -> int:
        return 4 * self.d_model if self.ffn_dim is None else self.ffn_dim

    @property
    def rms_eps(self) -> float:
        return 1e-6 if self.arch == "ref" else 1e-5

    @property
    def native_dtype(self) -> int:
        return _native.ALORA_BF16 if self.dtype == "bf16" else _native.ALORA_F32


@dataclass
class SeqInput:
    """One request's span of a step (model.py:198-214)."""

    request_id: str
    tokens: np.ndarray
    start_pos: int
    block_ids: list
    adapter: LoraAdapter | None = None
    mask: np.ndarray | None = None


GLU_BLOCK = 64  # gate|up interleave granularity of the fused SwiGLU weight (kernels.h kGluBlock)


def _interleave_gate_up(gate: np.ndarray, up: np.ndarray) -> np.ndarray:
    """[d, F] gate and up -> [2F, d] rows: per 64-column block, 64 gate rows then 64 up rows."""
    d, F = gate.shape
    if F % GLU_BLOCK:
        raise ValueError(f"ffn_dim {F} must be a multiple of {GLU_BLOCK}")
    g = gate.T.reshape(F // GLU_BLOCK, GLU_BLOCK, d)
    u = up.T.reshape(F // GLU_BLOCK, GLU_BLOCK, d)
    return np.ascontiguousarray(np.concatenate([g, u], axis=1).reshape(2 * F, d))


class _StepBuffers:
    """Pinned host + device staging for one step's packed int32 metadata."""

    def __init__(self, torch, n_int32: int):
        self.cap = max(1024, n_int32)
        self.host = torch.empty(self.cap, dtype=torch.int32, pin_memory=True)
        self.dev = torch.empty(self.cap, dtype=torch.int32, device="cuda")


class Model:
    """Weights on the device plus the native step executor."""

    GRAPH_BLOCK_BUCKET = 32  # decode steps pad the block table to a multiple of this many blocks

    def __init__(self, config: ModelConfig | None = None, weights: BaseWeights | None = None, init: str = "philox",
                 max_tokens: int = 2048, max_seqs: int = 256, graphs: bool = True, shared_prefix: bool = True,
                 batch_invariant: bool = False):
        torch = _native.require_cuda()
        self._torch = torch
        # decode steps (one row per span, bf16) replay a captured CUDA graph of the whole forward
        self._graphs = bool(graphs) and (config or ModelConfig()).dtype == "bf16"
        c0 = config or ModelConfig()
        # shared-prefix attention: spans holding the same leading blocks (adapters on one conversation) read
        # that prefix once (alora_plan_attention + the grouped kernel) when a cost estimate says it pays
        # (_plan_attention); shared_prefix="always" takes every group, False / ALORA_SHARED_PREFIX=0 none
        import os
        self._shared_prefix_always = shared_prefix == "always"
        # batch_invariant (bf16): a token's KV / logits are bitwise independent of the step that computed it
        # (alora_sm100a.h AloraModelDesc.batch_invariant); the fp32 tier is invariant by construction
        self.batch_invariant = bool(batch_invariant) and c0.dtype == "bf16"
        self._shared_prefix = (bool(shared_prefix) and not self.batch_invariant and c0.dtype == "bf16"
                               and c0.head_dim in (64, 128)
                               and os.environ.get("ALORA_SHARED_PREFIX", "1") != "0")
        self._attn_partial_cap = int(_native.lib.alora_attn_partial_capacity(c0.n_heads, c0.head_dim)) \
            if c0.dtype == "bf16" else 0
        self._prefill_shapes = {}  # prefill step shape -> times seen (graph capture from the second)
        self._graph_stream = torch.cuda.Stream() if self._graphs else None
        self._staged_graphable = False
        self.config = cfg = config or ModelConfig()
        if init == "philox" or weights is not None:
            self.weights = weights if weights is not None else generate_weights(cfg)
        elif init == "device":
            self.weights = None
        else:
            raise ValueError(f"unknown init {init!r}")
        self._tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        self._upload_weights(init)
        self._adapters = {}  # adapter_id -> (slot, adapter)
        self._bank = None
        self._bank_version = 0
        self._ws = None
        self._ws_tokens = 0
        self._max_seqs = max_seqs
        self._grow_workspace(max_tokens)
        self._handle = None
        self._handle_key = None
        self._steps = _StepBuffers(torch, 8 * max_tokens + 8 * max_seqs)
        self._logits = torch.empty((max_seqs, cfg.vocab_size), dtype=torch.float32, device="cuda")
        self._ids = torch.empty(max_seqs, dtype=torch.int32, device="cuda")
        self._ids_host = torch.empty(max_seqs, dtype=torch.int32, pin_memory=True)
        # pipelined decode (launch_async / resolve): two pinned id buffers, the last launch's span count
        self._ids_pin = [torch.empty(max_seqs, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self._pin_slot = 0
        self._last_S = 0
        self._h2d_event = None  # the last metadata upload; the pinned staging buffer is rewritten only after it
        self.last_launches = 0

    # ------------------------------------------------------------ weights ---
    def _dev(self, a, dtype=None):
        t = self._torch
        return t.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype or self._tdt).contiguous()

    def _upload_weights(self, init):
        t, cfg = self._torch, self.config
        d, L = cfg.d_model, cfg.n_layers
        self._keep = []
        if self.weights is not None:
            w = self.weights
            self.embed = self._dev(w.embed)
            self.unembed_t = self.embed if w.unembed is None else self._dev(w.unembed.T)
            self.final_norm = None if w.final_norm is None else self._dev(w.final_norm, t.float32)
            self.w_qkv_t, self.w_o_t, self.w_in_t, self.w_out_t, self.attn_norm, self.mlp_norm = [], [], [], [], [], []
            for lw in w.layers:
                self.w_qkv_t.append(self._dev(np.concatenate([lw.wq, lw.wk, lw.wv], axis=1).T))
                self.w_o_t.append(self._dev(lw.wo.T))
                if cfg.arch == "llama":
                    self.w_in_t.append(self._dev(_interleave_gate_up(lw.w_in, lw.w_up)))
                else:
                    self.w_in_t.append(self._dev(lw.w_in.T))
                self.w_out_t.append(self._dev(lw.w_out.T))
                self.attn_norm.append(None if lw.attn_norm is None else self._dev(lw.attn_norm, t.float32))
                self.mlp_norm.append(None if lw.mlp_norm is None else self._dev(lw.mlp_norm, t.float32))
        else:  # random init directly in HBM (large configs; values do not change speed)
            g = t.Generator(device="cuda").manual_seed(cfg.seed)

            def rnd(shape, bound):
                return (t.rand(shape, generator=g, device="cuda", dtype=t.float32) * 2 - 1).mul_(bound).to(self._tdt)

            nqkv = cfg.q_width + 2 * cfg.kv_width
            self.embed = rnd((cfg.vocab_size, d), float(np.sqrt(3.0 / d)) if cfg.arch == "llama" else 0.1)
            self.unembed_t = self.embed if cfg.arch == "llama" else rnd((cfg.vocab_size, d), 0.1)
            self.final_norm = (1 + 0.1 * (2 * t.rand(d, generator=g, device="cuda") - 1)) if cfg.arch == "llama" else None
            b_d, b_q, b_f = (np.sqrt(3.0 / d), np.sqrt(3.0 / cfg.q_width), np.sqrt(3.0 / cfg.ffn)) \
                if cfg.arch == "llama" else (0.1, 0.1, 0.1)
            nin = 2 * cfg.ffn if cfg.arch == "llama" else cfg.ffn
            self.w_qkv_t = [rnd((nqkv, d), b_d) for _ in range(L)]
            self.w_o_t = [rnd((d, cfg.q_width), b_q) for _ in range(L)]
            self.w_in_t = [rnd((nin, d), b_d) for _ in range(L)]
            self.w_out_t = [rnd((d, cfg.ffn), b_f) for _ in range(L)]
            norm = (lambda: 1 + 0.1 * (2 * t.rand(d, generator=g, device="cuda") - 1)) if cfg.arch == "llama" else (lambda: None)
            self.attn_norm = [norm() for _ in range(L)]
            self.mlp_norm = [norm() for _ in range(L)]
        if cfg.arch == "ref":
            self.pos_table = self._dev(position_table(cfg.max_seq_len, d), t.float32)
            self.rope_cos = self.rope_sin = None
        else:
            c, s = rope_tables(cfg.max_seq_len, cfg.head_dim, cfg.rope_theta)
            self.pos_table = None
            self.rope_cos, self.rope_sin = self._dev(c, t.float32), self._dev(s, t.float32)

    @property
    def positions(self):
        return self.pos_table

    # ----------------------------------------------------------- adapters ---
    def _slot_for(self, adapter: LoraAdapter | None) -> int:
        if adapter is None:
            return -1
        hit = self._adapters.get(adapter.adapter_id)
        if hit is not None and hit[1] is adapter:
            return hit[0]
        if hit is not None:  # same id, different object: refresh its factors
            self._adapters[adapter.adapter_id] = (hit[0], adapter)
        else:
            self._adapters[adapter.adapter_id] = (len(self._adapters), adapter)
        self._rebuild_bank()
        return self._adapters[adapter.adapter_id][0]

    def register_adapter(self, adapter: LoraAdapter) -> int:
        """Upload an adapter's factors into the device bank; returns its slot."""
        return self._slot_for(adapter)

    def _rebuild_bank(self):
        cfg = self.config
        d, L = cfg.d_model, cfg.n_layers
        n = len(self._adapters)
        rank = max(a.rank for _, a in self._adapters.values())
        if cfg.dtype == "bf16":
            rank = -(-rank // 8) * 8  # 16-byte rows for the vector loads / TMA
            while (n * rank) % 64:  # shrink runs as a tcgen05 GEMM over [3 * n * rank] stacked rows
                n += 1
        if n > 32 and cfg.dtype == "bf16":
            raise ValueError("the bf16 tier supports at most 32 adapters per model")
        shapes = target_shapes(d, cfg.q_width, cfg.kv_width, cfg.ffn)
        offs = {"q": 0, "k": cfg.q_width, "v": cfg.q_width + cfg.kv_width}
        nqkv = cfg.q_width + 2 * cfg.kv_width
        llama = cfg.arch == "llama"
        used = {t for _, a in self._adapters.values() for t in a.targets}
        if used - set("qkv") and cfg.dtype != "bf16":
            raise ValueError("O / MLP adapter targets are served by the bf16 tier (dtype='bf16')")
        if "gate" in used and not llama:
            raise ValueError("the reference architecture's MLP has no gate projection")
        # planes of the MLP-in adapter bank: llama gate|up (interleaved SwiGLU weight), ref: up only
        in_names = ("gate", "up") if llama else ("up",)
        nin = 2 * cfg.ffn if llama else cfg.ffn
        targets = np.zeros(n, dtype=np.uint8)
        bank = {k: [] for k in ("down", "up_t", "o_down", "o_up_t", "in_down", "in_up_t", "out_down", "out_up_t")}

        def factors(a, tname, li):
            dn, upm = np.asarray(a.down[tname]), np.asarray(a.up[tname])
            if dn.ndim == 3:
                dn, upm = dn[li], upm[li]
            n_in, n_out = shapes[tname]
            if dn.shape != (n_in, a.rank) or upm.shape != (a.rank, n_out):
                raise ValueError(f"adapter {a.adapter_id} factor shapes do not match the model")
            return dn, upm

        for li in range(L):
            down = np.zeros((3, n, rank, d), dtype=np.float32)
            up_t = np.zeros((nqkv, n * rank), dtype=np.float32)
            o_down = np.zeros((1, n, rank, cfg.q_width), np.float32) if "o" in used else None
            o_up = np.zeros((d, n * rank), np.float32) if "o" in used else None
            has_in = bool(used & set(in_names))
            in_down = np.zeros((len(in_names), n, rank, d), np.float32) if has_in else None
            in_up = np.zeros((nin, len(in_names) * n * rank), np.float32) if has_in else None
            out_down = np.zeros((1, n, rank, cfg.ffn), np.float32) if "down" in used else None
            out_up = np.zeros((d, n * rank), np.float32) if "down" in used else None
            for slot, a in self._adapters.values():
                cols = slice(slot * rank, slot * rank + a.rank)
                for tname in a.targets:
                    targets[slot] |= 1 << TARGET_BITS[tname]
                    dn, upm = factors(a, tname, li)
                    if tname in offs:
                        down[TARGET_BITS[tname], slot, :a.rank, :] = dn.T
                        up_t[offs[tname]:offs[tname] + upm.shape[1], cols] = upm.T
                    elif tname == "o":
                        o_down[0, slot, :a.rank] = dn.T
                        o_up[:, cols] = upm.T
                    elif tname == "down":
                        out_down[0, slot, :a.rank] = dn.T
                        out_up[:, cols] = upm.T
                    else:  # gate / up: plane p, rows as the (interleaved) w_in_t rows
                        p = in_names.index(tname)
                        in_down[p, slot, :a.rank] = dn.T
                        pc = slice(p * n * rank + slot * rank, p * n * rank + slot * rank + a.rank)
                        if llama:
                            F = cfg.ffn
                            rows = (np.arange(F) // GLU_BLOCK) * 2 * GLU_BLOCK + np.arange(F) % GLU_BLOCK
                            in_up[rows + (GLU_BLOCK if tname == "up" else 0), pc] = upm.T
                        else:
                            in_up[:, pc] = upm.T
            bank["down"].append(self._dev(down))
            bank["up_t"].append(self._dev(up_t))
            for key, arr in (("o_down", o_down), ("o_up_t", o_up), ("in_down", in_down), ("in_up_t", in_up),
                             ("out_down", out_down), ("out_up_t", out_up)):
                if arr is not None:
                    bank[key].append(self._dev(arr))
        self._bank = dict(bank, rank=rank, n=n, targets=self._dev(targets, self._torch.uint8))
        self._bank_version += 1

    # ---------------------------------------------------------- workspace ---
    def _grow_workspace(self, tokens: int):
        if self._ws is not None and tokens <= self._ws_tokens:
            return
        self._ws_tokens = max(tokens, 2 * self._ws_tokens)
        self._ws = None
        desc = self._desc(kv=None, probe=True)
        nbytes = _native.lib.alora_model_workspace_bytes(ctypes.byref(desc))
        if nbytes < 0:
            raise ValueError("invalid model description")
        self._ws = self._torch.zeros(int(nbytes), dtype=self._torch.uint8, device="cuda")  # split-K counters = 0
        self._handle_key = None

    def _ptr_array(self, tensors):
        arr = (ctypes.c_void_p * len(tensors))(*[0 if x is None else x.data_ptr() for x in tensors])
        self._keep.append(arr)
        return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))

    def _desc(self, kv, probe=False):
        cfg = self.config
        D = _native.AloraModelDesc()
        D.arch = _native.ALORA_ARCH_LLAMA if cfg.arch == "llama" else _native.ALORA_ARCH_REF
        D.dtype = cfg.native_dtype
        D.n_layers, D.d_model, D.n_heads, D.n_kv_heads = cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.kv_heads
        D.head_dim, D.ffn_dim, D.vocab, D.max_seq_len = cfg.head_dim, cfg.ffn, cfg.vocab_size, cfg.max_seq_len
        D.rms_eps, D.rope_theta = cfg.rms_eps, cfg.rope_theta
        D.max_tokens, D.max_seqs = self._ws_tokens, self._max_seqs
        D.batch_invariant = int(self.batch_invariant)
        bank = self._bank
        D.n_slots = 0 if bank is None else bank["n"]
        D.lora_rank = 0 if bank is None else bank["rank"]
        tp = getattr(self, "_tp", None)  # (size, allreduce hook address): set by tp.TPModel
        if tp is not None:
            D.tp_size, D.tp_allreduce = tp
        tpf = getattr(self, "_tp_fused", None)  # (rank, peer buffer array, colocated): fused all-reduce
        if tpf is not None:
            D.tp_rank, D.tp_peers, D.tp_colocated = tpf
        if probe:
            return D
        D.embed, D.unembed_t = self.embed.data_ptr(), self.unembed_t.data_ptr()
        D.pos_table = None if self.pos_table is None else self.pos_table.data_ptr()
        D.rope_cos = None if self.rope_cos is None else self.rope_cos.data_ptr()
        D.rope_sin = None if self.rope_sin is None else self.rope_sin.data_ptr()
        D.final_norm = None if self.final_norm is None else self.final_norm.data_ptr()
        D.w_qkv_t, D.w_o_t = self._ptr_array(self.w_qkv_t), self._ptr_array(self.w_o_t)
        D.w_in_t, D.w_out_t = self._ptr_array(self.w_in_t), self._ptr_array(self.w_out_t)
        D.attn_norm, D.mlp_norm = self._ptr_array(self.attn_norm), self._ptr_array(self.mlp_norm)
        if bank is not None:
            D.lora_down, D.lora_up_t = self._ptr_array(bank["down"]), self._ptr_array(bank["up_t"])
            D.slot_targets = bank["targets"].data_ptr()
            for key in ("o_down", "o_up_t", "in_down", "in_up_t", "out_down", "out_up_t"):
                if bank[key]:
                    setattr(D, "lora_" + key, self._ptr_array(bank[key]))
        D.kv_pool = kv.data_ptr()
        D.total_blocks, D.block_size = kv.shape[0], kv.shape[3]
        D.workspace, D.workspace_bytes = self._ws.data_ptr(), self._ws.numel()
        return D

    def _native_handle(self, kv):
        key = (kv.data_ptr(), tuple(kv.shape), self._ws.data_ptr(), self._bank_version)
        if self._handle is not None and self._handle_key == key:
            return self._handle
        self.close()
        self._keep = []
        need = _native.lib.alora_model_workspace_bytes(ctypes.byref(self._desc(kv=None, probe=True)))
        if need > self._ws.numel():  # the adapter bank grew: the LoRA workspace grows with it
            self._ws = self._torch.zeros(int(need), dtype=self._torch.uint8, device="cuda")
            key = (kv.data_ptr(), tuple(kv.shape), self._ws.data_ptr(), self._bank_version)
        desc = self._desc(kv)
        h = ctypes.c_void_p()
        _native.check(_native.lib.alora_model_create(ctypes.byref(desc), ctypes.byref(h)), "alora_model_create")
        self._handle, self._handle_key = h, key
        if getattr(self, "_profiling", False):
            _native.lib.alora_model_set_profiling(h, 1)
        return h

    def close(self):
        if getattr(self, "_handle", None) is not None:
            _native.lib.alora_model_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ forward ---
    def _check_pool(self, kv):
        t, cfg = self._torch, self.config
        if not isinstance(kv, t.Tensor) or not kv.is_cuda:
            raise ValueError("kv must be the BlockPool's device tensor (BlockPool(..., storage='cuda').kv)")
        if kv.dtype != self._tdt or kv.dim() != 5 or kv.shape[1] != cfg.n_layers or kv.shape[2] != 2 \
                or kv.shape[4] != cfg.kv_width or not kv.is_contiguous():
            raise ValueError(f"kv pool shape/dtype {tuple(kv.shape)} {kv.dtype} does not match the model")

    def pack(self, seqs, block_size: int, token_refs: bool = False) -> dict:
        """Validate (model.py:250-259, 160-163) and pack all spans into one varlen int32 record."""
        cfg = self.config
        S = len(seqs)
        if S == 0:
            raise ValueError("no spans")
        if S > self._max_seqs:
            raise ValueError(f"{S} spans exceed max_seqs {self._max_seqs}")
        lens, starts, slot_ids, masked, toks, tables = [], [], [], [], [], []
        const_apply = []
        for i, seq in enumerate(seqs):
            tk = np.asarray(seq.tokens, dtype=np.int64).reshape(-1)
            n = len(tk)
            if n == 0:
                raise ValueError("empty span")
            if seq.start_pos < 0 or seq.start_pos + n > cfg.max_seq_len:
                raise ValueError("span exceeds max_seq_len")
            need = -(-(seq.start_pos + n) // block_size)
            if len(seq.block_ids) < need:
                raise ValueError(f"block table has {len(seq.block_ids)} blocks, need {need}")
            ad = seq.adapter
            if ad is None:
                const_apply.append(0)
            elif ad.mode == MODE_ACTIVATED:
                if seq.mask is None:
                    raise ValueError(f"activated adapter span for {seq.request_id} is missing its mask")
                m = np.asarray(seq.mask, dtype=bool)
                if m.shape != (n,):
                    raise ValueError(f"mask shape {m.shape} does not match {n} rows")
                const_apply.append(0)
                masked.append((i, m))
            else:  # standard LoRA: adapted on every row (model.py:260-261)
                const_apply.append(1)
            slot_ids.append(self._slot_for(ad))
            lens.append(n)
            starts.append(int(seq.start_pos))
            toks.append(tk)
            tables.append(seq.block_ids[:need])
        tokens = np.concatenate(toks) if S > 1 else toks[0]
        if tokens.max() >= cfg.vocab_size:
            raise ValueError("token id outside the vocabulary")
        if tokens.min() < 0:
            # token_refs: -(j+1) = the previous launch's greedy id of its span j (resolved on the device)
            if not token_refs or int(tokens.min()) < -self._last_S:
                raise ValueError("token id outside the vocabulary")
        M = int(sum(lens))
        lens_a = np.asarray(lens, dtype=np.int64)
        starts_a = np.asarray(starts, dtype=np.int64)
        cu = np.zeros(S + 1, dtype=np.int32)
        np.cumsum(lens_a, out=cu[1:])
        row_seq = np.repeat(np.arange(S), lens_a)
        positions = (np.arange(M, dtype=np.int64) - np.repeat(cu[:-1] - starts_a, lens_a)).astype(np.int32)
        row_apply = np.repeat(np.asarray(const_apply, dtype=np.uint8), lens_a)
        for i, m in masked:
            row_apply[cu[i]:cu[i + 1]] = ~m
        maxb = max(len(tb) for tb in tables)
        graphable = self._graphs and max(lens) == 1  # a decode step: replay a captured graph
        if graphable:  # bucket the table width (and the context bound below) so one capture serves many steps
            bb = self.GRAPH_BLOCK_BUCKET
            maxb = -(-maxb // bb) * bb
        elif self._graphs:
            # a prefill step whose exact shape recurs (fixed-batch pipelines: every eval turn of a conversation
            # set) is captured on its second sighting and replayed after that; one-off shapes stay eager, so
            # they never pay a capture. Replay removes the host launch gaps of the eager executor (~4%).
            key = (int(lens_a.sum()), S, maxb, int(lens_a.max()), int((starts_a + lens_a).max()))
            seen = self._prefill_shapes.get(key, 0) + 1
            self._prefill_shapes[key] = seen
            if len(self._prefill_shapes) > 4096:
                self._prefill_shapes.clear()
            graphable = seen >= 2
        bt = np.zeros((S, maxb), dtype=np.int32)
        for i, tb in enumerate(tables):
            bt[i, :len(tb)] = tb
        slot_map = (bt[row_seq, positions // block_size] * block_size + positions % block_size).astype(np.int32)
        ends = starts_a + lens_a
        plan, kv_tokens = None, float(ends.sum())
        if getattr(self, "_shared_prefix", False) and S >= 2:
            plan = self._plan_attention(cu, starts_a.astype(np.int32), bt, block_size)
            if plan is not None:
                kv_tokens = float(plan[5])  # distinct keys: a shared prefix is read once
        row_slot = np.repeat(np.asarray(slot_ids, dtype=np.int32), lens_a)
        take = row_slot[(row_slot >= 0) & (row_apply != 0)]
        return {
            "lora_rows_max": int(np.bincount(take).max()) if take.size else 0,
            "attn_plan": plan, "row_seq": row_seq.astype(np.int32),
            "attn_kv_tokens": kv_tokens,
            "attn_qk_pairs": float((lens_a * (starts_a + (lens_a + 1) / 2)).sum()),
            "M": M, "S": S, "maxb": maxb, "max_q": int(lens_a.max()),
            "max_ctx": maxb * block_size if graphable else int(ends.max()),
            "graphable": graphable,
            "tokens": tokens.astype(np.int32), "positions": positions, "slot_mapping": slot_map,
            "row_slot": row_slot, "row_apply": row_apply,
            "cu_q": cu, "start_pos": starts_a.astype(np.int32), "last_row": (cu[1:] - 1).astype(np.int32),
            "block_table": bt,
        }

    def _plan_attention(self, cu, starts, bt, block_size):
        """Shared-prefix attention plan (alora_plan_attention) for steps whose spans hold the same leading
        physical blocks (adapters evaluated on one conversation); None when no span shares a prefix."""
        cfg = self.config
        S, maxb = bt.shape
        if block_size > 64 or 64 % block_size:  # the kernel's TMA page boxes tile a 64-key tile
            return None
        cap = 8 + 64 * (int(cu[-1]) + S) + 4096
        for _ in range(2):
            out = np.empty(cap, dtype=np.int32)
            n = _native.lib.alora_plan_attention(S, cu.ctypes.data, starts.ctypes.data, bt.ctypes.data, maxb,
                                                 block_size, cfg.n_heads, cfg.kv_heads, cfg.head_dim, 1,
                                                 self._attn_partial_cap, out.ctypes.data, cap)
            if n >= 0:
                break
            if n == _native.ALORA_EINVAL:
                _native.check(int(n), "alora_plan_attention")
            cap = int(-n)
        else:
            raise RuntimeError("alora_plan_attention: plan buffer sizing failed")
        if int(out[2]) == S:  # no group formed: the per-span kernels serve the step
            return None
        # Grouping pays when the prefix bytes it saves outweigh its fixed cost: the per-span kernels stream
        # every span's keys at ~5 TB/s, the grouped one runs at ~0.8 PFLOP/s plus ~25 us of per-CTA setup and
        # partition merge (B200, measured: C3, 8 adapters x 8k, grouped 169 vs per-span 432 us per layer; C2,
        # 3 adapters x 2k, grouped 33 vs per-span 25 us)
        n_q = np.diff(cu).astype(np.float64)
        ends = starts.astype(np.float64) + n_q
        span_s = float(ends.sum()) * 2 * cfg.kv_width * 2 / 5e12
        grp_s = 4.0 * cfg.n_heads * cfg.head_dim * float((n_q * (starts + n_q / 2)).sum()) / 0.8e15 + 25e-6
        if span_s < grp_s and not self._shared_prefix_always:
            return None
        return out[:n]

    _FIELDS = ("tokens", "positions", "slot_mapping", "row_slot", "cu_q", "start_pos", "last_row", "block_table",
               "row_seq")

    def run_packed(self, p: dict, kv, want_logits: bool = True):
        """One native forward over a packed step. Returns (next_ids[S], logits[S, V] or None) on the host."""
        t = self._torch
        st = self.stage(p, kv)
        self.launch(st)
        S = p["S"]
        self._ids_host[:S].copy_(self._ids[:S], non_blocking=True)
        logits = self._logits[:S].cpu().numpy() if want_logits else None
        t.cuda.current_stream().synchronize()
        self.last_d2h_bytes = 4 * S + (logits.nbytes if logits is not None else 0)
        self._last_S = S
        return self._ids_host[:S].numpy().copy(), logits

    def launch_async(self, p: dict, kv):
        """Stage and launch a packed step without waiting for it; the greedy ids come back through `resolve`.
        The step may reference the previous launch's ids (pack(token_refs=True)): pipelined decode."""
        t = self._torch
        st = self.stage(p, kv)
        self._h2d_event = t.cuda.Event()  # the pinned staging buffer is rewritten only after this upload ran
        self._h2d_event.record()
        self.launch(st)
        S = p["S"]
        self._pin_slot ^= 1
        buf = self._ids_pin[self._pin_slot]
        buf[:S].copy_(self._ids[:S], non_blocking=True)
        ev = t.cuda.Event()
        ev.record()
        self._last_S = S
        self.last_d2h_bytes = 4 * S
        return ev, buf, S

    @staticmethod
    def resolve(handle) -> np.ndarray:
        """Wait for a launch_async step and return its greedy ids."""
        ev, buf, S = handle
        ev.synchronize()
        return buf[:S].numpy().copy()

    def launch(self, st) -> None:
        """Enqueue one staged step on the current stream (decode steps: a CUDA-graph replay); no host sync."""
        cur = self._torch.cuda.current_stream()
        if self._staged_graphable and not getattr(self, "_profiling", False):
            gs = self._graph_stream  # capture/replay needs a non-legacy stream; ordered against the caller's
            gs.wait_stream(cur)
            _native.check(_native.lib.alora_model_forward_graph(self._handle, ctypes.byref(st),
                                                                ctypes.c_void_p(gs.cuda_stream)),
                          "alora_model_forward_graph")
            cur.wait_stream(gs)
        else:
            _native.check(_native.lib.alora_model_forward(self._handle, ctypes.byref(st),
                                                          ctypes.c_void_p(cur.cuda_stream)), "alora_model_forward")
        self.last_launches = _native.lib.alora_model_last_launches(self._handle)

    def stage(self, p: dict, kv):
        """Upload a packed step's metadata (one pinned H2D copy on the current stream); returns its descriptor."""
        t = self._torch
        self._check_pool(kv)
        self._grow_workspace(p["M"])
        handle = self._native_handle(kv)
        plan = p.get("attn_plan")
        parts = [p[f] for f in self._FIELDS]
        # row_apply: bytes packed in int32, then the attention plan (if any)
        sizes = [x.size for x in parts] + [(len(p["row_apply"]) + 3) // 4] + [0 if plan is None else plan.size]
        offs = np.cumsum([0] + sizes)
        total = int(offs[-1])
        if total > self._steps.cap:
            self._steps = _StepBuffers(t, 2 * total)
        if self._h2d_event is not None:  # a pipelined step's upload may still be queued behind the running one
            self._h2d_event.synchronize()
            self._h2d_event = None
        host = self._steps.host.numpy()
        for i, x in enumerate(parts):  # straight into the pinned staging buffer (no intermediate concatenation)
            host[offs[i]:offs[i + 1]] = np.asarray(x).reshape(-1)
        ap = host[offs[-3]:offs[-2]].view(np.uint8)
        ap[:len(p["row_apply"])] = p["row_apply"]
        ap[len(p["row_apply"]):] = 0
        if plan is not None:
            host[offs[-2]:offs[-1]] = plan
        dev = self._steps.dev
        dev[:total].copy_(self._steps.host[:total], non_blocking=True)
        base = dev.data_ptr()
        ptr = {f: base + 4 * int(offs[i]) for i, f in enumerate(self._FIELDS)}
        st = _native.AloraStepDesc()
        st.n_tokens, st.n_seqs, st.max_blocks, st.max_q, st.max_ctx = p["M"], p["S"], p["maxb"], p["max_q"], p["max_ctx"]
        st.tokens, st.positions, st.slot_mapping = ptr["tokens"], ptr["positions"], ptr["slot_mapping"]
        st.row_slot, st.cu_q, st.start_pos = ptr["row_slot"], ptr["cu_q"], ptr["start_pos"]
        st.last_row, st.block_table = ptr["last_row"], ptr["block_table"]
        st.row_apply = base + 4 * int(offs[len(self._FIELDS)])
        st.logits, st.next_ids = self._logits.data_ptr(), self._ids.data_ptr()
        st.attn_kv_tokens, st.attn_qk_pairs = p.get("attn_kv_tokens", 0.0), p.get("attn_qk_pairs", 0.0)
        st.row_seq = ptr["row_seq"]
        st.lora_rows_max = p.get("lora_rows_max", 1 << 30)
        if plan is not None:
            st.attn_plan = base + 4 * int(offs[-2])
            st.attn_items, st.attn_segs, st.attn_sets, st.attn_max_parts = (int(x) for x in plan[:4])
        self._staged_graphable = bool(p.get("graphable", False))
        self.last_h2d_bytes = 4 * total
        return st

    def set_profiling(self, enable: bool, kv=None) -> None:
        """CUDA-event bracketing of every native launch (per-kernel time + algorithmic bytes/flops)."""
        self._profiling = bool(enable)
        if self._handle is not None:
            _native.check(_native.lib.alora_model_set_profiling(self._handle, int(enable)), "set_profiling")

    def profile_read(self) -> dict:
        """{kind: {"ms", "launches", "bytes", "flops"}} accumulated since set_profiling(True); syncs the stream."""
        if self._handle is None:
            return {}
        self._torch.cuda.current_stream().synchronize()
        k = 32
        names = ctypes.create_string_buffer(32 * k)
        ms = (ctypes.c_float * k)()
        cnt = (ctypes.c_int32 * k)()
        by = (ctypes.c_double * k)()
        fl = (ctypes.c_double * k)()
        n = _native.lib.alora_model_profile_read(self._handle, k, names, ms, cnt, by, fl)
        if n < 0:
            _native.check(n, "profile_read")
        out = {}
        for i in range(n):
            name = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
            out[name] = {"ms": float(ms[i]), "launches": int(cnt[i]), "bytes": float(by[i]), "flops": float(fl[i])}
        return out

    def profile_kernels(self) -> list:
        """[(kind, kernel name, grid CTAs, launches)] of the launches recorded since set_profiling(True)."""
        if self._handle is None:
            return []
        n = _native.lib.alora_model_profile_kernels(self._handle, None, 0)
        if n < 0:
            _native.check(int(n), "profile_kernels")
        buf = ctypes.create_string_buffer(int(n))
        _native.lib.alora_model_profile_kernels(self._handle, buf, int(n))
        rows = []
        for line in buf.value.decode().splitlines():
            kind, name, grid, cnt = line.split("\t")
            rows.append((kind, name, int(grid), int(cnt)))
        return rows

    def forward_step(self, seqs, kv) -> dict:
        """Run every span of a step; returns {request_id: float32[V] logits of the span's last row}."""
        p = self.pack(seqs, int(kv.shape[3]))
        _, logits = self.run_packed(p, kv, want_logits=True)
        return {seq.request_id: logits[i] for i, seq in enumerate(seqs)}


# ----------------------------------------------------- function-level API ---
def _np_or_torch(x):
    t = _native.require_cuda()
    if isinstance(x, t.Tensor):
        return x, True
    return t.as_tensor(np.ascontiguousarray(x, dtype=np.float32)), False


def project_qkv_masked(x, weights: LayerWeights, adapter: LoraAdapter | None = None, mask=None):
    """Masked Q/K/V projection (model.py:117-146) via alora_qkv_proj, fp32 tier (reference numerics)."""
    t = _native.require_cuda()
    xt, was_torch = _np_or_torch(x)
    xt = xt.to(device="cuda", dtype=t.float32).contiguous()
    M, K = xt.shape
    wq, wk, wv = (np.asarray(w, dtype=np.float32) for w in (weights.wq, weights.wk, weights.wv))
    nq, nkv = wq.shape[1], wk.shape[1]
    if adapter is not None and mask is not None:
        mask = np.asarray(mask, dtype=bool)
        if mask.shape != (M,):
            raise ValueError(f"mask shape {mask.shape} does not match {M} rows")
    w_t = t.as_tensor(np.ascontiguousarray(np.concatenate([wq, wk, wv], axis=1).T)).cuda()
    out = t.empty((M, nq + 2 * nkv), dtype=t.float32, device="cuda")
    args = [None] * 6
    n_slots = rank = 0
    keep = []
    if adapter is not None:
        rank = adapter.rank
        n_slots = 1
        down = np.zeros((3, 1, rank, K), np.float32)
        up_t = np.zeros((nq + 2 * nkv, rank), np.float32)
        offs = {"q": (0, nq), "k": (nq, nkv), "v": (nq + nkv, nkv)}
        tb = 0
        for ti, tn in enumerate("qkv"):
            if tn in adapter.targets:
                tb |= 1 << ti
                down[ti, 0] = np.asarray(adapter.down[tn]).T
                o, w = offs[tn]
                up_t[o:o + w] = np.asarray(adapter.up[tn]).T
        apply = np.ones(M, np.uint8) if (adapter.mode != MODE_ACTIVATED or mask is None) else (~mask).astype(np.uint8)
        if adapter.mode == MODE_ACTIVATED and mask is None:
            apply = np.ones(M, np.uint8)  # mask None == standard path (model.py:142-143)
        keep = [t.zeros(M, dtype=t.int32, device="cuda"), t.as_tensor(apply).cuda(),
                t.as_tensor(down).cuda(), t.as_tensor(up_t).cuda(),
                t.tensor([tb], dtype=t.uint8, device="cuda"),
                t.empty(3 * M * rank + 256, dtype=t.float32, device="cuda")]
        args = [k.data_ptr() for k in keep]
    stream = t.cuda.current_stream().cuda_stream
    rc = _native.lib.alora_qkv_proj(_native.ALORA_F32, xt.data_ptr(), M, K, w_t.data_ptr(), nq, nkv,
                                    args[0], args[1], args[2], args[3], n_slots, rank, args[4], args[5],
                                    out.data_ptr(), nq + 2 * nkv, ctypes.c_void_p(stream))
    _native.check(rc, "alora_qkv_proj")
    q, k, v = out[:, :nq], out[:, nq:nq + nkv], out[:, nq + nkv:]
    if was_torch:
        return q, k, v
    t.cuda.current_stream().synchronize()
    return q.cpu().numpy(), k.cpu().numpy(), v.cpu().numpy()


def write_kv(kv, layer: int, block_ids, start_pos: int, k, v) -> None:
    """Paged scatter of k/v rows into the device pool (model.py:217-222) via alora_kv_write."""
    t = _native.require_cuda()
    B = kv.shape[3]
    kt = t.as_tensor(np.ascontiguousarray(k)) if not isinstance(k, t.Tensor) else k
    vt = t.as_tensor(np.ascontiguousarray(v)) if not isinstance(v, t.Tensor) else v
    kt = kt.to(device="cuda", dtype=kv.dtype).contiguous()
    vt = vt.to(device="cuda", dtype=kv.dtype).contiguous()
    n = kt.shape[0]
    pos = start_pos + np.arange(n)
    ids = np.asarray(block_ids, dtype=np.int64)[pos // B]
    slots = t.as_tensor((ids * B + pos % B).astype(np.int32)).cuda()
    dt = _native.ALORA_BF16 if kv.dtype == t.bfloat16 else _native.ALORA_F32
    rc = _native.lib.alora_kv_write(dt, kt.data_ptr(), vt.data_ptr(), kt.shape[1], slots.data_ptr(), n,
                                    kt.shape[1], kv.data_ptr(), kv.shape[1], layer, B,
                                    ctypes.c_void_p(t.cuda.current_stream().cuda_stream))
    _native.check(rc, "alora_kv_write")


def paged_attention(q, kv, layer: int, block_ids, fresh_k, fresh_v, start_pos: int, n_heads: int,
                    n_kv_heads: int | None = None):
    """Causal attention over cached context + fresh span (model.py:149-187) via alora_paged_prefill_attn.

    Like the reference it does not modify `kv`: the needed blocks are gathered
    into a scratch pool together with the fresh rows, then attended.
    """
    t = _native.require_cuda()
    was_torch = isinstance(q, t.Tensor)
    n = q.shape[0]
    B = kv.shape[3]
    total = start_pos + n
    need = -(-total // B)
    if len(block_ids) < need:
        raise ValueError(f"block table has {len(block_ids)} blocks, need {need}")
    kvt = kv if isinstance(kv, t.Tensor) else t.as_tensor(np.ascontiguousarray(kv))
    dtype = t.bfloat16 if kvt.dtype == t.bfloat16 else t.float32
    ids = t.as_tensor(np.asarray(block_ids[:need], dtype=np.int64))
    scratch = kvt[ids.to(kvt.device), layer:layer + 1].to(device="cuda", dtype=dtype).contiguous()
    write_kv(scratch, 0, list(range(need)), start_pos, fresh_k, fresh_v)
    qt = (q if was_torch else t.as_tensor(np.ascontiguousarray(q))).to(device="cuda", dtype=dtype).contiguous()
    hkv = n_heads if n_kv_heads is None else n_kv_heads
    D = qt.shape[1] // n_heads
    out = t.empty_like(qt)
    cu = t.tensor([0, n], dtype=t.int32, device="cuda")
    sp = t.tensor([start_pos], dtype=t.int32, device="cuda")
    bt = t.arange(need, dtype=t.int32, device="cuda")
    dt = _native.ALORA_BF16 if dtype == t.bfloat16 else _native.ALORA_F32
    wsb = _native.lib.alora_attn_workspace_bytes(dt, n, 1, n, total, n_heads, hkv, D)
    ws = t.zeros(max(int(wsb), 1), dtype=t.uint8, device="cuda")  # split-KV merge counters start at 0
    rc = _native.lib.alora_paged_prefill_attn(dt, qt.data_ptr(), qt.shape[1], n, 1, cu.data_ptr(), sp.data_ptr(),
                                              bt.data_ptr(), need, n, total, scratch.data_ptr(), need, 1, 0, B, n_heads,
                                              hkv, D, out.data_ptr(), out.shape[1], ws.data_ptr(), ws.numel(),
                                              ctypes.c_void_p(t.cuda.current_stream().cuda_stream))
    _native.check(rc, "alora_paged_prefill_attn")
    if was_torch:
        return out
    return out.float().cpu().numpy()


def greedy_next_token(logits) -> int:
    """Argmax with ties to the lowest id (model.py:190-195), on the device via alora_argmax."""
    t = _native.require_cuda()
    lt = logits if isinstance(logits, t.Tensor) else t.as_tensor(np.asarray(logits))
    if lt.dim() != 1:
        raise ValueError(f"expected a logits vector, got shape {tuple(lt.shape)}")
    lt = lt.to(device="cuda", dtype=t.float32).contiguous()
    out = t.empty(1, dtype=t.int32, device="cuda")
    rc = _native.lib.alora_argmax(lt.data_ptr(), 1, lt.shape[0], out.data_ptr(),
                                  ctypes.c_void_p(t.cuda.current_stream().cuda_stream))
    _native.check(rc, "alora_argmax")
    return int(out.item())
