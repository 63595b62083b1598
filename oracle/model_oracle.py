"""CPU ORACLE (test infrastructure only) — numpy restatement of the model hot path.

Follows /root/reference/pkg/src/aloraserve/model.py line by line for the
reference ("ref") architecture:

  * deterministic weights ............ model.py:62-92, adapters.py:29-33, 85-91
  * mm = fp32(fp64 @ fp64) ........... model.py:95-98
  * rmsnorm (no gain, eps 1e-6) ...... model.py:101-104
  * sinusoidal position table ........ model.py:107-114
  * project_qkv_masked (row select) .. model.py:117-146
  * paged_attention (fp64 softmax) ... model.py:149-187
  * greedy_next_token ................ model.py:190-195
  * _write_kv ........................ model.py:217-222
  * forward of one span .............. model.py:247-272

and adds two things the reference does not have (parity unpinned: no
reference file pins them, they are checked only through the shared pieces):

  * arch="llama": RoPE (rotate-half), GQA (n_kv_heads < n_heads), SwiGLU MLP,
    weighted RMSNorm (eps 1e-5), lm_head tied to the embedding.
  * numerics="bf16": the rounding points of the B200 bf16 path (weights, GEMM
    inputs, q/k/v, KV cache, attention output are bf16 values; every
    accumulation here is fp64, the GPU's is fp32), so GPU-vs-oracle error is
    accumulation order only.
  * adapter targets "o", "gate", "up", "down" (the reference accepts q/k/v only,
    adapters.py:26, 61-63): the same masked base + (x @ down) @ up of
    model.py:141-145 applied to the O-projection and MLP projections
    (`_adapted`). Parity unpinned: an extension checked GPU vs this oracle.
"""

import hashlib
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OracleConfig", "bf16_round", "oracle_weights", "oracle_adapter", "mm", "rmsnorm",
    "position_table", "rope_tables", "apply_rope", "project_qkv_masked", "paged_attention",
    "write_kv", "greedy_next_token", "OracleModel", "OracleAdapter", "OracleSpan",
    "detect_invocation", "activation_mask",
]

MODE_ACTIVATED = "activated"
MODE_STANDARD = "standard"


@dataclass(frozen=True)
class OracleConfig:
    """Shape of the model. arch "ref" is aloraserve.model.ModelConfig (model.py:25-42)."""

    arch: str = "ref"
    n_layers: int = 2
    n_heads: int = 4
    head_dim: int = 16
    d_model: int = 64
    vocab_size: int = 256
    max_seq_len: int = 8192
    seed: int = 0
    n_kv_heads: int | None = None  # None -> n_heads (MHA, the reference)
    ffn_dim: int | None = None  # None -> 4*d_model (ref ReLU MLP)
    rope_theta: float = 500000.0
    numerics: str = "fp64acc"  # "fp64acc" (reference) | "bf16"

    @property
    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def ffn(self) -> int:
        return 4 * self.d_model if self.ffn_dim is None else self.ffn_dim

    @property
    def q_width(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_width(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def rms_eps(self) -> float:
        return 1e-6 if self.arch == "ref" else 1e-5


def bf16_round(x) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 values."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def _tensor_rng(tag: str) -> np.random.Generator:
    # Philox keyed by blake2b-128(tag), little endian (model.py:62-66, adapters.py:29-33)
    key = int.from_bytes(hashlib.blake2b(tag.encode(), digest_size=16).digest(), "little")
    return np.random.Generator(np.random.Philox(key=key))


def _init(seed: int, name: str, shape, scale: float = 0.1) -> np.ndarray:
    # model.py:69-70 (scale 0.1); llama tensors use a fan-in scale
    return _tensor_rng(f"weights:{seed}:{name}").uniform(-scale, scale, shape).astype(np.float32)


def oracle_weights(cfg: OracleConfig) -> dict:
    """Deterministic weights. For arch="ref" byte-identical to generate_weights (model.py:73-92)."""
    d = cfg.d_model
    w = {"layers": []}
    if cfg.arch == "ref":
        if cfg.kv_heads != cfg.n_heads or cfg.q_width != d:
            raise ValueError("ref arch is MHA with d_model == n_heads*head_dim")
        for li in range(cfg.n_layers):
            w["layers"].append({
                "wq": _init(cfg.seed, f"l{li}.wq", (d, d)),
                "wk": _init(cfg.seed, f"l{li}.wk", (d, d)),
                "wv": _init(cfg.seed, f"l{li}.wv", (d, d)),
                "wo": _init(cfg.seed, f"l{li}.wo", (d, d)),
                "w_in": _init(cfg.seed, f"l{li}.w_in", (d, cfg.ffn)),
                "w_out": _init(cfg.seed, f"l{li}.w_out", (cfg.ffn, d)),
            })
        w["embed"] = _init(cfg.seed, "embed", (cfg.vocab_size, d))
        w["unembed"] = _init(cfg.seed, "unembed", (d, cfg.vocab_size))
    elif cfg.arch == "llama":
        s_d = float(np.sqrt(3.0 / d))
        s_q = float(np.sqrt(3.0 / cfg.q_width))
        s_f = float(np.sqrt(3.0 / cfg.ffn))
        for li in range(cfg.n_layers):
            w["layers"].append({
                "attn_norm": 1.0 + _init(cfg.seed, f"l{li}.attn_norm", (d,)),
                "wq": _init(cfg.seed, f"l{li}.wq", (d, cfg.q_width), s_d),
                "wk": _init(cfg.seed, f"l{li}.wk", (d, cfg.kv_width), s_d),
                "wv": _init(cfg.seed, f"l{li}.wv", (d, cfg.kv_width), s_d),
                "wo": _init(cfg.seed, f"l{li}.wo", (cfg.q_width, d), s_q),
                "mlp_norm": 1.0 + _init(cfg.seed, f"l{li}.mlp_norm", (d,)),
                "w_gate": _init(cfg.seed, f"l{li}.w_gate", (d, cfg.ffn), s_d),
                "w_up": _init(cfg.seed, f"l{li}.w_up", (d, cfg.ffn), s_d),
                "w_down": _init(cfg.seed, f"l{li}.w_down", (cfg.ffn, d), s_f),
            })
        w["embed"] = _init(cfg.seed, "embed", (cfg.vocab_size, d), s_d)  # tied lm_head: unit-scale logits
        w["final_norm"] = 1.0 + _init(cfg.seed, "final_norm", (d,))
        w["unembed"] = None  # tied: logits = h @ embed.T
    else:
        raise ValueError(f"unknown arch {cfg.arch!r}")
    if cfg.numerics == "bf16":
        # GEMM operands are bf16 on the GPU; RMSNorm gains stay fp32 there, so they do here
        for layer in w["layers"]:
            for k in layer:
                if not k.endswith("_norm"):
                    layer[k] = bf16_round(layer[k])
        for k in ("embed", "unembed"):
            if w.get(k) is not None:
                w[k] = bf16_round(w[k])
    return w


@dataclass
class OracleAdapter:
    """LoraAdapter (adapters.py:36-66): down[t] (d, r), up[t] (r, out_t)."""

    adapter_id: str
    rank: int
    mode: str = MODE_ACTIVATED
    targets: tuple = ("q", "k", "v")
    invocation_tokens: tuple | None = None
    down: dict = field(default_factory=dict)
    up: dict = field(default_factory=dict)


def oracle_adapter(adapter_id, cfg: OracleConfig, rank, seed=0, targets=("q", "k", "v"),
                   invocation_tokens=None, mode=MODE_ACTIVATED) -> OracleAdapter:
    """generate_adapter (adapters.py:68-101); out width per target for GQA."""
    d, q, kv, f = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.ffn
    shapes = {"q": (d, q), "k": (d, kv), "v": (d, kv), "o": (q, d), "gate": (d, f), "up": (d, f), "down": (f, d)}
    down, up = {}, {}
    for t in targets:
        n_in, n_out = shapes[t]
        dn = _tensor_rng(f"adapter:{adapter_id}:{seed}:{t}:down").uniform(-0.1, 0.1, (n_in, rank)).astype(np.float32)
        upm = _tensor_rng(f"adapter:{adapter_id}:{seed}:{t}:up").uniform(-0.1, 0.1, (rank, n_out)).astype(np.float32)
        if cfg.numerics == "bf16":
            dn, upm = bf16_round(dn), bf16_round(upm)
        down[t], up[t] = dn, upm
    inv = tuple(int(x) for x in invocation_tokens) if invocation_tokens is not None else None
    return OracleAdapter(adapter_id, rank, mode, tuple(targets), inv, down, up)


def mm(a, b) -> np.ndarray:
    """fp64 accumulation, one rounding to fp32 (model.py:95-98)."""
    return (np.asarray(a).astype(np.float64, copy=False) @ np.asarray(b).astype(np.float64, copy=False)).astype(np.float32)


def rmsnorm(x, weight=None, eps: float = 1e-6) -> np.ndarray:
    """model.py:101-104; optional gain (llama)."""
    x64 = np.asarray(x).astype(np.float64)
    scale = np.sqrt((x64 * x64).mean(axis=-1, keepdims=True) + eps)
    y = x64 / scale
    if weight is not None:
        y = y * np.asarray(weight).astype(np.float64)
    return y.astype(np.float32)


def position_table(max_len: int, d_model: int) -> np.ndarray:
    """Sinusoidal absolute positions: sin at even, cos at odd columns (model.py:107-114)."""
    pos = np.arange(max_len, dtype=np.float64)[:, None]
    i = np.arange(d_model // 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2.0 * i / d_model)
    table = np.zeros((max_len, d_model), dtype=np.float64)
    table[:, 0::2] = np.sin(ang)
    table[:, 1::2] = np.cos(ang)
    return table.astype(np.float32)


def rope_tables(max_len: int, head_dim: int, theta: float):
    """cos/sin [max_len, head_dim/2] as fp32 (the GPU reads these same fp32 tables)."""
    half = head_dim // 2
    inv = 1.0 / np.power(theta, np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_len, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x, positions, n_heads, head_dim, cos, sin) -> np.ndarray:
    """Rotate-half RoPE on [n, n_heads*head_dim] fp32 values, computed in fp64 -> fp32."""
    n = x.shape[0]
    half = head_dim // 2
    x64 = np.asarray(x, np.float64).reshape(n, n_heads, head_dim)
    c = cos[positions].astype(np.float64)[:, None, :]
    s = sin[positions].astype(np.float64)[:, None, :]
    x1, x2 = x64[..., :half], x64[..., half:]
    out = np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)
    return out.reshape(n, n_heads * head_dim).astype(np.float32)


def project_qkv_masked(x, wq, wk, wv, adapter: OracleAdapter | None = None, mask=None, bf16=False):
    """model.py:117-146: base projections, adapted = base + (x@down)@up, row SELECT by mask.

    mask True keeps the base row exactly; mask None applies the adapter to
    every row (standard LoRA); adapter None returns the base projections.
    With bf16=True the shrink output is rounded to bf16 and the delta is added
    inside the same (fp64 here, fp32 on GPU) accumulation as the base product.
    """
    x = np.asarray(x, np.float32)
    bases = {"q": wq, "k": wk, "v": wv}
    if adapter is not None and mask is not None:
        mask = np.asarray(mask, dtype=bool)
        if mask.shape != (len(x),):
            raise ValueError(f"mask shape {mask.shape} does not match {len(x)} rows")
    out = []
    for name in ("q", "k", "v"):
        w = bases[name]
        base64 = x.astype(np.float64) @ np.asarray(w).astype(np.float64, copy=False)
        base = base64.astype(np.float32)
        if adapter is None or name not in adapter.targets:
            out.append(base)
            continue
        if bf16:
            s = bf16_round(mm(x, adapter.down[name]))
            adapted = (base64 + s.astype(np.float64) @ adapter.up[name].astype(np.float64, copy=False)).astype(np.float32)
        else:
            adapted = base + mm(mm(x, adapter.down[name]), adapter.up[name])
        if mask is None:
            out.append(adapted)
        else:
            out.append(np.where(mask[:, None], base, adapted))
    return tuple(out)


def _adapted(x, w, name, adapter: OracleAdapter | None, mask, bf16: bool) -> np.ndarray:
    """x @ w with the adapter's masked delta on target `name` (model.py:141-145 at another projection), as
    fp64 (the caller rounds where the GPU rounds: the delta shares the base product's accumulator)."""
    out = np.asarray(x).astype(np.float64, copy=False) @ np.asarray(w).astype(np.float64, copy=False)
    if adapter is None or name not in adapter.targets:
        return out
    if bf16:
        s = bf16_round(mm(x, adapter.down[name]))
        delta = s.astype(np.float64) @ adapter.up[name].astype(np.float64, copy=False)
    else:  # reference rounding: base and delta are fp32 (mm) before the add
        out = out.astype(np.float32).astype(np.float64)
        delta = (mm(mm(x, adapter.down[name]), adapter.up[name])).astype(np.float64)
    if mask is None:
        return out + delta
    return np.where(np.asarray(mask, bool)[:, None], out, out + delta)


def paged_attention(q, kv, layer, block_ids, fresh_k, fresh_v, start_pos, n_heads, n_kv_heads=None):
    """model.py:149-187 generalised to GQA (query head h reads kv head h // (H/Hkv))."""
    q = np.asarray(q)
    n, dq = q.shape
    block_size = kv.shape[3]
    kvw = kv.shape[4]
    hkv = n_heads if n_kv_heads is None else n_kv_heads
    hd = dq // n_heads
    total = start_pos + n
    need = -(-total // block_size)
    if len(block_ids) < need:
        raise ValueError(f"block table has {len(block_ids)} blocks, need {need}")
    if start_pos > 0:
        ids = np.asarray(block_ids[:need], dtype=np.intp)
        gathered = kv[ids, layer]
        k_ctx = gathered[:, 0].reshape(-1, kvw)[:start_pos]
        v_ctx = gathered[:, 1].reshape(-1, kvw)[:start_pos]
        keys = np.concatenate([k_ctx, fresh_k], axis=0)
        vals = np.concatenate([v_ctx, fresh_v], axis=0)
    else:
        keys, vals = np.asarray(fresh_k), np.asarray(fresh_v)
    group = n_heads // hkv
    if group > 1:  # GQA (llama mode, no reference counterpart): the same math batched per kv head, no K/V repeat
        qg = q.astype(np.float64).reshape(n, hkv, group, hd).transpose(1, 2, 0, 3).reshape(hkv, group * n, hd)
        kg = np.asarray(keys, np.float64).reshape(total, hkv, hd).transpose(1, 2, 0)
        vg = np.asarray(vals, np.float64).reshape(total, hkv, hd).transpose(1, 0, 2)
        sc = (qg @ kg / np.sqrt(hd)).reshape(hkv, group, n, total)
        qpos = start_pos + np.arange(n)[:, None]
        sc = np.where(np.arange(total)[None, :] <= qpos, sc, -np.inf)
        sc -= sc.max(axis=-1, keepdims=True)
        w = np.exp(sc)
        w /= w.sum(axis=-1, keepdims=True)
        ctx = (w.reshape(hkv, group * n, total) @ vg).reshape(hkv, group, n, hd).transpose(2, 0, 1, 3)
        return ctx.reshape(n, dq).astype(np.float32)
    q64 = q.astype(np.float64).reshape(n, n_heads, hd)
    k64 = np.repeat(np.asarray(keys, np.float64).reshape(total, hkv, hd), group, axis=1)
    v64 = np.repeat(np.asarray(vals, np.float64).reshape(total, hkv, hd), group, axis=1)
    scores = np.einsum("nhd,thd->hnt", q64, k64) / np.sqrt(hd)
    key_pos = np.arange(total)[None, :]
    query_pos = start_pos + np.arange(n)[:, None]
    scores = np.where(key_pos <= query_pos, scores, -np.inf)
    scores -= scores.max(axis=-1, keepdims=True)
    w = np.exp(scores)
    w /= w.sum(axis=-1, keepdims=True)
    ctx = np.einsum("hnt,thd->nhd", w, v64)
    return ctx.reshape(n, dq).astype(np.float32)


def write_kv(kv, layer, block_ids, start_pos, k, v) -> None:
    """model.py:217-222: slot = block_ids[pos // B], row = pos % B."""
    block_size = kv.shape[3]
    pos = start_pos + np.arange(len(k))
    ids = np.asarray(block_ids, dtype=np.intp)[pos // block_size]
    kv[ids, layer, 0, pos % block_size] = k
    kv[ids, layer, 1, pos % block_size] = v


def greedy_next_token(logits) -> int:
    """Argmax, ties to the lowest id (model.py:190-195)."""
    logits = np.asarray(logits)
    if logits.ndim != 1:
        raise ValueError(f"expected a logits vector, got shape {logits.shape}")
    return int(np.argmax(logits))


def detect_invocation(prompt_tokens, invocation_tokens) -> int:
    """Last occurrence of the invocation sequence (engine.py:29-45)."""
    prompt = np.asarray(prompt_tokens)
    inv = np.asarray(invocation_tokens)
    m = len(inv)
    if m == 0:
        raise ValueError("invocation_tokens is empty")
    for start in range(len(prompt) - m, -1, -1):
        if np.array_equal(prompt[start:start + m], inv):
            return start
    raise ValueError("invocation sequence not found")


def activation_mask(start, end, inv_start) -> np.ndarray:
    """values = pos < effective inv_start (engine.py:64-79)."""
    return np.arange(start, end) < inv_start


@dataclass
class OracleSpan:
    """SeqInput (model.py:198-214)."""

    request_id: str
    tokens: np.ndarray
    start_pos: int
    block_ids: list
    adapter: OracleAdapter | None = None
    mask: np.ndarray | None = None


class OracleModel:
    """Model.forward_step over a numpy pool kv[NB, L, 2, B, kv_width] (model.py:225-272)."""

    def __init__(self, cfg: OracleConfig, weights: dict | None = None):
        self.cfg = cfg
        self.w = weights if weights is not None else oracle_weights(cfg)
        self.positions = position_table(cfg.max_seq_len, cfg.d_model) if cfg.arch == "ref" else None
        if cfg.arch == "llama":
            self.cos, self.sin = rope_tables(cfg.max_seq_len, cfg.head_dim, cfg.rope_theta)

    def to_f64(self):
        """Hold every GEMM weight as float64 (exact: the values are fp32/bf16) so repeated forwards skip the
        per-call up-cast of model.py:95-98. Same results; for large test geometries only."""
        for layer in self.w["layers"]:
            for k in list(layer):
                if not k.endswith("_norm"):
                    layer[k] = np.asarray(layer[k]).astype(np.float64)
        for k in ("embed", "unembed"):
            if self.w.get(k) is not None:
                self.w[k] = np.asarray(self.w[k]).astype(np.float64)
        return self

    def new_pool(self, total_blocks, block_size):
        c = self.cfg
        return np.zeros((total_blocks, c.n_layers, 2, block_size, c.kv_width), np.float32)

    def forward_step(self, seqs, kv, batch_head: bool = False) -> dict:
        """batch_head=True runs the lm_head once over every span's last row (the same per-row fp64 math as
        model.py:272; for large vocabularies in tests) instead of once per span."""
        if not batch_head:
            return {s.request_id: self.forward_one(s, kv) for s in seqs}
        hf = np.concatenate([self.last_hidden(s, kv) for s in seqs])
        logits = mm(hf, self._unembed())
        return {s.request_id: logits[i] for i, s in enumerate(seqs)}

    def _unembed(self):
        return self.w["unembed"] if self.w.get("unembed") is not None else self.w["embed"].T

    def forward_one(self, seq: OracleSpan, kv) -> np.ndarray:
        return mm(self.last_hidden(seq, kv), self._unembed())[0]

    def last_hidden(self, seq: OracleSpan, kv) -> np.ndarray:
        """Every layer of model.py:263-271 for one span (KV written into kv); the final-normed last row."""
        c = self.cfg
        bf = c.numerics == "bf16"
        rb = bf16_round if bf else (lambda a: np.asarray(a, np.float32))
        tokens = np.asarray(seq.tokens, dtype=np.int64)
        n = len(tokens)
        if n == 0:
            raise ValueError("empty span")
        if seq.start_pos + n > c.max_seq_len:
            raise ValueError("span exceeds max_seq_len")
        mask = None
        if seq.adapter is not None and seq.adapter.mode == MODE_ACTIVATED:
            if seq.mask is None:
                raise ValueError(f"activated adapter span for {seq.request_id} is missing its mask")
            mask = seq.mask
        positions = np.arange(seq.start_pos, seq.start_pos + n)
        if c.arch == "ref":
            x = self.w["embed"][tokens].astype(np.float32, copy=False) + self.positions[seq.start_pos:seq.start_pos + n]
        else:
            x = self.w["embed"][tokens].astype(np.float32)
        for li, L in enumerate(self.w["layers"]):
            h = rb(rmsnorm(x, L.get("attn_norm"), c.rms_eps))
            q, k, v = project_qkv_masked(h, L["wq"], L["wk"], L["wv"], seq.adapter, mask, bf16=bf)
            if c.arch == "llama":
                q = apply_rope(q, positions, c.n_heads, c.head_dim, self.cos, self.sin)
                k = apply_rope(k, positions, c.kv_heads, c.head_dim, self.cos, self.sin)
            q, k, v = rb(q), rb(k), rb(v)
            write_kv(kv, li, seq.block_ids, seq.start_pos, k, v)
            attn = rb(paged_attention(q, kv, li, seq.block_ids, k, v, seq.start_pos, c.n_heads, c.kv_heads))
            ad = seq.adapter
            o = _adapted(attn, L["wo"], "o", ad, mask, bf)
            x = (x.astype(np.float64) + o).astype(np.float32) if bf else x + o.astype(np.float32)
            h2 = rb(rmsnorm(x, L.get("mlp_norm"), c.rms_eps))
            if c.arch == "ref":
                a = rb(np.maximum(_adapted(h2, L["w_in"], "up", ad, mask, bf).astype(np.float32), 0.0))
                w_down = L["w_out"]
            else:
                g = _adapted(h2, L["w_gate"], "gate", ad, mask, bf).astype(np.float32).astype(np.float64)
                u = _adapted(h2, L["w_up"], "up", ad, mask, bf).astype(np.float32).astype(np.float64)
                a = rb((g / (1.0 + np.exp(-g)) * u).astype(np.float32))
                w_down = L["w_down"]
            dn = _adapted(a, w_down, "down", ad, mask, bf)
            x = (x.astype(np.float64) + dn).astype(np.float32) if bf else x + dn.astype(np.float32)
        return rb(rmsnorm(x[-1:], self.w.get("final_norm"), c.rms_eps))
