"""Deterministic model weights (host numpy) for both architectures.

arch "ref" reproduces aloraserve.model.generate_weights byte for byte
(reference model.py:62-92): every tensor is uniform(-0.1, 0.1) from a Philox
stream keyed by blake2b-128("weights:{seed}:{name}"), stored [in, out].
arch "llama" uses the same keyed streams with fan-in scaled ranges, weighted
RMSNorm gains and an lm_head tied to the embedding (no reference
counterpart).
"""

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass
class LayerWeights:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w_in: np.ndarray  # ref: [d, 4d] ReLU input; llama: gate [d, F]
    w_out: np.ndarray  # [F, d]
    w_up: np.ndarray | None = None  # llama: up [d, F]
    attn_norm: np.ndarray | None = None
    mlp_norm: np.ndarray | None = None


@dataclass
class BaseWeights:
    embed: np.ndarray
    layers: list
    unembed: np.ndarray | None  # None = tied to embed
    final_norm: np.ndarray | None = None


def _uniform(seed: int, name: str, shape, bound: float) -> np.ndarray:
    key = int.from_bytes(hashlib.blake2b(f"weights:{seed}:{name}".encode(), digest_size=16).digest(), "little")
    return np.random.Generator(np.random.Philox(key=key)).uniform(-bound, bound, shape).astype(np.float32)


def generate_weights(config) -> BaseWeights:
    c = config
    d = c.d_model
    layers = []
    if c.arch == "ref":
        for li in range(c.n_layers):
            layers.append(LayerWeights(
                wq=_uniform(c.seed, f"l{li}.wq", (d, d), 0.1), wk=_uniform(c.seed, f"l{li}.wk", (d, d), 0.1),
                wv=_uniform(c.seed, f"l{li}.wv", (d, d), 0.1), wo=_uniform(c.seed, f"l{li}.wo", (d, d), 0.1),
                w_in=_uniform(c.seed, f"l{li}.w_in", (d, c.ffn), 0.1),
                w_out=_uniform(c.seed, f"l{li}.w_out", (c.ffn, d), 0.1)))
        return BaseWeights(embed=_uniform(c.seed, "embed", (c.vocab_size, d), 0.1), layers=layers,
                           unembed=_uniform(c.seed, "unembed", (d, c.vocab_size), 0.1))
    b_d, b_q, b_f = np.sqrt(3.0 / d), np.sqrt(3.0 / c.q_width), np.sqrt(3.0 / c.ffn)
    for li in range(c.n_layers):
        layers.append(LayerWeights(
            attn_norm=1.0 + _uniform(c.seed, f"l{li}.attn_norm", (d,), 0.1),
            wq=_uniform(c.seed, f"l{li}.wq", (d, c.q_width), b_d),
            wk=_uniform(c.seed, f"l{li}.wk", (d, c.kv_width), b_d),
            wv=_uniform(c.seed, f"l{li}.wv", (d, c.kv_width), b_d),
            wo=_uniform(c.seed, f"l{li}.wo", (c.q_width, d), b_q),
            mlp_norm=1.0 + _uniform(c.seed, f"l{li}.mlp_norm", (d,), 0.1),
            w_in=_uniform(c.seed, f"l{li}.w_gate", (d, c.ffn), b_d),
            w_up=_uniform(c.seed, f"l{li}.w_up", (d, c.ffn), b_d),
            w_out=_uniform(c.seed, f"l{li}.w_down", (c.ffn, d), b_f)))
    return BaseWeights(embed=_uniform(c.seed, "embed", (c.vocab_size, d), b_d), layers=layers, unembed=None,
                       final_norm=1.0 + _uniform(c.seed, "final_norm", (d,), 0.1))


def position_table(max_len: int, d_model: int) -> np.ndarray:
    """Sinusoidal table, sin at even / cos at odd columns, fp64 -> fp32 (reference model.py:107-114)."""
    pos = np.arange(max_len, dtype=np.float64)[:, None]
    i = np.arange(d_model // 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2.0 * i / d_model)
    t = np.empty((max_len, d_model), dtype=np.float64)
    t[:, 0::2] = np.sin(ang)
    t[:, 1::2] = np.cos(ang)
    return t.astype(np.float32)


def rope_tables(max_len: int, head_dim: int, theta: float):
    half = head_dim // 2
    inv = 1.0 / np.power(theta, np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_len, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
