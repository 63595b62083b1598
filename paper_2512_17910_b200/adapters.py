"""Adapter registry data: LoRA factors for q/k/v and their activation mode.

Mirrors aloraserve/adapters.py (reference adapters.py:1-133):
  * MODE_ACTIVATED / MODE_STANDARD and the validation rules (adapters.py:36-66)
  * generate_adapter: uniform(-0.1, 0.1) factors from a Philox stream keyed by
    blake2b-128("adapter:{id}:{seed}:{t}:down|up") (adapters.py:29-33, 68-101),
    byte-identical to the reference for the reference geometry
  * adapter_from_dict / load_adapter_file: the JSON schema (adapters.py:104-133)

Extensions: `kv_width` (default d_model) sizes the k/v up-projections for GQA
models, where the k/v projections are narrower than d_model. Targets may also
name the O-projection and the MLP ("o", "gate", "up", "down"; EXTENDED_TARGETS),
which the reference rejects (adapters.py:26, 61-63): the same masked
base + (x @ down) @ up delta, applied by the bf16 tier inside those GEMMs.
`q_width` / `ffn_width` size their factors (defaults d_model / 4 * d_model).
Factors stay host numpy arrays here; Model uploads them into its device
adapter bank the first time a span uses them.
"""

import hashlib
import json
from dataclasses import dataclass, field

import numpy as np

MODE_ACTIVATED = "activated"
MODE_STANDARD = "standard"
PROJECTIONS = ("q", "k", "v")
EXTENDED_TARGETS = PROJECTIONS + ("o", "gate", "up", "down")
TARGET_BITS = {t: i for i, t in enumerate(EXTENDED_TARGETS)}  # slot_targets bit of each target (alora_sm100a.h)


def _philox_for(tag: str) -> np.random.Generator:
    digest = hashlib.blake2b(tag.encode(), digest_size=16).digest()
    return np.random.Generator(np.random.Philox(key=int.from_bytes(digest, "little")))


@dataclass(frozen=True)
class LoraAdapter:
    """down[t]: (d_model, rank); up[t]: (rank, out_width(t)); adapted = x@W + (x@down)@up."""

    adapter_id: str
    rank: int
    mode: str = MODE_ACTIVATED
    targets: tuple = PROJECTIONS
    invocation_tokens: tuple | None = None
    down: dict = field(default_factory=dict, repr=False)
    up: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        if self.mode not in (MODE_ACTIVATED, MODE_STANDARD):
            raise ValueError(f"unknown adapter mode {self.mode!r}")
        if self.rank < 1:
            raise ValueError("rank must be >= 1")
        if not self.targets or any(t not in EXTENDED_TARGETS for t in self.targets):
            raise ValueError(f"targets must be a non-empty subset of {EXTENDED_TARGETS}, got {self.targets}")
        if self.mode == MODE_ACTIVATED and not self.invocation_tokens:
            raise ValueError("activated adapter needs a non-empty invocation_tokens")


def generate_adapter(adapter_id: str, d_model: int, rank: int, seed: int = 0, targets=PROJECTIONS,
                     invocation_tokens=None, mode: str = MODE_ACTIVATED, kv_width: int | None = None,
                     q_width: int | None = None, ffn_width: int | None = None) -> LoraAdapter:
    if rank > d_model:
        raise ValueError(f"rank {rank} exceeds d_model {d_model}")
    shapes = target_shapes(d_model, q_width, kv_width, ffn_width)
    down, up = {}, {}
    for t in targets:
        if t not in shapes:
            raise ValueError(f"unknown target {t!r}")
        n_in, n_out = shapes[t]
        down[t] = _philox_for(f"adapter:{adapter_id}:{seed}:{t}:down").uniform(-0.1, 0.1, (n_in, rank)).astype(np.float32)
        up[t] = _philox_for(f"adapter:{adapter_id}:{seed}:{t}:up").uniform(-0.1, 0.1, (rank, n_out)).astype(np.float32)
    inv = None if invocation_tokens is None else tuple(int(t) for t in invocation_tokens)
    return LoraAdapter(adapter_id=adapter_id, rank=rank, mode=mode, targets=tuple(targets),
                       invocation_tokens=inv, down=down, up=up)


def target_shapes(d_model: int, q_width: int | None = None, kv_width: int | None = None,
                  ffn_width: int | None = None) -> dict:
    """(in, out) width of each target's projection: q/k/v d -> q|kv width, o q -> d, gate/up d -> F, down F -> d."""
    q, kv, f = q_width or d_model, kv_width or d_model, ffn_width or 4 * d_model
    return {"q": (d_model, q), "k": (d_model, kv), "v": (d_model, kv), "o": (q, d_model), "gate": (d_model, f),
            "up": (d_model, f), "down": (f, d_model)}


def adapter_from_dict(spec: dict, d_model: int, mode: str | None = None, kv_width: int | None = None,
                      q_width: int | None = None, ffn_width: int | None = None) -> LoraAdapter:
    """{"adapter_id", "rank", "seed", "targets"?, "invocation_tokens"?}; no invocation => standard."""
    for key in ("adapter_id", "rank", "seed"):
        if key not in spec:
            raise ValueError(f"adapter definition missing {key!r}")
    inv = spec.get("invocation_tokens")
    if mode is None:
        mode = MODE_ACTIVATED if inv else MODE_STANDARD
    return generate_adapter(spec["adapter_id"], d_model, int(spec["rank"]), seed=int(spec["seed"]),
                            targets=tuple(spec.get("targets", PROJECTIONS)), invocation_tokens=inv, mode=mode,
                            kv_width=kv_width, q_width=q_width, ffn_width=ffn_width)


def load_adapter_file(path, d_model: int, mode: str | None = None, kv_width: int | None = None,
                      q_width: int | None = None, ffn_width: int | None = None) -> LoraAdapter:
    with open(path) as f:
        return adapter_from_dict(json.load(f), d_model, mode=mode, kv_width=kv_width, q_width=q_width,
                                 ffn_width=ffn_width)
