"""Multi-turn pipelines that drive the engine (the measured workload).

Same turn algebra and token layout as aloraserve/bench.py (bench.py:1-21, 99-113,
245-306): base turn conv -> y tokens + EOT; eval turn conv + invocation -> r
tokens on adapter k; final turn conv + Σ(inv + eval output + EOT) through the
base model. The top 32 ids are reserved; EOT = V-1; adapter k owns the
invocation (V-32+3k, +1, +2). run_sync_pipeline submits each phase back to
back and drains the engine before the next phase (phase barriers).
"""

from dataclasses import dataclass

import numpy as np

from .engine import AdapterSpec, Engine, EngineConfig
from .model import ModelConfig
from .scheduler import SchedulerConfig
from .clock import VirtualClock, WallClock

RESERVED_TOKENS = 32
INVOCATION_LEN = 3


@dataclass(frozen=True)
class PipelineSpec:
    pipeline: str = "base_adapter"  # base_adapter | adapter_base | base_adapter_base | multi_adapter
    mode: str = "alora"  # alora | lora
    prompt_len: int = 64
    gen_len: int = 64
    adapter_gen_len: int = 16
    n_adapters: int = 1
    batch: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.pipeline not in ("base_adapter", "adapter_base", "base_adapter_base", "multi_adapter"):
            raise ValueError(f"unknown pipeline {self.pipeline!r}")
        if self.mode not in ("alora", "lora"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if min(self.prompt_len, self.gen_len, self.adapter_gen_len, self.n_adapters, self.batch) < 1:
            raise ValueError("pipeline dimensions must be >= 1")


def end_of_turn_token(vocab_size: int) -> int:
    return vocab_size - 1


def invocation_for(vocab_size: int, k: int) -> tuple:
    first = vocab_size - RESERVED_TOKENS + INVOCATION_LEN * k
    if first + INVOCATION_LEN >= vocab_size:
        raise ValueError(f"adapter index {k} does not fit in the reserved token range")
    return tuple(range(first, first + INVOCATION_LEN))


def random_conversation(rng: np.random.Generator, n: int, vocab_size: int) -> np.ndarray:
    return rng.integers(0, vocab_size - RESERVED_TOKENS, n, dtype=np.int64)


def pipeline_shape(spec: PipelineSpec):
    """(base turn first, has final turn, number of eval turns)."""
    return {"base_adapter": (True, False, 1), "adapter_base": (False, True, 1),
            "base_adapter_base": (True, True, 1), "multi_adapter": (True, True, spec.n_adapters)}[spec.pipeline]


def build_engine(spec: PipelineSpec, model: ModelConfig | None = None, pool_blocks: int = 512, block_size: int = 4,
                 token_budget: int = 64, virtual_clock: bool = True, rank: int = 8,
                 max_batch_requests: int | None = None, prefix_caching: bool = True, chunked_prefill: bool = True,
                 engine_model=None, pool_storage: str = "cuda", pipelined_decode: bool = False,
                 batch_invariant: bool = False) -> Engine:
    """One registered adapter per eval slot: adapter{k} with invocation_for(V, k) (bench.py:175-213)."""
    model = model or ModelConfig()
    _, _, n_eval = pipeline_shape(spec)
    adapters = tuple(AdapterSpec(adapter_id=f"adapter{k}", rank=rank, seed=spec.seed,
                                 invocation_tokens=invocation_for(model.vocab_size, k)) for k in range(n_eval))
    if max_batch_requests is None:
        max_batch_requests = max(8, 2 * spec.batch, n_eval * spec.batch + 2)
    cfg = EngineConfig(model=model,
                       scheduler=SchedulerConfig(token_budget=token_budget, max_batch_requests=max_batch_requests,
                                                 chunked_prefill=chunked_prefill),
                       pool_blocks=pool_blocks, block_size=block_size, adapters=adapters,
                       comparison_mode=spec.mode, prefix_caching=prefix_caching)
    return Engine(cfg, clock=VirtualClock() if virtual_clock else WallClock(), model=engine_model,
                  pool_storage=pool_storage, max_tokens=max(token_budget, max_batch_requests),
                  pipelined_decode=pipelined_decode, batch_invariant=batch_invariant)


def _rid(prefix, idx, stage):
    return f"{prefix}i{idx}-{stage}"


def run_phase(engine: Engine, submits) -> None:
    for rid, prompt, adapter_id, gen, meta in submits:
        engine.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    engine.run_until_idle()


def pipeline_phases(spec: PipelineSpec, engine: Engine, rid_prefix: str = "", instances=None):
    """Yield (stage, submits) per phase; each phase's prompts depend on the previous phase's outputs.

    `instances` (replicas.py) restricts the run to a subset of the spec's pipeline instances; the
    conversations are still drawn for all `spec.batch` instances, so instance i is the same on every
    replica count.
    """
    base_first, has_final, n_eval = pipeline_shape(spec)
    V = engine.config.model.vocab_size
    eot = end_of_turn_token(V)
    rng = np.random.default_rng(spec.seed)
    convs = [random_conversation(rng, spec.prompt_len, V) for _ in range(spec.batch)]
    mine = list(range(spec.batch)) if instances is None else [int(i) for i in instances]
    meta = lambda stage, i: {"pipeline": spec.pipeline, "mode": spec.mode, "stage": stage, "instance": i}
    inv = {k: np.asarray(engine.adapters[f"adapter{k}"].invocation_tokens, dtype=np.int64) for k in range(n_eval)}
    if base_first:
        yield "base", [(_rid(rid_prefix, i, "base"), convs[i], None, spec.gen_len, meta("base", i))
                       for i in mine]
        for i in mine:
            gen = engine.finished[_rid(rid_prefix, i, "base")].generated
            convs[i] = np.concatenate([convs[i], np.asarray(gen, dtype=np.int64), [eot]])
    yield "eval", [(_rid(rid_prefix, i, f"eval{k}"), np.concatenate([convs[i], inv[k]]), f"adapter{k}",
                    spec.adapter_gen_len, meta("eval", i)) for i in mine for k in range(n_eval)]
    if has_final:
        finals = []
        for i in mine:
            parts = [convs[i]]
            for k in range(n_eval):
                out = np.asarray(engine.finished[_rid(rid_prefix, i, f"eval{k}")].generated, dtype=np.int64)
                parts.append(np.concatenate([inv[k], out, [eot]]))
            finals.append((_rid(rid_prefix, i, "final"), np.concatenate(parts), None, spec.gen_len, meta("final", i)))
        yield "final", finals


def run_sync_pipeline(spec: PipelineSpec, engine: Engine) -> list:
    """Run all phases with barriers; returns the engine's metrics rows (bench.py:264-306)."""
    for _, submits in pipeline_phases(spec, engine):
        run_phase(engine, submits)
    return list(engine.metrics)
