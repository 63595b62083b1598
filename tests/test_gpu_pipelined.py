"""Pipelined decode (Engine(pipelined_decode=True)): a pure-decode step is launched before the previous
step's ids are read back, its input tokens resolved on the device from the previous launch's ids.

The run must match the synchronous engine: generated ids, cache hits, the scheduled spans of every step
and the pool's digests, over multi-turn pipelines (base and aLoRA turns, decode steps that cross block
boundaries, requests finishing at different steps). Only the free-block count may lag by a step."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")

LLAMA = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512,
             vocab_size=384, max_seq_len=2048, seed=3, dtype="bf16")


def _run(pipelined: bool, pipeline: str, gen: int):
    spec = P.PipelineSpec(pipeline=pipeline, mode="alora", prompt_len=90, gen_len=gen, adapter_gen_len=gen + 3,
                          n_adapters=2, batch=3, seed=7)
    eng = P.build_engine(spec, model=P.ModelConfig(**LLAMA), pool_blocks=256, block_size=16, token_budget=256,
                         pipelined_decode=pipelined)
    rows = P.run_sync_pipeline(spec, eng)
    torch.cuda.synchronize()
    gen_ids = {rid: list(r.generated) for rid, r in eng.finished.items()}
    hits = {rid: (r.hit_tokens, r.computed_tokens) for rid, r in eng.finished.items()}
    digests = [row["digest"] for row in eng.pool.dump_state()]
    return gen_ids, hits, eng.trace, digests, len(rows)


@pytest.mark.parametrize("pipeline,gen", [("multi_adapter", 21), ("base_adapter_base", 9)])
def test_pipelined_decode_matches_synchronous(pipeline, gen):
    a = _run(False, pipeline, gen)
    b = _run(True, pipeline, gen)
    assert a[0] == b[0]  # generated ids
    assert a[1] == b[1]  # hits / computed tokens
    # step trace: identical schedules; only pool_free may lag (a pipelined step retires its finished requests
    # when its ids are read back, one step later)
    strip = lambda tr: [{k: v for k, v in row.items() if k != "pool_free"} for row in tr]
    assert strip(a[2]) == strip(b[2])
    assert all(y["pool_free"] <= x["pool_free"] for x, y in zip(a[2], b[2]))
    assert a[3] == b[3]  # pool digests (commit hashes the generated tokens)
    assert a[4] == b[4]
    assert all(t >= 0 for ids in b[0].values() for t in ids)  # no placeholder left behind
