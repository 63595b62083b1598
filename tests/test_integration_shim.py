"""INTEGRATION.md §1 run for real: the reference's own Engine (aloraserve, imported read-only from
/root/reference in the build container) with the maintainer shim's BlockPool rebinding applied, on the
reference's pipelines; tokens, hits, first block tables, virtual-clock metrics CSV, step trace and pool dump
must equal the golden fixtures the stock reference produced (oracle/gen_golden.py).

The shim's Model rebinding needs a GPU, and the reference cannot travel to the GPU box, so this host-side
test exercises the pool half of the drop-in (the native block manager behind aloraserve's scheduler and
engine); the model half is pinned by tests/test_gpu_fp32.py against the same fixtures. Skipped when the
reference is absent (the GPU box)."""

import json
import os
import sys

import pytest

REF_SRC = os.environ.get("ALORA_REFERENCE_SRC", "/root/reference/pkg/src")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "aloraserve")),
                                reason="reference package not present (GPU box)")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import aloraserve
    from aloraserve import bench as ref_bench
    from aloraserve import engine as ref_engine
    from aloraserve.metrics import render_csv
    yield aloraserve, ref_bench, ref_engine, render_csv
    sys.path.remove(REF_SRC)


def _shim_pool_class():
    """The INTEGRATION.md §1 BlockPool shim (host storage: no GPU here)."""
    import paper_2512_17910_b200 as b200

    class BlockPool(b200.BlockPool):
        def __init__(self, total_blocks, block_size, n_layers, d_model):
            super().__init__(total_blocks, block_size, n_layers, d_model, dtype="fp32", storage="numpy")

    return BlockPool


@pytest.mark.parametrize("name", ["d64_multi_alora", "d64_adapter_base_alora", "d64_ba_lora", "d64_bab_alora_b8"])
def test_reference_engine_with_shim_pool_reproduces_goldens(ref, name):
    aloraserve, ref_bench, ref_engine, render_csv = ref
    with open(os.path.join(GOLDEN, "pipelines.json")) as f:
        g = json.load(f)[name]
    spec = aloraserve.PipelineSpec(**g["spec"])
    _, _, n_eval = ref_bench._pipeline_shape(spec)
    mcfg = aloraserve.ModelConfig(**g["model"])
    adapters = tuple(aloraserve.AdapterSpec(adapter_id=f"adapter{k}", rank=8, seed=spec.seed,
                                            invocation_tokens=aloraserve.invocation_for(mcfg.vocab_size, k))
                     for k in range(n_eval))
    e = g["engine"]
    cfg = aloraserve.EngineConfig(
        model=mcfg,
        scheduler=aloraserve.SchedulerConfig(token_budget=e["token_budget"],
                                             max_batch_requests=max(8, 2 * spec.batch, n_eval * spec.batch + 2)),
        pool_blocks=e["pool_blocks"], block_size=e["block_size"], adapters=adapters, comparison_mode=spec.mode)
    stock = ref_engine.BlockPool
    ref_engine.BlockPool = _shim_pool_class()  # the shim: aloraserve.engine binds BlockPool at import
    try:
        eng = aloraserve.Engine(cfg, clock=aloraserve.VirtualClock())
        import paper_2512_17910_b200 as b200
        assert isinstance(eng.pool, b200.BlockPool)  # the native block manager serves aloraserve's scheduler
        first_tables = {}
        orig = eng.scheduler._cache_lookup

        def spy(req):
            orig(req)
            bt = eng.pool.block_table(req.request_id)
            first_tables[req.request_id] = {"block_ids": list(bt.block_ids), "reused": list(bt.reused)}
        eng.scheduler._cache_lookup = spy
        res = aloraserve.run_sync_pipeline(spec, engine=eng)
    finally:
        ref_engine.BlockPool = stock
    for rid, r in eng.finished.items():
        want = g["requests"][rid]
        assert list(map(int, r.generated)) == want["generated"], rid
        assert (r.hit_tokens, r.computed_tokens) == (want["hit_tokens"], want["computed_tokens"]), rid
    assert first_tables == g["first_tables"]
    assert render_csv(res.rows) == g["metrics_csv"]
    assert eng.trace == g["trace"]
    assert eng.pool.dump_state() == g["pool_dump"]
