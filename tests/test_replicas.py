"""Request-parallel replicas (replicas.py) on CPU: world_size-2 gloo processes, one engine each.

Every replica runs its share of a multi_adapter pipeline (instance i on replica i mod 2) through
the drop-in Engine (driven by the CPU oracle model, host pool, virtual clock) and the rows are
gathered over gloo. Instance affinity must preserve cross-model prefix reuse: every request's
generated ids and hit/computed token counts equal those of the single-engine run, and the eval
turns hit the base-aligned law ((x+y-1)//B)*B.
"""

import os
import socket

import pytest

import oracle as O
import paper_2512_17910_b200 as P

DIMS = dict(n_layers=2, n_heads=4, head_dim=16, d_model=64, vocab_size=128, seed=0)
SPEC = dict(pipeline="multi_adapter", mode="alora", prompt_len=37, gen_len=8, adapter_gen_len=4, n_adapters=2,
            batch=5, seed=11)
B = 8


def _engine():
    model = O.OracleModel(O.OracleConfig(**DIMS))
    return P.build_engine(P.PipelineSpec(**SPEC), model=P.ModelConfig(**DIMS), pool_blocks=512, block_size=B,
                          token_budget=256, engine_model=model, pool_storage="numpy")


def _summary(rows, engine_finished=None):
    return {r.request_id: (r.hit_tokens, r.computed_tokens, r.stage) for r in rows}


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = _engine()
        rows = P.run_replica_pipeline(P.PipelineSpec(**SPEC), eng, rank, world)
        ids = {rid: list(map(int, req.generated)) for rid, req in eng.finished.items()}
        merged = P.gather_replica_rows(rows)
        all_ids = [None] * world
        dist.all_gather_object(all_ids, ids)
        if rank == 0:
            q.put((_summary(merged), {k: v for d in all_ids for k, v in d.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_replica_instances_affinity():
    assert P.replica_instances(5, 2, 0) == [0, 2, 4]
    assert P.replica_instances(5, 2, 1) == [1, 3]
    assert sorted(sum((P.replica_instances(7, 3, r) for r in range(3)), [])) == list(range(7))
    with pytest.raises(ValueError):
        P.replica_instances(4, 2, 2)


@pytest.mark.timeout(300)
def test_two_replicas_gloo_match_single_engine_and_keep_reuse():
    import torch.multiprocessing as mp

    single = _engine()
    rows = P.run_sync_pipeline(P.PipelineSpec(**SPEC), single)
    want = _summary(rows)
    want_ids = {rid: list(map(int, r.generated)) for rid, r in single.finished.items()}

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    got, got_ids = q.get()
    assert got == want
    assert got_ids == want_ids
    x, y = SPEC["prompt_len"], SPEC["gen_len"]
    for rid, (hit, comp, stage) in got.items():
        if stage == "eval":
            assert hit == ((x + y - 1) // B) * B, rid  # the adapter turn reuses the base turn's blocks


def test_bench_gpus_flag_spawns_ranks():
    """bench.py --gpus 2 run directly (no torchrun) re-launches itself with one process per rank; on CPU the
    --probe-ranks plumbing check inits gloo and rank 0 reports n_gpus 2 with the instance-affinity split."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--probe-ranks"],
                         capture_output=True, text=True, timeout=240, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["instances_per_rank"] == [list(range(0, 16, 2)), list(range(1, 16, 2))]
    assert line["eval_requests_total"] == 128


def test_bench_c5_ranks_are_one_tensor_parallel_model():
    """--config c5: the ranks are the shards of one TP model, so every rank runs every pipeline instance (no
    instance split) and the requests are counted once."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--probe-ranks",
                          "--config", "c5"], capture_output=True, text=True, timeout=240, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["instances_per_rank"] == [[0, 1], [0, 1]]
    assert line["eval_requests_total"] == 8
    assert line["config"]["parallelism"].startswith("TP=2")
