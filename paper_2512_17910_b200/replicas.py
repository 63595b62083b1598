"""Request-parallel replicas (8B + 8 adapters, replicas at 1/2/4/8 B200).

A model that fits one GPU is served by N independent engines, one process per GPU, each with its
own BlockPool. Cross-model prefix reuse only hits inside one pool, so every turn of a pipeline
instance (its base turn, its adapter turns, its final turn) must land on the same replica: the
affinity key is the instance index, and instance i is served by replica i mod N. There is no
data-path collective; the only communication is the metrics gather (and the max/sum of the bench
timers), which torch.distributed does over gloo on CPU or NCCL on GPUs.
"""

from .pipeline import PipelineSpec, pipeline_phases, run_phase

__all__ = ["replica_instances", "run_replica_pipeline", "gather_replica_rows"]


def replica_instances(batch: int, world: int, rank: int) -> list:
    """Pipeline instances served by replica `rank` of `world` (affinity: instance index mod world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad replica rank {rank} of {world}")
    return [i for i in range(batch) if i % world == rank]


def run_replica_pipeline(spec: PipelineSpec, engine, rank: int, world: int, rid_prefix: str = "") -> list:
    """This replica's share of `spec` (all phases, with barriers); returns its engine's metrics rows."""
    mine = replica_instances(spec.batch, world, rank)
    if mine:
        for _, submits in pipeline_phases(spec, engine, rid_prefix, instances=mine):
            run_phase(engine, submits)
    return list(engine.metrics)


def gather_replica_rows(rows: list, group=None) -> list:
    """All replicas' metrics rows (every rank gets the merged list, ordered by request id)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, rows, group=group)
    merged = [r for part in out for r in part]
    return sorted(merged, key=lambda r: r.request_id)
