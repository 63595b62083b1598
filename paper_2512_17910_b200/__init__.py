"""B200-native drop-in for the aLoRA hot path of aloraserve (arXiv 2512.17910).

Same public names as aloraserve/__init__.py:13-72 for the path: the model
(Model.forward_step, project_qkv_masked, paged_attention, SeqInput,
greedy_next_token), adapter registration, the paged BlockPool with its
base-aligned block-hash chain, and the engine/scheduler that call them.
Compute runs in libalora_sm100a.so (hand-written sm_100a CUDA); importing
this package without the library raises — there is no CPU fallback.
"""

from . import _native
from .adapters import MODE_ACTIVATED, MODE_STANDARD, LoraAdapter, adapter_from_dict, generate_adapter, load_adapter_file
from .clock import VirtualClock, WallClock
from .engine import (ActivationMask, AdapterSpec, Engine, EngineConfig, InvocationNotFoundError,
                     build_activation_mask, detect_invocation, load_engine_config)
from .kv_cache import (Block, BlockPool, BlockTable, KVEntry, PoolExhaustedError, compute_block_keys, hash_block,
                       hash_chain)
from .metrics import RequestMetrics, finalize_request, render_csv
from .model import (BaseWeights, LayerWeights, Model, ModelConfig, SeqInput, generate_weights, greedy_next_token,
                    paged_attention, project_qkv_masked, write_kv)
from .pipeline import (PipelineSpec, build_engine, end_of_turn_token, invocation_for, random_conversation,
                       run_sync_pipeline)
from .scheduler import Request, RequestState, ScheduledSpan, Scheduler, SchedulerConfig
from .replicas import gather_replica_rows, replica_instances, run_replica_pipeline
from .tp import ThreadGroup, TorchDistGroup, TPModel, shard_adapter, shard_config, shard_weights

__version__ = "0.1.0"
native_version = _native.version
