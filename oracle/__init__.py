"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/hashlib, the reference algorithm of the aLoRA
hot path (/root/reference/pkg/src/aloraserve/model.py, kv_cache.py,
adapters.py, engine.py). It is the checker the GPU path is compared against.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import it. The product package (paper_2512_17910_b200) never does:
its compute runs through libalora_sm100a.so and fails loudly without it.

Parity pinning: the ref-architecture functions are pinned bit-for-bit against
golden vectors produced by importing the reference in the build container
(oracle/gen_golden.py -> tests/golden/). The Llama-architecture deltas
(RoPE, GQA, SwiGLU, weighted RMSNorm, tied lm_head) have no counterpart in
the reference and are "parity unpinned" beyond the shared kernels they reuse.
"""

from .model_oracle import *  # noqa: F401,F403
from .kv_oracle import *  # noqa: F401,F403
