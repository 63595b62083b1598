"""Eval-turn TTFT breakdown on the GPU: host phases of the first step vs the forward (C2 geometry)."""
import sys, time, statistics
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P
C2 = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
          vocab_size=128256, max_seq_len=4096, seed=0)
mcfg = P.ModelConfig(**C2, dtype="bf16")
spec = P.PipelineSpec(pipeline="multi_adapter", mode="alora", prompt_len=1792, gen_len=256, adapter_gen_len=16,
                      n_adapters=3, batch=4)
cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=64),
                     pool_blocks=4096, block_size=16,
                     adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=32, seed=k,
                                                  invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                    for k in range(3)), comparison_mode="alora")
model = P.Model(mcfg, init="device", max_tokens=8192, max_seqs=64)
eng = P.Engine(cfg, clock=P.WallClock(), model=model)
tm = {}
def wrap(obj, name, key=None):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); tm[key or name] = tm.get(key or name, 0) + time.perf_counter() - t; return r
    setattr(obj, name, w)
wrap(eng.scheduler, "schedule_step"); wrap(eng, "_seq_inputs"); wrap(model, "pack"); wrap(model, "stage")
wrap(model, "launch"); wrap(model, "run_packed"); wrap(eng.pool, "find_cached_prefix"); wrap(eng.scheduler, "_prehash")
import paper_2512_17910_b200.scheduler as SCH
_hr = SCH.hash_requests
def _hr_w(*a, **k):
    t = time.perf_counter(); r = _hr(*a, **k); tm["hash_requests"] = tm.get("hash_requests", 0) + time.perf_counter() - t; return r
SCH.hash_requests = _hr_w
import gc, os
from paper_2512_17910_b200 import _native as _N
_fn = _N.lib.alora_hash_requests
class _W:
    def __call__(self, *a):
        t = time.perf_counter(); r = _fn(*a); tm["ctypes_hash"] = tm.get("ctypes_hash", 0) + time.perf_counter() - t; return r
_N.lib.alora_hash_requests = _W()
_fl = _N.lib.alora_pool_lookup
class _W2:
    def __call__(self, *a):
        t = time.perf_counter(); r = _fl(*a); tm["ctypes_lookup"] = tm.get("ctypes_lookup", 0) + time.perf_counter() - t; return r
_N.lib.alora_pool_lookup = _W2()
if os.environ.get("GC_MODE") == "off":
    gc.disable()
elif os.environ.get("GC_MODE") == "freeze":
    gc.collect(); gc.freeze()
rows = []
for i in range(8):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"w{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    torch.cuda.synchronize()
    tm.clear()
    t0 = time.perf_counter()
    for rid, prompt, adapter_id, gen, meta in sub:
        eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    t1 = time.perf_counter()
    eng.step()
    t2 = time.perf_counter()
    r = {"submit": t1 - t0, "step": t2 - t1, **tm}
    ttft = max(m.ttft_s for m in eng.metrics[-len(sub):]) if False else None
    eng.run_until_idle()
    if i >= 2:
        rows.append(r)
for k in rows[0]:
    print(f"{k:20s} {1e3*statistics.median(r[k] for r in rows):.3f} ms")
