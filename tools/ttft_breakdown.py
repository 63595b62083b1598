"""Eval-turn TTFT breakdown on the GPU: host phases of the first step vs the forward.

usage: python tools/ttft_breakdown.py [c2|c3]   (C2: Llama-3.2-1B, 4 x 3 adapters x 2k; C3: Llama-3-8B, 8 x 8 x 8k)
"""
import sys, time, statistics
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P
geom = sys.argv[1] if len(sys.argv) > 1 else "c2"
if geom == "c3":
    dims = dict(arch="llama", n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, ffn_dim=14336,
                vocab_size=128256, max_seq_len=8192 + 80, seed=0)
    n_ad, batch, x, pool_blocks, max_seqs, iters = 8, 8, 7932, (8 * 9 + 8) * 513, 72, 5
else:
    dims = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
                vocab_size=128256, max_seq_len=4096, seed=0)
    n_ad, batch, x, pool_blocks, max_seqs, iters = 3, 4, 1792, 4096, 64, 8
mcfg = P.ModelConfig(**dims, dtype="bf16")
spec = P.PipelineSpec(pipeline="multi_adapter", mode="alora", prompt_len=x, gen_len=256, adapter_gen_len=16,
                      n_adapters=n_ad, batch=batch)
cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=max_seqs),
                     pool_blocks=pool_blocks, block_size=16,
                     adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=32, seed=k,
                                                  invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                    for k in range(n_ad)), comparison_mode="alora")
model = P.Model(mcfg, init="device", max_tokens=8192, max_seqs=max_seqs)
eng = P.Engine(cfg, clock=P.WallClock(), model=model)
tm = {}
def wrap(obj, name, key=None):
    if not hasattr(obj, name):
        return
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); tm[key or name] = tm.get(key or name, 0) + time.perf_counter() - t; return r
    setattr(obj, name, w)
wrap(eng.scheduler, "schedule_step"); wrap(eng, "_seq_inputs"); wrap(model, "pack"); wrap(model, "stage")
wrap(model, "launch"); wrap(model, "run_packed"); wrap(eng.pool, "find_cached_prefix"); wrap(eng.scheduler, "_prehash")
import paper_2512_17910_b200.scheduler as SCH
_hr = getattr(SCH, "hash_requests", None)
def _hr_w(*a, **k):
    t = time.perf_counter(); r = _hr(*a, **k); tm["hash_requests"] = tm.get("hash_requests", 0) + time.perf_counter() - t; return r
if _hr is not None:
    SCH.hash_requests = _hr_w
import gc, os
from paper_2512_17910_b200 import _native as _N
def _wrap_lib(name):
    fn = getattr(_N.lib, name, None)
    if fn is None:
        return
    def w(*a):
        t = time.perf_counter(); r = fn(*a); tm[name] = tm.get(name, 0) + time.perf_counter() - t; return r
    setattr(_N.lib, name, w)
for _name in ("alora_hash_requests", "alora_pool_lookup", "alora_sched_submit", "alora_sched_step",
              "alora_sched_info", "alora_sched_step_done", "alora_sched_blocks", "alora_model_forward",
              "alora_model_forward_graph"):
    _wrap_lib(_name)
if os.environ.get("GC_MODE") == "off":
    gc.disable()
elif os.environ.get("GC_MODE") == "freeze":
    gc.collect(); gc.freeze()
rows = []
for i in range(iters):
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
