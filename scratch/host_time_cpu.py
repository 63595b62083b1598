"""Wall time of the eval turn's host path (no profiler), stub model, split by phase."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P
exec(open("scratch/host_prof_cpu.py").read().split("eng = P.Engine")[0])
eng = P.Engine(cfg, clock=P.WallClock(), model=Stub(), pool_storage="meta")
tm = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); tm[name] = tm.get(name, 0) + time.perf_counter() - t; return r
    setattr(obj, name, w)
for n in ("find_cached_prefix", "allocate", "set_fill", "commit_and_free"):
    wrap(eng.pool, n)
wrap(eng.scheduler, "schedule_step"); wrap(eng, "_seq_inputs"); wrap(eng.scheduler, "_prehash")
for i in range(6):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"w{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    tm.clear()
    t0 = time.perf_counter()
    for rid, prompt, adapter_id, gen, meta in sub:
        eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    t1 = time.perf_counter()
    eng.step()
    t2 = time.perf_counter()
    print(f"submit {1e3*(t1-t0):.3f} ms  first step {1e3*(t2-t1):.3f} ms", {k: round(v*1e3, 3) for k, v in tm.items()})
    eng.run_until_idle()

import cProfile, pstats
sp = P.PipelineSpec(**{**spec.__dict__, "seed": 99})
ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix="prof-")
st, sub = next(ph); P.pipeline.run_phase(eng, sub)
st, sub = next(ph)
for rid, prompt, adapter_id, gen, meta in sub:
    eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
pr = cProfile.Profile(); pr.enable()
eng.scheduler.schedule_step(0.0)
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
