"""Decode-step host/device split on the GPU (C2 eval turn, 12 requests): per-phase medians over decode steps."""
import sys, time, statistics
import numpy as np, torch
sys.path.insert(0, '.')
exec(open("tools/ttft_breakdown.py").read().split("rows = []")[0])
dec = []
for i in range(6):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"d{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    for rid, prompt, adapter_id, gen, meta in sub:
        eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    eng.step()
    torch.cuda.synchronize()
    while True:
        tm.clear()
        t0 = time.perf_counter()
        more = eng.step()
        t1 = time.perf_counter()
        if not more:
            break
        if i >= 2:
            dec.append({"step": t1 - t0, **tm})
print(f"{len(dec)} decode steps")
for k in dec[0]:
    print(f"{k:20s} {1e3*statistics.median(r.get(k, 0) for r in dec):.3f} ms")
