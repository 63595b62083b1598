"""cProfile of one eval-turn schedule_step + pack on the GPU box (relative shares only)."""
import sys, time, cProfile, pstats
sys.path.insert(0, '.')
exec(open("scratch/ttft_breakdown.py").read().split("import paper_2512_17910_b200.scheduler as SCH")[0])
for i in range(4):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"p{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    pr = cProfile.Profile()
    if i == 3: pr.enable()
    for rid, prompt, adapter_id, gen, meta in sub:
        eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    eng.step()
    if i == 3:
        pr.disable()
        st_ = pstats.Stats(pr).stats
        rows = sorted(((v[2], v[3], v[1], k) for k, v in st_.items()), reverse=True)
        tot = sum(r[0] for r in rows)
        print(f"total tottime {tot*1e6:.0f} us")
        for tt, ct, n, k in rows[:28]:
            print(f"{tt*1e6:8.1f} us self {ct*1e6:8.1f} us cum {n:5d}x  {k[2]} {k[0].split('/')[-1]}:{k[1]}")
    eng.run_until_idle()
