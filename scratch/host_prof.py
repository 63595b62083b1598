"""cProfile of the aLoRA eval turn through the Engine (host overhead per step)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P
C2 = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
          vocab_size=128256, max_seq_len=4096, seed=0)
mcfg = P.ModelConfig(**C2, dtype="bf16")
spec = P.PipelineSpec(pipeline="multi_adapter", mode="alora", prompt_len=1792, gen_len=256, adapter_gen_len=16, n_adapters=3, batch=4)
cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=64), pool_blocks=4096, block_size=16,
                     adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=32, seed=k, invocation_tokens=P.invocation_for(mcfg.vocab_size, k)) for k in range(3)),
                     comparison_mode="alora")
model = P.Model(mcfg, init="device", max_tokens=8192, max_seqs=64)
eng = P.Engine(cfg, clock=P.WallClock(), model=model)
for i in range(3):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"w{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    if i < 2:
        P.pipeline.run_phase(eng, sub)
    else:
        torch.cuda.synchronize()
        pr = cProfile.Profile(); t0 = time.perf_counter()
        import paper_2512_17910_b200.engine as E
        tm = {}
        orig_sched = eng.scheduler.schedule_step
        def sched(now):
            a = time.perf_counter(); r = orig_sched(now); tm["sched"] = time.perf_counter() - a; return r
        eng.scheduler.schedule_step = sched
        orig_rp = eng.model.run_packed
        def rp(p, kv, want_logits=True):
            a = time.perf_counter(); r = orig_rp(p, kv, want_logits); tm["run_packed"] = time.perf_counter() - a; return r
        eng.model.run_packed = rp
        orig_pack = eng.model.pack
        def pk(seqs, bs):
            a = time.perf_counter(); r = orig_pack(seqs, bs); tm["pack"] = time.perf_counter() - a; return r
        eng.model.pack = pk
        for rid, prompt, adapter_id, gen, meta in sub:
            eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
        t1 = time.perf_counter()
        eng.step()
        pr.disable(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"submit {1e3*(t1-t0):.2f} ms, first step {1e3*(time.perf_counter()-t1):.2f} ms", {k: round(v*1e3, 3) for k, v in tm.items()})
        eng.run_until_idle()
