"""CPU cProfile of the eval turn's host path (submit + schedule + seq inputs) with a stub model."""
import cProfile, pstats, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P

C2 = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
          vocab_size=128256, max_seq_len=4096, seed=0)
mcfg = P.ModelConfig(**C2, dtype="bf16")

class Stub:
    def forward_step(self, seqs, kv):
        return {s.request_id: np.zeros(8, np.float32) for s in seqs}

spec = P.PipelineSpec(pipeline="multi_adapter", mode="alora", prompt_len=1792, gen_len=256, adapter_gen_len=16,
                      n_adapters=3, batch=4)
cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=64),
                     pool_blocks=4096, block_size=16,
                     adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=4, seed=k,
                                                  invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                    for k in range(3)), comparison_mode="alora")
import paper_2512_17910_b200.engine as E
E.register = None
eng = P.Engine(cfg, clock=P.VirtualClock() if hasattr(P, "VirtualClock") else P.WallClock(), model=Stub(),
               pool_storage="meta")
for i in range(3):
    sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
    ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"w{i}-")
    st, sub = next(ph); P.pipeline.run_phase(eng, sub)
    st, sub = next(ph)
    if i < 2:
        P.pipeline.run_phase(eng, sub)
        continue
    pr = cProfile.Profile(); pr.enable()
    t0 = time.perf_counter()
    for rid, prompt, adapter_id, gen, meta in sub:
        eng.submit(prompt, adapter_id=adapter_id, max_new_tokens=gen, request_id=rid, meta=meta)
    t1 = time.perf_counter()
    eng.step()
    t2 = time.perf_counter()
    pr.disable()
    print(f"submit {1e3*(t1-t0):.2f} ms  first step {1e3*(t2-t1):.2f} ms  ({len(sub)} requests)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
