#!/usr/bin/env python
"""bench.py — aLoRA-turn TTFT & E2E vs standard-LoRA recompute, prefill tok/s (BASELINE.json metric).

Workload (BASELINE.json configs[1], C2): Llama-3.2-1B geometry (16 layers, d 2048,
32 q / 8 kv heads, head_dim 64, SwiGLU 8192, vocab 128256, tied lm_head), bf16,
random-init weights in HBM, 3 activated adapters r=32 on q/k/v, the reference's
multi_adapter turn algebra (bench.py:1-21): base turn (x=1792 prompt, y=256
generated) -> eval turn on all 3 adapters (conv + 3-token invocation, 16
generated tokens) per pipeline instance, `--batch` instances per step, B=16,
token budget 8192, 2k context. The same turns run twice, in aLoRA mode
(base-aligned reuse of the 2048 cached tokens) and LoRA mode (full recompute).

One timed "step" = the aLoRA eval turn's TTFT-defining forward (all 3*batch
suffix prefills in one packed varlen step), replayed with its metadata staged
in HBM; value = eval prompt tokens served per second of that forward
("effective prefill": cached + computed prompt tokens / TTFT forward time).
`e2e` = the same metric through the public Engine API (host prompts, per-step
H2D of packed metadata and D2H of ids), over the turn's wall-clock TTFT.
Whole-turn TTFT/E2E for both modes and their ratio are in "alora"/"lora"/"speedup".

--impl reference times the reference algorithm on the host CPU: the numpy
oracle (oracle/model_oracle.py, fp64 accumulation like aloraserve) running one
aLoRA eval request's suffix forward over a 2048-token cached prefix at C2 dims.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aLoRA-turn TTFT & e2e pipeline latency vs LoRA recompute; prefill tok/s"
UNIT = "prompt tok/s (eval turn, effective)"
C2 = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
          vocab_size=128256, max_seq_len=4096, seed=0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4, help="pipeline instances per step (x3 adapters = eval requests)")
    ap.add_argument("--prompt-len", type=int, default=1792)
    ap.add_argument("--gen-len", type=int, default=256)
    ap.add_argument("--adapter-gen", type=int, default=16)
    ap.add_argument("--rank", type=int, default=32)
    ap.add_argument("--lora-steps", type=int, default=2, help="timed LoRA-recompute eval turns")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default=None, help="write per-kernel profile here")
    ap.add_argument("--sweep", choices=["c3", "c4"], default=None,
                    help="c4: Llama-3-8B long-context prefix-reuse sweep (aLoRA vs LoRA eval TTFT at 4k-32k); "
                         "c3: Llama-3-8B + 8 aLoRA adapters, 64 eval requests over 8k contexts (one replica)")
    ap.add_argument("--contexts", default="4096,8192,16384,32768")
    ap.add_argument("--sync-decode", action="store_true",
                    help="read every decode step's ids back before launching the next (default: pipelined decode)")
    return ap.parse_args()


# ------------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def eval_split(args, B=16):
    """(cached, computed) prompt tokens of an aLoRA eval request: hits ((x+y-1)//B)*B, SURVEY.md Appendix B."""
    total = args.prompt_len + args.gen_len + 4  # conversation + base output + EOT + 3-token invocation
    cached = ((args.prompt_len + args.gen_len - 1) // B) * B
    return cached, total - cached


def c2_config(args, world):
    """The workload both arms report (BASELINE.json configs[1])."""
    return {"workload": "C2: Llama-3.2-1B geometry + 3 aLoRA adapters r=32, multi_adapter pipeline "
                        f"(x={args.prompt_len}, y={args.gen_len}, eval gen {args.adapter_gen}), "
                        f"{args.batch} instances x 3 adapters per eval turn, B=16, budget 8192; metric = eval "
                        "prompt tokens (cached + computed) per second of the TTFT-defining forward",
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
            "l2": "working set (2.5 GB weights + KV) exceeds the 126 MB L2; no flush needed",
            "decode": "synchronous" if getattr(args, "sync_decode", False) else "pipelined (Engine pipelined_decode)",
            **{k: v for k, v in C2.items() if k != "seed"}}


# --------------------------------------------------------------- reference ---
def oracle_c2(n_layers=None):
    """C2 geometry in the numpy oracle; random fp32 weights (values do not change CPU time)."""
    import oracle as O

    dims = dict(C2)
    if n_layers:
        dims["n_layers"] = n_layers
    cfg = O.OracleConfig(**dims, numerics="fp64acc")
    rng = np.random.default_rng(0)
    d, F = cfg.d_model, cfg.ffn

    def r(*shape):
        return (rng.random(shape, dtype=np.float32) - 0.5) * np.float32(0.05)

    w = {"layers": [{"attn_norm": np.ones(d, np.float32), "mlp_norm": np.ones(d, np.float32),
                     "wq": r(d, cfg.q_width), "wk": r(d, cfg.kv_width), "wv": r(d, cfg.kv_width),
                     "wo": r(cfg.q_width, d), "w_gate": r(d, F), "w_up": r(d, F), "w_down": r(F, d)}
                    for _ in range(cfg.n_layers)],
         "embed": r(cfg.vocab_size, d), "final_norm": np.ones(d, np.float32), "unembed": None}
    model = O.OracleModel(cfg, w)
    ad = O.oracle_adapter("adapter0", cfg, 32, seed=0, invocation_tokens=(cfg.vocab_size - 32,
                                                                          cfg.vocab_size - 31, cfg.vocab_size - 30))
    return O, cfg, model, ad


def cpu_sample(O, cfg, model, ad, prefix, suffix, B=16):
    """One aLoRA eval request: suffix forward over a `prefix`-token paged cache (random KV rows). Returns seconds."""
    n_blocks = -(-(prefix + suffix) // B)
    kv = np.random.default_rng(1).standard_normal((n_blocks, cfg.n_layers, 2, B, cfg.kv_width)).astype(np.float32)
    toks = np.random.default_rng(2).integers(0, cfg.vocab_size - 32, suffix)
    mask = np.arange(prefix, prefix + suffix) < prefix + suffix - 3  # the base path up to the invocation
    span = O.OracleSpan("r", toks, prefix, list(range(n_blocks)), ad, mask)
    t0 = time.perf_counter()
    model.forward_step([span], kv)
    return time.perf_counter() - t0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    prefix, suffix = eval_split(args)
    O, cfg, model, ad = oracle_c2()
    for _ in range(args.warmup):
        cpu_sample(O, cfg, model, ad, prefix, suffix)
    times = [cpu_sample(O, cfg, model, ad, prefix, suffix) for _ in range(args.steps)]
    t = statistics.mean(times)
    value = (prefix + suffix) / t
    cores = os.cpu_count()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": c2_config(args, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"1 of the turn's eval requests per step ({suffix}-token suffix over {prefix} "
                                       "cached tokens; the reference forward loops over spans, model.py:243, so "
                                       "tok/s per request is the turn's), oracle/model_oracle.py fp64 numpy "
                                       "(OpenBLAS threads = cores)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C4 sweep ---
C4 = dict(arch="llama", n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, ffn_dim=14336,
          vocab_size=128256, seed=0)


def run_sweep_c4(args):
    """BASELINE.json configs[3]: Llama-3-8B, one base->adapter pipeline per context length; the eval turn's TTFT
    with base-aligned reuse (aLoRA) vs standard-LoRA full recompute (budget 8192, chunked like vLLM)."""
    import torch
    import paper_2512_17910_b200 as P

    torch.cuda.set_device(0)
    rows = []
    for ctx in [int(c) for c in args.contexts.split(",")]:
        y = 256
        x = ctx - y - 4
        mcfg = P.ModelConfig(**C4, max_seq_len=ctx + 64, dtype="bf16")
        model = P.Model(mcfg, init="device", max_tokens=8192, max_seqs=16)
        res = {"context": ctx}
        for mode in ("alora", "lora"):
            spec = P.PipelineSpec(pipeline="base_adapter", mode=mode, prompt_len=x, gen_len=y, adapter_gen_len=16,
                                  n_adapters=1, batch=1)
            cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=8),
                                 pool_blocks=2 * (-(-(ctx + 64) // 16)) * 3 + 64, block_size=16,
                                 adapters=(P.AdapterSpec(adapter_id="adapter0", rank=32, seed=0,
                                                         invocation_tokens=P.invocation_for(mcfg.vocab_size, 0)),),
                                 comparison_mode=mode)
            eng = P.Engine(cfg, clock=P.WallClock(), model=model, pipelined_decode=not args.sync_decode)
            ttft, e2e, comp, base_tps = [], [], [], []
            for i in range(1 + max(1, args.lora_steps)):  # first pipeline is warm-up
                sp = P.PipelineSpec(**{**spec.__dict__, "seed": i})
                ph = P.pipeline.pipeline_phases(sp, eng, rid_prefix=f"{mode}{i}-")
                _, sub = next(ph)
                n0 = len(eng.metrics)
                P.pipeline.run_phase(eng, sub)
                b = eng.metrics[n0]
                _, sub = next(ph)
                torch.cuda.synchronize()
                n0 = len(eng.metrics)
                P.pipeline.run_phase(eng, sub)
                r = eng.metrics[n0]
                if i > 0:
                    ttft.append(r.ttft_s)
                    e2e.append(r.e2e_s)
                    comp.append(r.computed_tokens)
                    base_tps.append(b.prompt_len / b.prefill_s)
            res[mode] = {"ttft_ms": 1e3 * statistics.mean(ttft), "e2e_ms": 1e3 * statistics.mean(e2e),
                         "computed_tokens": int(statistics.mean(comp)),
                         "base_prefill_tok_s": statistics.mean(base_tps)}
            del eng
            torch.cuda.empty_cache()
        res["ttft_speedup"] = res["lora"]["ttft_ms"] / res["alora"]["ttft_ms"]
        res["e2e_speedup"] = res["lora"]["e2e_ms"] / res["alora"]["e2e_ms"]
        rows.append(res)
        print(json.dumps(res), flush=True)
        del model
        torch.cuda.empty_cache()
    print(json.dumps({"metric": "C4 eval-turn TTFT aLoRA vs LoRA recompute (Llama-3-8B geometry, bf16, 1 B200)",
                      "config": {"workload": "base_adapter pipeline, y=256, eval gen 16, B=16, budget 8192",
                                 **{k: v for k, v in C4.items() if k != "seed"}},
                      "data": "synthetic (random-init weights in HBM)", "sweep": rows}), flush=True)


def run_c3(args):
    """BASELINE.json configs[2] on one replica: Llama-3-8B bf16 + 8 activated adapters (r=32), a multi_adapter
    pipeline over 8 conversations of 8k tokens -> 64 concurrent eval requests (8 adapters x 8 instances),
    aLoRA (base-aligned reuse) vs LoRA recompute (budget 8192). Replicas scale it weakly (replicas.py)."""
    import torch
    import paper_2512_17910_b200 as P

    torch.cuda.set_device(0)
    ctx, y, n_ad, batch = 8192, 256, 8, 8
    x = ctx - y - 4
    mcfg = P.ModelConfig(**C4, max_seq_len=ctx + 64, dtype="bf16")
    model = P.Model(mcfg, init="device", max_tokens=8192, max_seqs=96)
    out = {}
    for mode in ("alora", "lora"):
        spec = P.PipelineSpec(pipeline="multi_adapter", mode=mode, prompt_len=x, gen_len=y, adapter_gen_len=16,
                              n_adapters=n_ad, batch=batch)
        blocks = -(-(ctx + 64) // 16)
        cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=8192, max_batch_requests=96),
                             pool_blocks=(batch * (n_ad + 1) + 8) * blocks, block_size=16,
                             adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=32, seed=k,
                                                          invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                            for k in range(n_ad)),
                             comparison_mode=mode)
        eng = P.Engine(cfg, clock=P.WallClock(), model=model, pipelined_decode=not args.sync_decode)
        ph = P.pipeline.pipeline_phases(spec, eng, rid_prefix=f"{mode}-")
        _, sub = next(ph)
        P.pipeline.run_phase(eng, sub)
        _, sub = next(ph)
        torch.cuda.synchronize()
        n0 = len(eng.metrics)
        t0 = time.perf_counter()
        P.pipeline.run_phase(eng, sub)
        wall = time.perf_counter() - t0
        rows = eng.metrics[n0:]
        out[mode] = {"requests": len(rows), "ttft_ms_mean": 1e3 * statistics.mean(r.ttft_s for r in rows),
                     "turn_ttft_ms": 1e3 * max(r.ttft_s for r in rows),
                     "e2e_ms_mean": 1e3 * statistics.mean(r.e2e_s for r in rows), "turn_wall_ms": 1e3 * wall,
                     "hit_tokens_per_request": statistics.mean(r.hit_tokens for r in rows),
                     "computed_tokens": int(sum(r.computed_tokens for r in rows)),
                     "eval_prompt_tok_s": sum(r.prompt_len for r in rows) / max(r.ttft_s for r in rows)}
        del eng
        torch.cuda.empty_cache()
    out["turn_ttft_speedup"] = out["lora"]["turn_ttft_ms"] / out["alora"]["turn_ttft_ms"]
    out["e2e_speedup"] = out["lora"]["e2e_ms_mean"] / out["alora"]["e2e_ms_mean"]
    print(json.dumps({"metric": "C3 eval turn, 64 requests: TTFT/E2E aLoRA vs LoRA recompute (1 replica, 1 B200)",
                      "config": {"workload": "multi_adapter, 8 conversations x 8 adapters, 8k context, y=256, "
                                             "eval gen 16, B=16, budget 8192",
                                 **{k: v for k, v in C4.items() if k != "seed"}},
                      "data": "synthetic (random-init weights in HBM)", **out}), flush=True)


# --------------------------------------------------------------------- ours ---
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.sweep == "c4":
        return run_sweep_c4(args)
    if args.sweep == "c3":
        return run_c3(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2512_17910_b200 as P

    mcfg = P.ModelConfig(**C2, dtype="bf16")
    n_eval = 3
    B = 16
    budget = 8192
    peak_tokens = args.prompt_len + args.gen_len + 1 + 3 + args.adapter_gen
    pool_blocks = max(4096, 2 * args.batch * (1 + n_eval) * (-(-peak_tokens // B)) + 64)

    def make_engine(mode):
        spec = P.PipelineSpec(pipeline="multi_adapter", mode=mode, prompt_len=args.prompt_len, gen_len=args.gen_len,
                              adapter_gen_len=args.adapter_gen, n_adapters=n_eval, batch=args.batch)
        cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=budget,
                                                                        max_batch_requests=4 * n_eval * args.batch + 8),
                             pool_blocks=pool_blocks, block_size=B,
                             adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=args.rank, seed=k,
                                                          invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                            for k in range(n_eval)),
                             comparison_mode=mode)
        model = P.Model(mcfg, init="device", max_tokens=budget, max_seqs=cfg.scheduler.max_batch_requests)
        return spec, P.Engine(cfg, clock=P.WallClock(), model=model, pipelined_decode=not args.sync_decode)

    # instrument the engine: capture the eval turn's first packed step and count native launches
    class Spy:
        def __init__(self, model):
            self.model, self.first, self.launches, self.h2d, self.d2h, self.armed = model, None, 0, 0, 0, False
            orig = model.run_packed

            def wrapped(p, kv, want_logits=True):
                out = orig(p, kv, want_logits)
                if self.armed:
                    if self.first is None:
                        self.first = p
                        self.h2d, self.d2h = model.last_h2d_bytes, model.last_d2h_bytes
                    self.launches += model.last_launches
                return out
            model.run_packed = wrapped
            orig_async = model.launch_async

            def wrapped_async(p, kv):  # pipelined decode steps count too
                out = orig_async(p, kv)
                if self.armed:
                    self.launches += model.last_launches
                return out
            model.launch_async = wrapped_async

    def run_turns(engine, spec, step_idx, spy, timed):
        """Base turn (untimed) then the eval turn; returns eval rows and the turn's wall/device times."""
        spec_i = P.PipelineSpec(**{**spec.__dict__, "seed": 1000 * rank + step_idx})
        phases = P.pipeline.pipeline_phases(spec_i, engine, rid_prefix=f"s{step_idx}-")
        stage, submits = next(phases)
        assert stage == "base"
        n0 = len(engine.metrics)
        P.pipeline.run_phase(engine, submits)
        base_rows = engine.metrics[n0:]
        stage, submits = next(phases)
        assert stage == "eval"
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        spy.armed, spy.first, spy.launches = timed, None, 0
        n0 = len(engine.metrics)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        t0 = time.perf_counter()
        P.pipeline.run_phase(engine, submits)
        ev1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        spy.armed = False
        return base_rows, engine.metrics[n0:], wall, ev0.elapsed_time(ev1) / 1e3

    results = {}
    device_value = None
    for mode in ("alora", "lora"):
        spec, eng = make_engine(mode)
        spy = Spy(eng.model)
        n_steps = args.steps if mode == "alora" else args.lora_steps
        n_warm = args.warmup if mode == "alora" else 1
        rows_t, walls, base_rows_all = [], [], []
        sampler = ClockSampler(local) if mode == "alora" else None
        for i in range(n_warm):
            run_turns(eng, spec, i, spy, timed=False)
        if sampler:
            sampler.__enter__()
        for i in range(n_steps):
            base_rows, rows, wall, dev = run_turns(eng, spec, n_warm + i, spy, timed=True)
            rows_t.append(rows)
            walls.append((wall, dev))
            base_rows_all.append(base_rows)
        launches = spy.launches
        first = spy.first
        res = {"rows": rows_t, "walls": walls, "base": base_rows_all, "launches": launches, "h2d": spy.h2d,
               "d2h": spy.d2h}
        if mode == "alora":
            # device-resident replay of the TTFT-defining forward (metadata staged in HBM before the events)
            m = eng.model
            st = m.stage(first, eng.pool.kv)
            for _ in range(args.warmup):
                m.launch(st)
            torch.cuda.synchronize()
            times = []
            for _ in range(args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                m.launch(st)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3)
            sampler.__exit__()
            res["clocks"] = sampler.summary()
            res["forward_s"] = statistics.mean(times)
            res["prompt_tokens"] = int(sum(r.prompt_len for r in rows_t[0]))
            res["fwd_rows"] = int(first["M"])
            res["fwd_launches"] = m.last_launches
            # per-kernel profile of the same forward (separate pass, not the timed one)
            m.set_profiling(True)
            m.launch(st)
            torch.cuda.synchronize()
            res["profile"] = m.profile_read()
            m.set_profiling(False)
        results[mode] = res
        del eng, spy
        torch.cuda.empty_cache()

    def turn_stats(res):
        ttft = [r.ttft_s for rows in res["rows"] for r in rows]
        e2e = [r.e2e_s for rows in res["rows"] for r in rows]
        turn_ttft = [max(r.ttft_s for r in rows) for rows in res["rows"]]
        comp = sum(r.computed_tokens for rows in res["rows"] for r in rows)
        hit = sum(r.hit_tokens for rows in res["rows"] for r in rows)
        prefill = [r.prefill_s for rows in res["rows"] for r in rows]
        return {"ttft_ms_mean": 1e3 * statistics.mean(ttft), "turn_ttft_ms": 1e3 * statistics.mean(turn_ttft),
                "e2e_ms_mean": 1e3 * statistics.mean(e2e), "turn_wall_ms": 1e3 * statistics.mean(w for w, _ in res["walls"]),
                "hit_rate": hit / (hit + comp), "hit_tokens_per_request": hit / sum(len(r) for r in res["rows"]),
                "computed_tokens": comp,
                "prefill_tok_s": sum(r.prompt_len - r.hit_tokens for rows in res["rows"] for r in rows)
                / max(1e-9, sum(max(r.prefill_s for r in rows) for rows in res["rows"]))}

    a, l = turn_stats(results["alora"]), turn_stats(results["lora"])
    # base turn: all instances' prompts prefill together; tok/s = prompt tokens / slowest prefill, per step
    base_prefill_tok_s = statistics.mean(sum(r.prompt_len for r in rows) / max(r.prefill_s for r in rows)
                                         for rows in results["alora"]["base"])
    ra = results["alora"]
    tokens = ra["prompt_tokens"]
    fwd = ra["forward_s"]
    turn_ttft_s = a["turn_ttft_ms"] / 1e3
    # aggregate over ranks (replicas): tokens summed, times max
    vals = torch.tensor([tokens, fwd, turn_ttft_s], dtype=torch.float64, device="cuda")
    if world > 1:
        tok_sum = vals[0:1].clone()
        dist.all_reduce(tok_sum, op=dist.ReduceOp.SUM)
        tmax = vals[1:].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tokens_all, fwd_max, ttft_max = float(tok_sum[0]), float(tmax[0]), float(tmax[1])
    else:
        tokens_all, fwd_max, ttft_max = float(tokens), fwd, turn_ttft_s
    if rank != 0:
        dist.destroy_process_group()
        return

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tf_peak = peaks.get("bf16_tflops", 1590.0)
    prof = ra["profile"]
    kernels = {}
    for k, v in prof.items():
        t = v["ms"] / 1e3 / v["launches"]
        by = v["bytes"] / v["launches"]
        fl = v["flops"] / v["launches"]
        kernels[k] = {"ms_total": round(v["ms"], 4), "launches": v["launches"], "us_per_launch": round(t * 1e6, 2),
                      "gb_s": round(by / t / 1e9, 1), "tflop_s": round(fl / t / 1e12, 2),
                      "hbm_frac": round(by / t / 1e9 / hbm_peak, 3), "tensor_frac": round(fl / t / 1e12 / tf_peak, 3)}
    dom = max(prof, key=lambda k: prof[k]["ms"])
    dv = prof[dom]
    dt = dv["ms"] / 1e3 / dv["launches"]
    ai = dv["flops"] / max(1.0, dv["bytes"])
    bound = "tensor" if ai > tf_peak * 1e12 / (hbm_peak * 1e9) else "hbm"
    if bound == "hbm":
        achieved, peak, unit = dv["bytes"] / dv["launches"] / dt / 1e9, hbm_peak, "GB/s"
    else:
        achieved, peak, unit = dv["flops"] / dv["launches"] / dt / 1e12, tf_peak, "TFLOP/s"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(dom)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            O, ocfg, om, oad = oracle_c2()
            prefix, suffix = eval_split(args)
            cpu_sample(O, ocfg, om, oad, prefix, suffix)
            t = min(cpu_sample(O, ocfg, om, oad, prefix, suffix) for _ in range(2))
            cpu = {"value": (prefix + suffix) / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"1 aLoRA eval request ({suffix}-token suffix over {prefix} cached tokens) at C2 dims, "
                             f"oracle/model_oracle.py fp64 numpy, best of 2 after 1 warm-up: {t:.2f} s"}
        except Exception as e:  # the CPU leg must not sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    value = tokens_all / fwd_max
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": fwd_max * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights in HBM, random conversations)",
        "config": {**c2_config(args, world), "eval_requests_per_step": int(tokens / (args.prompt_len + args.gen_len + 4)),
                   "forward_rows": ra["fwd_rows"]},
        "e2e": {"value": tokens_all / ttft_max, "unit": UNIT, "h2d_bytes_per_step": ra["h2d"],
                "d2h_bytes_per_step": ra["d2h"],
                "how": "Engine.submit/run_until_idle (public API), turn TTFT from the engine's WallClock stamps"},
        "alora": a, "lora": l,
        "speedup_vs_lora": {"ttft_mean": l["ttft_ms_mean"] / a["ttft_ms_mean"], "turn_ttft": l["turn_ttft_ms"] / a["turn_ttft_ms"],
                            "e2e_mean": l["e2e_ms_mean"] / a["e2e_ms_mean"]},
        "base_turn_prefill_tok_s": base_prefill_tok_s,
        "lora_recompute_prefill_tok_s": l["prefill_tok_s"],
        "roofline": {"kernel": dom, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak, "traffic": traffic,
                     "basis": "algorithmic bytes/flops per launch (runtime.cu tags) / CUDA-event launch time",
                     "peak_source": "MEASURED_PEAKS.json" if peaks else "B200_PROFILING.md fallback"},
        "kernels": kernels,
        "cpu_baseline": cpu,
        "clocks": ra["clocks"],
        "gpu_launches": ra["launches"],
    }
    if args.profile_json:
        with open(args.profile_json, "w") as f:
            json.dump({"kernels": kernels, "alora": a, "lora": l}, f, indent=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
