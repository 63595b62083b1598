#!/usr/bin/env python
"""bench.py -- aLoRA-turn TTFT & E2E vs standard-LoRA recompute, prefill tok/s (BASELINE.json metric).

Default workload (--config c3, BASELINE.json configs[2], the north-star configuration): Llama-3-8B
geometry (32 layers, d 4096, 32 q / 8 kv heads, head_dim 128, SwiGLU 14336, vocab 128256, tied
lm_head), bf16, random-init weights in HBM, 8 activated adapters r=32 on q/k/v, the reference's
multi_adapter turn algebra (reference bench.py:1-21, 245-306): per pipeline instance a base turn
(x = 7932 prompt tokens, y = 256 generated) then an eval turn on all 8 adapters (conversation + EOT +
3-token invocation = 8k context, 16 generated tokens). 8 instances per replica -> 64 concurrent eval
requests, B=16, token budget 8192. The same turns run in aLoRA mode (base-aligned reuse of the
8,176 cached tokens per request) and in LoRA mode (full recompute). --config c2 is configs[1]
(Llama-3.2-1B, 3 adapters, 4 instances, 2k context).

One timed "step" = the aLoRA eval turn's TTFT-defining forward (all eval requests' suffix prefills
in one packed varlen step), replayed with its metadata staged in HBM; `value` = eval prompt tokens
served per second of that forward ("effective prefill": cached + computed prompt tokens / forward
time), summed over replicas with the max time over ranks. `e2e` = the same metric through the public
Engine API (host prompts, per-step H2D of the packed metadata and D2H of the ids) over the turn's
TTFT from the engine's WallClock stamps (reference metrics.py:69-73). Whole-turn TTFT / E2E for both
modes and their ratio are in "alora" / "lora" / "speedup_vs_lora" (reference bench.py:422-435,
525-551).

--gpus N (N > 1) without torchrun re-launches itself under torch.distributed.run, one process per
GPU: N request-parallel replicas (replicas.py; pipeline instance i on replica i mod N, no data-path
collective), `scaling` weak (each replica serves the config's instances).

--impl reference times the reference algorithm on the host CPU: the numpy oracle
(oracle/model_oracle.py, fp64 accumulation like aloraserve model.py:95-98) running one aLoRA eval
request's suffix forward over its cached prefix at the config's dims. A full-depth 8B forward does
not fit a bounded CPU sample, so 2 layers are timed and the per-layer time is extrapolated to the
full depth ("extrapolated" in the sample string); the reference loops over spans (model.py:243), so
one request's tok/s is the turn's.
"""

import argparse
import json
import os
import socket
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
LLAMA_1B = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
                vocab_size=128256, seed=0)
LLAMA_8B = dict(arch="llama", n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, ffn_dim=14336,
                vocab_size=128256, seed=0)
LLAMA_70B = dict(arch="llama", n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128, d_model=8192, ffn_dim=28672,
                 vocab_size=128256, seed=0)
CONFIGS = {
    # BASELINE.json configs[1]: 1B + 3 adapters, 2k context, 4 instances x 3 adapters = 12 eval requests
    "c2": dict(model=LLAMA_1B, n_adapters=3, batch=4, context=2048, name="C2: Llama-3.2-1B + 3 aLoRA adapters r=32"),
    # BASELINE.json configs[2]: 8B + 8 adapters, 8k context, 8 instances x 8 adapters = 64 eval requests / replica
    "c3": dict(model=LLAMA_8B, n_adapters=8, batch=8, context=8192, name="C3: Llama-3-8B + 8 aLoRA adapters r=32"),
    # BASELINE.json configs[4]: 70B + 4 adapters, 16k context, tensor parallel over the ranks (TP = world size;
    # every rank runs the same requests on its shard, fused NVLink all-reduce + residual + RMSNorm)
    "c5": dict(model=LLAMA_70B, n_adapters=4, batch=2, context=16384, tp=True,
               name="C5: Llama-3-70B + 4 aLoRA adapters r=32, tensor parallel"),
}
B = 16
BUDGET = 8192
RANK_R = 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--gen-len", type=int, default=256, help="base-turn generated tokens (y)")
    ap.add_argument("--layers", type=int, default=None,
                    help="override the model depth (C5 on fewer GPUs than its shards need; reported in config)")
    ap.add_argument("--adapter-gen", type=int, default=16)
    ap.add_argument("--lora-steps", type=int, default=5, help="timed LoRA-recompute eval turns")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default=None, help="write the per-kernel profile here")
    ap.add_argument("--sweep", choices=["c4"], default=None,
                    help="c4: Llama-3-8B long-context prefix-reuse sweep (aLoRA vs LoRA eval TTFT at 4k-32k)")
    ap.add_argument("--contexts", default="4096,8192,16384,32768")
    ap.add_argument("--probe-ranks", action="store_true",
                    help="launch plumbing check only: init the ranks (gloo without CUDA), print each replica's "
                         "pipeline instances and n_gpus as rank 0 sees it; no model work")
    ap.add_argument("--sync-decode", action="store_true",
                    help="read every decode step's ids back before launching the next (default: pipelined decode)")
    return ap.parse_args()


def workload(args):
    c = dict(CONFIGS[args.config])
    if args.layers:
        c["model"] = dict(c["model"], n_layers=args.layers)
    x = c["context"] - args.gen_len - 4  # conversation + base output + EOT + 3-token invocation = context
    cached = ((x + args.gen_len - 1) // B) * B  # base-aligned hits ((x+y-1)//B)*B, SURVEY.md Appendix B
    return dict(c, x=x, cached=cached, suffix=c["context"] - cached)


def config_dict(args, world):
    """The `config` object of both arms' JSON lines (identical for the same flags and world size)."""
    w = workload(args)
    n_eval = w["n_adapters"] * w["batch"]
    return {"workload": f"{w['name']}, multi_adapter pipeline (x={w['x']}, y={args.gen_len}, eval gen "
                        f"{args.adapter_gen}), {w['batch']} instances x {w['n_adapters']} adapters per replica "
                        f"= {n_eval} eval requests of {w['context']} tokens ({w['cached']} cached + {w['suffix']} "
                        f"computed), B={B}, token budget {BUDGET}; metric = eval prompt tokens (cached + computed) "
                        "per second of the TTFT-defining forward",
            "config": args.config, "context": w["context"], "eval_requests_per_replica": n_eval,
            "forward_rows_per_replica": n_eval * w["suffix"],
            "parallelism": (f"TP={world} (Megatron shards, fused peer-memory all-reduce)" if w.get("tp")
                            else f"replicas x{world} (request-parallel, instance affinity)") if world > 1 else "1 GPU",
            **({"depth": f"{args.layers} of {CONFIGS[args.config]['model']['n_layers']} layers (--layers)"}
               if args.layers else {}),
            "l2": "no flush needed: every step streams the weights (>= 2.5 GB) and the cached KV, both far above "
                  "the 126 MB L2",
            "decode": "synchronous" if args.sync_decode else "pipelined (Engine pipelined_decode)",
            **{k: v for k, v in w["model"].items() if k != "seed"}}


# ------------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, local_rank):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ids = [v.strip() for v in vis.split(",")] if vis else None
        self.index = ids[local_rank] if ids and local_rank < len(ids) else str(local_rank)
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.index, f"--query-gpu={self.Q}",
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
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- reference ---
def oracle_setup(args, n_layers=2):
    """The config's geometry in the numpy oracle at `n_layers` depth; random fp32 weights (values do not
    change CPU time)."""
    import oracle as O

    dims = dict(workload(args)["model"], n_layers=n_layers)
    cfg = O.OracleConfig(**dims, max_seq_len=workload(args)["context"] + 64, numerics="fp64acc")
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
    V = cfg.vocab_size
    ad = O.oracle_adapter("adapter0", cfg, RANK_R, seed=0, invocation_tokens=(V - 32, V - 31, V - 30))
    return O, cfg, model, ad


def cpu_sample(args, setup):
    """One aLoRA eval request's suffix forward over its cached prefix (random KV rows), timed on the host:
    (seconds extrapolated to the full depth, seconds measured, layers run)."""
    O, cfg, model, ad = setup
    w = workload(args)
    prefix, suffix = w["cached"], w["suffix"]
    n_blocks = -(-(prefix + suffix) // B)
    kv = np.random.default_rng(1).standard_normal((n_blocks, cfg.n_layers, 2, B, cfg.kv_width), dtype=np.float32)
    toks = np.random.default_rng(2).integers(0, cfg.vocab_size - 32, suffix)
    mask = np.arange(prefix, prefix + suffix) < prefix + suffix - 3  # base path up to the invocation
    span = O.OracleSpan("r", toks, prefix, list(range(n_blocks)), ad, mask)
    t0 = time.perf_counter()
    hf = model.last_hidden(span, kv)  # embed + the timed layers (model.py:263-271)
    t1 = time.perf_counter()
    O.mm(hf, model._unembed())  # lm_head of the last row (model.py:272), fp64 up-cast as in model.py:95-98
    t2 = time.perf_counter()
    full = w["model"]["n_layers"]
    return (t2 - t1) + (t1 - t0) * full / cfg.n_layers, t2 - t0, cfg.n_layers


def cpu_baseline_entry(args, times, layers):
    w = workload(args)
    t = statistics.median(times)
    return {"value": w["context"] / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"1 aLoRA eval request per sample ({w['suffix']}-token suffix over {w['cached']} cached tokens) "
                      f"at {args.config} widths; oracle/model_oracle.py fp64 numpy (OpenBLAS on all host cores); "
                      f"{layers} of {w['model']['n_layers']} layers timed, per-layer time extrapolated to the full "
                      f"depth + the measured lm_head (extrapolated); median of {len(times)}: {t:.2f} s/request"}


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    setup = oracle_setup(args, n_layers=1 if workload(args).get("tp") else 2)  # 70B widths: one timed layer
    for _ in range(args.warmup):
        cpu_sample(args, setup)
    samples = [cpu_sample(args, setup) for _ in range(args.steps)]
    times = [s[0] for s in samples]
    cpu = cpu_baseline_entry(args, times, samples[0][2])
    t = statistics.median(times)
    value = workload(args)["context"] / t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if workload(args).get("tp") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(args, world), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "measured_ms_per_step": 1e3 * statistics.median(s[1] for s in samples)}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C4 sweep ---
def run_sweep_c4(args):
    """BASELINE.json configs[3]: Llama-3-8B, one base->adapter pipeline per context length; the eval turn's TTFT
    with base-aligned reuse (aLoRA) vs standard-LoRA full recompute (budget 8192, chunked like vLLM)."""
    import torch
    import paper_2512_17910_b200 as P

    torch.cuda.set_device(0)
    rows = []
    sampler = ClockSampler(0)
    sampler.__enter__()
    for ctx in [int(c) for c in args.contexts.split(",")]:
        y = 256
        x = ctx - y - 4
        mcfg = P.ModelConfig(**LLAMA_8B, max_seq_len=ctx + 64, dtype="bf16")
        model = P.Model(mcfg, init="device", max_tokens=BUDGET, max_seqs=16)
        res = {"context": ctx}
        for mode in ("alora", "lora"):
            spec = P.PipelineSpec(pipeline="base_adapter", mode=mode, prompt_len=x, gen_len=y, adapter_gen_len=16,
                                  n_adapters=1, batch=1)
            cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=BUDGET, max_batch_requests=8),
                                 pool_blocks=2 * (-(-(ctx + 64) // B)) * 3 + 64, block_size=B,
                                 adapters=(P.AdapterSpec(adapter_id="adapter0", rank=RANK_R, seed=0,
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
            res[mode] = {"ttft_ms_median": 1e3 * statistics.median(ttft), "ttft_ms_min": 1e3 * min(ttft),
                         "e2e_ms_median": 1e3 * statistics.median(e2e),
                         "computed_tokens": int(statistics.mean(comp)),
                         "base_prefill_tok_s": statistics.median(base_tps), "turns": len(ttft)}
            del eng
            torch.cuda.empty_cache()
        res["ttft_speedup"] = res["lora"]["ttft_ms_median"] / res["alora"]["ttft_ms_median"]
        res["e2e_speedup"] = res["lora"]["e2e_ms_median"] / res["alora"]["e2e_ms_median"]
        rows.append(res)
        print(json.dumps(res), flush=True)
        del model
        torch.cuda.empty_cache()
    sampler.__exit__()
    print(json.dumps({"metric": "C4 eval-turn TTFT aLoRA vs LoRA recompute (Llama-3-8B geometry, bf16, 1 B200)",
                      "config": {"workload": "base_adapter pipeline, y=256, eval gen 16, B=16, budget 8192",
                                 **{k: v for k, v in LLAMA_8B.items() if k != "seed"}},
                      "data": "synthetic (random-init weights in HBM)", "clocks": sampler.summary(),
                      "sweep": rows}), flush=True)


# ------------------------------------------------------------- multi-rank ---
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args):
    """bench.py --gpus N run directly: one process per GPU under torch.distributed.run (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def probe_ranks(args):
    import torch
    import torch.distributed as dist
    from paper_2512_17910_b200.replicas import replica_instances

    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    w = workload(args)
    tp = bool(w.get("tp")) and world > 1
    mine = replica_instances(w["batch"], 1, 0) if tp else replica_instances(w["batch"] * world, world, rank)
    every = [None] * world
    if world > 1:
        dist.all_gather_object(every, mine)
    else:
        every = [mine]
    if rank == 0:
        print(json.dumps({"probe": "ranks", "n_gpus": world, "instances_per_rank": every,
                          "eval_requests_total": (len(every[0]) if tp else sum(len(m) for m in every)) * w["n_adapters"],
                          "config": config_dict(args, world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------- ours ---
def main():
    args = parse()
    if args.sweep == "c4":
        return run_sweep_c4(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # the CPU arm runs once (rank 0); no ranks to spawn
            os.environ["WORLD_SIZE"] = str(args.gpus)
        else:
            sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        return run_reference(args)
    if args.probe_ranks:
        return probe_ranks(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2512_17910_b200 as P
    from paper_2512_17910_b200.replicas import replica_instances

    w = workload(args)
    tp = bool(w.get("tp")) and world > 1  # C5: the ranks are one tensor-parallel model, not replicas
    mcfg = P.ModelConfig(**w["model"], max_seq_len=w["context"] + args.adapter_gen + 64, dtype="bf16")
    n_eval = w["n_adapters"]
    blocks = -(-(w["context"] + args.adapter_gen) // B)
    # the LoRA arm recomputes every eval request (its own blocks) while the base turn's blocks stay cached
    pool_blocks = (w["batch"] * (n_eval + 1) + 8) * blocks
    max_batch = n_eval * w["batch"] + 8
    if tp:
        model = P.TPModel(mcfg, P.TorchDistGroup(), init="device", max_tokens=BUDGET, max_seqs=max_batch)
    else:
        model = P.Model(mcfg, init="device", max_tokens=BUDGET, max_seqs=max_batch)
    n_inst = w["batch"] if tp else w["batch"] * world
    # this replica's pipeline instances (every instance on every rank under TP)
    mine = replica_instances(n_inst, 1, 0) if tp else replica_instances(n_inst, world, rank)

    def make_engine(mode):
        spec = P.PipelineSpec(pipeline="multi_adapter", mode=mode, prompt_len=w["x"], gen_len=args.gen_len,
                              adapter_gen_len=args.adapter_gen, n_adapters=n_eval, batch=n_inst)
        cfg = P.EngineConfig(model=mcfg, scheduler=P.SchedulerConfig(token_budget=BUDGET, max_batch_requests=max_batch),
                             pool_blocks=pool_blocks, block_size=B,
                             adapters=tuple(P.AdapterSpec(adapter_id=f"adapter{k}", rank=RANK_R, seed=k,
                                                          invocation_tokens=P.invocation_for(mcfg.vocab_size, k))
                                            for k in range(n_eval)),
                             comparison_mode=mode)
        return spec, P.Engine(cfg, clock=P.WallClock(), model=model, pipelined_decode=not args.sync_decode)

    class Spy:
        """Captures the eval turn's first packed step and counts native launches / copies."""

        def __init__(self, model):
            self.first, self.launches, self.h2d, self.d2h, self.armed = None, 0, 0, 0, False
            self.orig_run, self.orig_async = model.run_packed, model.launch_async

            def wrapped(p, kv, want_logits=True):
                out = self.orig_run(p, kv, want_logits)
                if self.armed:
                    if self.first is None:
                        self.first = p
                        self.h2d, self.d2h = model.last_h2d_bytes, model.last_d2h_bytes
                    self.launches += model.last_launches
                return out

            def wrapped_async(p, kv):  # pipelined decode steps count too
                out = self.orig_async(p, kv)
                if self.armed:
                    self.launches += model.last_launches
                return out
            model.run_packed, model.launch_async = wrapped, wrapped_async

        def detach(self):
            model.run_packed, model.launch_async = self.orig_run, self.orig_async

    def run_turns(engine, spec, step_idx, spy, timed):
        """Base turn (untimed) then the eval turn; returns (base rows, eval rows, eval requests, wall s)."""
        spec_i = P.PipelineSpec(**{**spec.__dict__, "seed": 1000 + step_idx})
        phases = P.pipeline.pipeline_phases(spec_i, engine, rid_prefix=f"s{step_idx}-", instances=mine)
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
        t0 = time.perf_counter()
        P.pipeline.run_phase(engine, submits)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        spy.armed = False
        rows = engine.metrics[n0:]
        return base_rows, rows, [engine.finished[r.request_id] for r in rows], wall

    def turn_stats(turns):
        """turns: [(eval rows, eval requests, wall)] of the timed eval turns."""
        ttft = [r.ttft_s for rows, _, _ in turns for r in rows]
        turn_ttft = [max(r.ttft_s for r in rows) for rows, _, _ in turns]
        e2e = [r.e2e_s for rows, _, _ in turns for r in rows]
        comp = sum(r.prompt_len - r.hit_tokens for rows, _, _ in turns for r in rows)
        hit = sum(r.hit_tokens for rows, _, _ in turns for r in rows)
        # prefill tok/s over the turn's prefill wall time: computed prompt tokens / (last prefill end - first start)
        pf = [sum(q.prompt_len - q.hit_tokens for q in reqs) /
              max(1e-9, max(q.decode_start for q in reqs) - min(q.prefill_start for q in reqs))
              for _, reqs, _ in turns]
        return {"turns": len(turns), "requests_per_turn": len(turns[0][0]),
                "ttft_ms_mean": 1e3 * statistics.mean(ttft), "turn_ttft_ms_median": 1e3 * statistics.median(turn_ttft),
                "turn_ttft_ms_min": 1e3 * min(turn_ttft), "e2e_ms_mean": 1e3 * statistics.mean(e2e),
                "e2e_ms_median": 1e3 * statistics.median(e2e),
                "turn_wall_ms_median": 1e3 * statistics.median(wl for _, _, wl in turns),
                "hit_rate": hit / max(1, hit + comp), "hit_tokens_per_request": hit / max(1, len(ttft)),
                "computed_prompt_tokens_per_turn": comp // len(turns),
                "prefill_tok_s": statistics.median(pf)}

    results = {}
    for mode in ("alora", "lora"):
        spec, eng = make_engine(mode)
        spy = Spy(model)
        n_steps = args.steps if mode == "alora" else max(5, args.lora_steps)
        n_warm = args.warmup if mode == "alora" else 1
        for i in range(n_warm):
            run_turns(eng, spec, i, spy, timed=False)
        sampler = ClockSampler(local).__enter__()
        turns, base_tps = [], []
        for i in range(n_steps):
            base_rows, rows, reqs, wall = run_turns(eng, spec, n_warm + i, spy, timed=True)
            turns.append((rows, reqs, wall))
            breqs = [eng.finished[r.request_id] for r in base_rows]
            base_tps.append(sum(q.prompt_len for q in breqs) /
                            max(1e-9, max(q.decode_start for q in breqs) - min(q.prefill_start for q in breqs)))
        res = {"stats": turn_stats(turns), "base_prefill_tok_s": statistics.median(base_tps),
               "e2e_launches": spy.launches, "h2d": spy.h2d, "d2h": spy.d2h}
        if mode == "alora":
            # device-resident replay of the TTFT-defining forward (metadata staged in HBM before the events)
            first = spy.first
            st = model.stage(first, eng.pool.kv)
            for _ in range(args.warmup):
                model.launch(st)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                model.launch(st)
            e1.record()
            torch.cuda.synchronize()
            res["forward_s"] = e0.elapsed_time(e1) / 1e3 / args.steps
            res["prompt_tokens"] = int(sum(r.prompt_len for r in turns[0][0]))
            res["fwd_rows"] = int(first["M"])
            res["fwd_launches"] = model.last_launches
            # per-kernel profile of the same forward (a separate, event-bracketed pass; not the timed one)
            model.set_profiling(True)
            model.launch(st)
            torch.cuda.synchronize()
            res["profile"] = model.profile_read()
            res["kernels_launched"] = model.profile_kernels()
            model.set_profiling(False)
        sampler.__exit__()
        res["clocks"] = sampler.summary()
        results[mode] = res
        spy.detach()
        del eng, spy
        torch.cuda.empty_cache()

    a, l = results["alora"]["stats"], results["lora"]["stats"]
    ra = results["alora"]
    tokens, fwd = ra["prompt_tokens"], ra["forward_s"]
    turn_ttft_s = a["turn_ttft_ms_median"] / 1e3
    vals = torch.tensor([tokens, fwd, turn_ttft_s], dtype=torch.float64, device="cuda")
    if world > 1:  # aggregate: replicas sum their tokens (TP ranks share them), times are the max over ranks
        tok_sum = vals[0:1].clone()
        if not tp:
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
            traffic = json.load(f).get(args.config, {}).get(dom)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            setup = oracle_setup(args, n_layers=1 if w.get("tp") else 2)
            samples = [cpu_sample(args, setup) for _ in range(2)]
            cpu = cpu_baseline_entry(args, [s[0] for s in samples], samples[0][2])
        except Exception as e:  # the CPU leg must not sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    value = tokens_all / fwd_max
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": fwd_max * 1e3, "higher_is_better": True, "scaling": "strong" if tp else "weak",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights in HBM, random conversations)",
        "config": config_dict(args, world),
        "e2e": {"value": tokens_all / ttft_max, "unit": UNIT, "h2d_bytes_per_step": ra["h2d"],
                "d2h_bytes_per_step": ra["d2h"],
                "how": "Engine.submit/run_until_idle (public API) from host prompts; median turn TTFT (slowest "
                       "request's queue + prefill) from the engine's WallClock stamps over the timed eval turns"},
        "alora": a, "lora": l,
        "speedup_vs_lora": {"ttft_mean": l["ttft_ms_mean"] / a["ttft_ms_mean"],
                            "turn_ttft_median": l["turn_ttft_ms_median"] / a["turn_ttft_ms_median"],
                            "e2e_median": l["e2e_ms_median"] / a["e2e_ms_median"]},
        "base_turn_prefill_tok_s": ra["base_prefill_tok_s"],
        "lora_recompute_prefill_tok_s": l["prefill_tok_s"],
        "roofline": {"kernel": dom, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak, "traffic": traffic,
                     "basis": "algorithmic bytes/flops per launch (runtime.cu tags, DESIGN.md §4) / CUDA-event "
                              "launch time on the launch stream",
                     "peak_source": ("MEASURED_PEAKS.json (burst: each kernel is timed on its own, event-bracketed)"
                                     if peaks else "B200_PROFILING.md fallback"),
                     # the sustained tensor figure (cuBLAS back to back for 4 s under the same power cap) beside it
                     "peak_sustained": peaks.get("bf16_tflops_sustained") if bound == "tensor" else None,
                     "frac_sustained": (achieved / peaks["bf16_tflops_sustained"]
                                        if bound == "tensor" and peaks.get("bf16_tflops_sustained") else None)},
        "kernels": kernels,
        "cpu_baseline": cpu,
        "clocks": ra["clocks"],
        "clocks_lora_arm": results["lora"]["clocks"],
        "gpu_launches": ra["fwd_launches"] * args.steps,
        "gpu_launches_e2e_turn": ra["e2e_launches"],
    }
    if args.profile_json:
        with open(args.profile_json, "w") as f:
            json.dump({"kernels": kernels, "kernels_launched": ra["kernels_launched"], "alora": a, "lora": l}, f,
                      indent=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
