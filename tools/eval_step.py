"""Time one aLoRA eval-turn step (suffix prefill, or a decode step) at the C2 / C3 bench geometry without the base
turn: random cached KV in the paged pool, requests of one conversation share its prefix blocks (as in the bench).

usage: python tools/eval_step.py [c2|c3] [decode] [reps] [layers]
prints the event-timed forward and, with PROFILE=1, the per-kernel table of one profiled pass.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2512_17910_b200 as P  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
decode = len(sys.argv) > 2 and sys.argv[2] == "decode"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
layers = int(sys.argv[4]) if len(sys.argv) > 4 else None
if cfg_name == "c3":
    dims = dict(arch="llama", n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, ffn_dim=14336,
                vocab_size=128256)
    n_conv, n_ad, ctx = 8, 8, 8192
else:
    dims = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
                vocab_size=128256)
    n_conv, n_ad, ctx = 4, 3, 2048
if layers:
    dims["n_layers"] = layers
B = 16
cached = ((ctx - 5) // B) * B
suffix = ctx - cached
cfg = P.ModelConfig(**dims, max_seq_len=ctx + 64, dtype="bf16")
n_req = n_conv * n_ad
model = P.Model(cfg, init="device", max_tokens=8192, max_seqs=max(64, n_req))
pre = cached // B
tail = -(-(ctx + 32) // B) - pre
nb = n_conv * pre + n_req * tail + 8
pool = P.BlockPool(nb, B, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
pool.kv.normal_()
V = cfg.vocab_size
ads = [P.generate_adapter(f"adapter{k}", cfg.d_model, 32, seed=k, invocation_tokens=P.invocation_for(V, k),
                          kv_width=cfg.kv_width, q_width=cfg.q_width) for k in range(n_ad)]
rng = np.random.default_rng(0)
seqs = []
for c in range(n_conv):
    for k in range(n_ad):
        i = len(seqs)
        table = list(range(c * pre, (c + 1) * pre)) + list(range(n_conv * pre + i * tail, n_conv * pre + (i + 1) * tail))
        if decode:
            start, toks = ctx + 3, rng.integers(0, V - 32, 1)
        else:
            start, toks = cached, rng.integers(0, V - 32, suffix)
        mask = np.arange(start, start + len(toks)) < ctx - 3
        seqs.append(P.SeqInput(f"c{c}a{k}", toks, start, table, ads[k], mask))
p = model.pack(seqs, B)
p["graphable"] = os.environ.get("GRAPH", "1") != "0"
st = model.stage(p, pool.kv)
for _ in range(3):
    model.launch(st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    model.launch(st)
e1.record()
torch.cuda.synchronize()
print(f"{cfg_name} {'decode' if decode else 'eval'} step M={p['M']} S={p['S']} layers={cfg.n_layers}: "
      f"{e0.elapsed_time(e1) / reps:.3f} ms/forward (launches {model.last_launches})", flush=True)
if os.environ.get("PROFILE"):
    model.set_profiling(True)
    model.launch(st)
    torch.cuda.synchronize()
    prof = model.profile_read()
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        t = v["ms"] / v["launches"]
        print(f"  {k:14s} {v['ms']:8.3f} ms  {v['launches']:4d} x {1e3 * t:8.2f} us  "
              f"{v['bytes'] / v['launches'] / (t * 1e-3) / 1e9:7.0f} GB/s  "
              f"{v['flops'] / v['launches'] / (t * 1e-3) / 1e12:6.1f} TF/s")
    for row in model.profile_kernels():
        print("   ", row[0], row[1].split("(")[0], "grid", row[2], "x", row[3])
    model.set_profiling(False)
