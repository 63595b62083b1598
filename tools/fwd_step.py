"""One aLoRA eval-turn forward at C2 dims without running the base turn (random cached KV).

usage: python tools/fwd_step.py [n_requests] [suffix] [cached] [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2512_17910_b200 as P

n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 12
suffix = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cached = int(sys.argv[3]) if len(sys.argv) > 3 else 2032
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
C2 = dict(arch="llama", n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
          vocab_size=128256, max_seq_len=4096, seed=0)
cfg = P.ModelConfig(**C2, dtype="bf16")
import os
model = P.Model(cfg, init="device", max_tokens=8192, max_seqs=64, graphs=os.environ.get("ALORA_GRAPHS", "1") != "0")
B = 16
nb = -(-(cached + suffix) // B)
pool = P.BlockPool(n_req * nb + 8, B, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
pool.kv.normal_()
ads = [P.generate_adapter(f"adapter{k}", cfg.d_model, 32, seed=k, invocation_tokens=P.invocation_for(cfg.vocab_size, k),
                          kv_width=cfg.kv_width, q_width=cfg.q_width) for k in range(3)]
rng = np.random.default_rng(0)
seqs = []
for r in range(n_req):
    ids = list(range(r * nb, (r + 1) * nb))
    toks = rng.integers(0, cfg.vocab_size - 32, suffix)
    mask = np.arange(cached, cached + suffix) < cached + suffix - 19  # adapter on the last 19 rows
    seqs.append(P.SeqInput(f"r{r}", toks, cached, ids, ads[r % 3], mask))
p = model.pack(seqs, B)
if os.environ.get("FORCE_GRAPH"): p["graphable"] = True
st = model.stage(p, pool.kv)
for _ in range(3):
    model.launch(st)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    model.launch(st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
hs = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model.launch(st)
    hs.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print(f"forward M={p['M']} S={p['S']}: {np.median(ts):.3f} ms device, host launch {1e3*np.median(hs):.3f} ms (launches {model.last_launches})", flush=True)
