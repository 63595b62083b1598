"""Generate the golden fixtures under tests/golden/ by IMPORTING THE REFERENCE.

Run in the build container only (the reference is not on the GPU box):

    python oracle/gen_golden.py

It imports aloraserve read-only from /root/reference/pkg/src (no bytecode is
written there) and records, for fixed seeds:

  hash_kat.json        hash_block known answers + full chains (kv_cache.py:41-96)
  projection.npz       project_qkv_masked outputs (model.py:117-146)
  attention.npz        paged_attention outputs (model.py:149-187)
  forward.npz          Model.forward_step logits and KV rows (model.py:233-272)
  pipelines.json/.npz  run_sync_pipeline runs (bench.py:264-306): generated ids,
                       hit/computed tokens, virtual-clock metrics CSV, step
                       trace, pool digest dump, sampled logits (engine.py:309-313)

Inputs are regenerated from seeds by the tests; outputs are what the reference
produced. These pin both oracle/ (CPU tests) and the CUDA path (GPU tests).
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = os.environ.get("ALORA_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

import aloraserve as ref  # noqa: E402
from aloraserve import bench as ref_bench  # noqa: E402
from aloraserve.metrics import render_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

# C1 of BASELINE.json / SURVEY.md §8(d): 2 layers, d 256, 4 heads, V 256, r 8, B 16
C1 = dict(n_layers=2, n_heads=4, head_dim=64, d_model=256, vocab_size=256, seed=0)


def hash_kats():
    rows = []
    cases = [
        (None, [1, 2, 3], "", 3),
        ("prev", [4, 5, 6], "", 3),
        (None, [1, 2, 3], "adapter0", 3),
        (None, list(range(16)), "", 16),
        (None, [2**32 - 1], "", 1),
        (None, [0] * 4, "ünïcode-key", 4),
    ]
    prev = None
    for parent, toks, key, B in cases:
        p = prev if parent == "prev" else None
        d = ref.hash_block(p, toks, key, B)
        rows.append({"parent": None if p is None else p.hex(), "tokens": toks, "key": key,
                     "block_size": B, "digest": d.hex()})
        prev = d
    rng = np.random.default_rng(1234)
    chains = []
    for i in range(24):
        B = int(rng.choice([1, 3, 4, 8, 16]))
        n = int(rng.integers(1, 200))
        toks = rng.integers(0, 2**31, n).tolist() if i % 3 else rng.integers(0, 256, n).tolist()
        mode = i % 3
        if mode == 0:
            keys = ref.compute_block_keys(toks, B)
            kw = {}
        elif mode == 1:
            keys = ref.compute_block_keys(toks, B, adapter_id=f"ad{i}")
            kw = {"adapter_id": f"ad{i}"}
        else:
            inv = int(rng.integers(0, n + 1))
            keys = ref.compute_block_keys(toks, B, adapter_id=f"ad{i}", inv_start=inv)
            kw = {"adapter_id": f"ad{i}", "inv_start": inv}
        digs, parent = [], None
        for b in range(n // B):
            parent = ref.hash_block(parent, toks[b * B:(b + 1) * B], keys[b], B)
            digs.append(parent.hex())
        chains.append({"tokens": toks, "block_size": B, "keys_kw": kw, "keys": keys, "digests": digs})
    return {"kats": rows, "chains": chains}


def projection_cases():
    out = {}
    for tag, mcfg in (("d64", {}), ("c1", C1)):
        cfg = ref.ModelConfig(**mcfg)
        w = ref.generate_weights(cfg).layers[0]
        rng = np.random.default_rng(7)
        menu = [("q", "k", "v"), ("q", "v"), ("k",), ("q",)]
        for i in range(24):
            n = int(rng.integers(1, 40))
            x = rng.standard_normal((n, cfg.d_model)).astype(np.float32)
            rank = int(rng.choice([4, 8]))
            targets = menu[i % 4]
            ad = ref.generate_adapter(f"a{i % 5}", cfg.d_model, rank, seed=i, targets=targets,
                                      invocation_tokens=(224, 225, 226))
            mode = i % 4
            mask = (np.ones(n, bool) if mode == 0 else np.zeros(n, bool) if mode == 1
                    else rng.random(n) < 0.5)
            use_mask = None if i % 6 == 5 else mask
            q, k, v = ref.project_qkv_masked(x, w, ad, use_mask)
            p = f"{tag}_{i}_"
            out[p + "x"] = x
            out[p + "mask"] = mask
            out[p + "use_mask"] = np.array(use_mask is not None)
            out[p + "meta"] = np.array([rank, i % 5, i, i % 4])
            out[p + "q"], out[p + "k"], out[p + "v"] = q, k, v
    return out


def attention_cases():
    out = {}
    rng = np.random.default_rng(13)
    n_heads, d = 4, 64
    i = 0
    for block_size in (1, 3, 4, 8, 16):
        for total in (1, 2, 5, 17, 33, 64, 130):
            start = int(rng.integers(0, total))
            k_all = rng.standard_normal((total, d)).astype(np.float32)
            v_all = rng.standard_normal((total, d)).astype(np.float32)
            q = rng.standard_normal((total - start, d)).astype(np.float32)
            nb = -(-total // block_size)
            pool = ref.BlockPool(nb + 8, block_size, 1, d)
            ids = list(rng.permutation(nb + 8)[:nb])
            for pos in range(start):
                pool.kv[ids[pos // block_size], 0, 0, pos % block_size] = k_all[pos]
                pool.kv[ids[pos // block_size], 0, 1, pos % block_size] = v_all[pos]
            o = ref.paged_attention(q, pool.kv, 0, ids, k_all[start:], v_all[start:], start, n_heads)
            p = f"a{i}_"
            out[p + "meta"] = np.array([block_size, total, start, nb + 8])
            out[p + "ids"] = np.asarray(ids)
            out[p + "k"], out[p + "v"], out[p + "q"], out[p + "o"] = k_all, v_all, q, o
            i += 1
    return out


def forward_cases():
    """forward_step at C1 dims: whole prefill, chunked continuation, adapter + mask."""
    out = {}
    cfg = ref.ModelConfig(**C1)
    model = ref.Model(cfg)
    rng = np.random.default_rng(21)
    ad = ref.generate_adapter("adapter0", cfg.d_model, 8, seed=0,
                              invocation_tokens=ref.invocation_for(cfg.vocab_size, 0))
    B = 16
    for i in range(6):
        n = int(rng.integers(20, 90))
        toks = rng.integers(0, 224, n).astype(np.int64)
        with_adapter = i % 2 == 1
        if with_adapter:
            toks = np.concatenate([toks, np.asarray(ad.invocation_tokens), rng.integers(0, 224, 3)])
            inv = len(toks) - 6
        nt = len(toks)
        nb = -(-nt // B)
        pool = ref.BlockPool(nb + 4, B, cfg.n_layers, cfg.d_model)
        ids = pool.allocate("r", nb)
        split = int(rng.integers(1, nt - 1))
        logits = []
        for s, e in ((0, split), (split, nt)):
            mask = (np.arange(s, e) < inv) if with_adapter else None
            seq = ref.SeqInput("r", toks[s:e], s, ids, ad if with_adapter else None, mask)
            logits.append(model.forward_step([seq], pool.kv)["r"])
        p = f"f{i}_"
        out[p + "tokens"] = toks
        out[p + "meta"] = np.array([split, int(with_adapter), inv if with_adapter else -1])
        out[p + "ids"] = np.asarray(ids)
        out[p + "logits"] = np.stack(logits)
        out[p + "kv"] = pool.kv[ids]
    return out


PIPELINES = [
    # (name, model dims, spec kwargs, engine kwargs)
    ("c1_bab_alora", C1, dict(pipeline="base_adapter_base", mode="alora", prompt_len=512, gen_len=16,
                              adapter_gen_len=16, batch=4, seed=0), dict(block_size=16, token_budget=2048, pool_blocks=4096)),
    ("c1_bab_lora", C1, dict(pipeline="base_adapter_base", mode="lora", prompt_len=512, gen_len=16,
                             adapter_gen_len=16, batch=4, seed=0), dict(block_size=16, token_budget=2048, pool_blocks=4096)),
    ("d64_multi_alora", {}, dict(pipeline="multi_adapter", mode="alora", prompt_len=37, gen_len=9,
                                 adapter_gen_len=5, n_adapters=3, batch=2, seed=3), dict(block_size=4, token_budget=16, pool_blocks=256)),
    ("d64_adapter_base_alora", {}, dict(pipeline="adapter_base", mode="alora", prompt_len=23, gen_len=7,
                                        adapter_gen_len=4, batch=3, seed=5), dict(block_size=4, token_budget=64, pool_blocks=256)),
    ("d64_ba_lora", {}, dict(pipeline="base_adapter", mode="lora", prompt_len=19, gen_len=6,
                             adapter_gen_len=3, batch=2, seed=8), dict(block_size=3, token_budget=64, pool_blocks=256)),
    ("d64_bab_alora_b8", {}, dict(pipeline="base_adapter_base", mode="alora", prompt_len=30, gen_len=10,
                                  adapter_gen_len=6, batch=2, seed=9), dict(block_size=8, token_budget=7, pool_blocks=64)),
]


def build_engine(model_dims, spec, block_size, token_budget, pool_blocks):
    _, _, n_eval = ref_bench._pipeline_shape(spec)
    mcfg = ref.ModelConfig(**model_dims)
    adapters = tuple(ref.AdapterSpec(adapter_id=f"adapter{k}", rank=8, seed=spec.seed,
                                     invocation_tokens=ref.invocation_for(mcfg.vocab_size, k))
                     for k in range(n_eval))
    cfg = ref.EngineConfig(
        model=mcfg,
        scheduler=ref.SchedulerConfig(token_budget=token_budget,
                                      max_batch_requests=max(8, 2 * spec.batch, n_eval * spec.batch + 2)),
        pool_blocks=pool_blocks, block_size=block_size, adapters=adapters,
        comparison_mode=spec.mode)
    return ref.Engine(cfg, clock=ref.VirtualClock())


def pipeline_runs():
    meta, arrays = {}, {}
    for name, dims, skw, ekw in PIPELINES:
        spec = ref.PipelineSpec(**skw)
        eng = build_engine(dims, spec, **ekw)
        sink = {}
        eng.on_logits = lambda rid, pos, row, sink=sink: sink.__setitem__(f"{rid}@{pos}", row.copy())
        first_tables = {}
        orig = eng.scheduler._cache_lookup

        def spy(req, orig=orig, first_tables=first_tables, eng=eng):
            orig(req)
            bt = eng.pool.block_table(req.request_id)
            first_tables[req.request_id] = {"block_ids": list(bt.block_ids), "reused": list(bt.reused)}
        eng.scheduler._cache_lookup = spy
        res = ref.run_sync_pipeline(spec, engine=eng)
        reqs = {rid: {"prompt": r.prompt.tolist(), "generated": list(map(int, r.generated)),
                      "hit_tokens": r.hit_tokens, "computed_tokens": r.computed_tokens,
                      "adapter": None if r.adapter is None else r.adapter.adapter_id}
                for rid, r in eng.finished.items()}
        meta[name] = {
            "model": dims, "spec": skw, "engine": ekw, "requests": reqs,
            "first_tables": first_tables,
            "metrics_csv": render_csv(res.rows),
            "trace": eng.trace,
            "pool_dump": eng.pool.dump_state(),
            "logit_keys": sorted(sink),
        }
        arrays[name] = np.stack([sink[k] for k in sorted(sink)])
    return meta, arrays


def main():
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "hash_kat.json"), "w") as f:
        json.dump(hash_kats(), f)
    np.savez_compressed(os.path.join(OUT, "projection.npz"), **projection_cases())
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **attention_cases())
    np.savez_compressed(os.path.join(OUT, "forward.npz"), **forward_cases())
    meta, arrays = pipeline_runs()
    with open(os.path.join(OUT, "pipelines.json"), "w") as f:
        json.dump(meta, f)
    np.savez_compressed(os.path.join(OUT, "pipeline_logits.npz"), **arrays)
    # weights fingerprint: numpy's Philox stream must be the same where tests run
    fp = {}
    for tag, dims in (("d64", {}), ("c1", C1)):
        w = ref.generate_weights(ref.ModelConfig(**dims))
        h = hashlib.sha256()
        for L in w.layers:
            for a in (L.wq, L.wk, L.wv, L.wo, L.w_in, L.w_out):
                h.update(a.tobytes())
        h.update(w.embed.tobytes())
        h.update(w.unembed.tobytes())
        fp[tag] = h.hexdigest()
    ad = ref.generate_adapter("adapter0", 256, 8, seed=0, invocation_tokens=(1, 2, 3))
    fp["adapter0_c1"] = hashlib.sha256(b"".join(ad.down[t].tobytes() + ad.up[t].tobytes() for t in "qkv")).hexdigest()
    with open(os.path.join(OUT, "weights_sha256.json"), "w") as f:
        json.dump(fp, f, indent=1)
    for fn in sorted(os.listdir(OUT)):
        print(fn, os.path.getsize(os.path.join(OUT, fn)))


if __name__ == "__main__":
    main()
