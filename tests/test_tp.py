"""Tensor-parallel sharding (tp.py) on CPU: world_size-2 gloo processes vs the unsharded oracle.

Each rank runs the llama-architecture forward of the numpy oracle (fp64 accumulation, the
reference's numerics: model.py:95-98) on ITS shard -- column-parallel q|k|v and gate|up,
row-parallel O and MLP-down, replicated aLoRA down factors and column-sharded up factors --
and all-reduces (gloo) the O-projection and MLP-down partial products before the residual add,
exactly where alora_model_forward calls its tp_allreduce hook. Logits must match the unsharded
oracle forward; the masked aLoRA rows and the GQA head grouping are exercised.
"""

import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2512_17910_b200.adapters import LoraAdapter
from paper_2512_17910_b200.model import ModelConfig
from paper_2512_17910_b200.tp import shard_adapter, shard_config, shard_weights
from paper_2512_17910_b200.weights import BaseWeights, LayerWeights

DIMS = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=4, head_dim=16, d_model=64, ffn_dim=256,
            vocab_size=96, max_seq_len=256, seed=3)


def _oracle(numerics="fp64acc", **over):
    return O.OracleConfig(**{**DIMS, **over}, numerics=numerics)


def _to_base(w) -> BaseWeights:
    layers = [LayerWeights(wq=L["wq"], wk=L["wk"], wv=L["wv"], wo=L["wo"], w_in=L["w_gate"], w_up=L["w_up"],
                           w_out=L["w_down"], attn_norm=L["attn_norm"], mlp_norm=L["mlp_norm"]) for L in w["layers"]]
    return BaseWeights(embed=w["embed"], layers=layers, unembed=None, final_norm=w["final_norm"])


def _from_base(b: BaseWeights) -> dict:
    return {"layers": [{"wq": L.wq, "wk": L.wk, "wv": L.wv, "wo": L.wo, "w_gate": L.w_in, "w_up": L.w_up,
                        "w_down": L.w_out, "attn_norm": L.attn_norm, "mlp_norm": L.mlp_norm} for L in b.layers],
            "embed": b.embed, "final_norm": b.final_norm, "unembed": None}


def _adapter(ocfg):
    oa = O.oracle_adapter("adapter0", ocfg, 4, seed=1, invocation_tokens=(90, 91, 92))
    return LoraAdapter("adapter0", 4, invocation_tokens=oa.invocation_tokens, down=oa.down, up=oa.up)


def tp_forward(scfg, sw, sad, tokens, mask, allreduce):
    """One span from position 0 through the sharded model; partial products are all-reduced in fp64."""
    c = scfg
    cos, sin = O.rope_tables(c.max_seq_len, c.head_dim, c.rope_theta)
    n = len(tokens)
    pos = np.arange(n)
    B = 16
    nb = -(-n // B)
    kv = np.zeros((nb, c.n_layers, 2, B, c.kv_width), np.float32)
    ad = None if sad is None else O.OracleAdapter(sad.adapter_id, sad.rank, sad.mode, sad.targets,
                                                  sad.invocation_tokens, dict(sad.down), dict(sad.up))
    x = sw["embed"][tokens].astype(np.float32)
    for li, L in enumerate(sw["layers"]):
        h = O.rmsnorm(x, L["attn_norm"], c.rms_eps)
        q, k, v = O.project_qkv_masked(h, L["wq"], L["wk"], L["wv"], ad, mask)
        q = O.apply_rope(q, pos, c.n_heads, c.head_dim, cos, sin)
        k = O.apply_rope(k, pos, c.kv_heads, c.head_dim, cos, sin)
        O.write_kv(kv, li, list(range(nb)), 0, k, v)
        attn = O.paged_attention(q, kv, li, list(range(nb)), k, v, 0, c.n_heads, c.kv_heads)
        x = x + allreduce(attn.astype(np.float64) @ L["wo"].astype(np.float64)).astype(np.float32)
        h2 = O.rmsnorm(x, L["mlp_norm"], c.rms_eps)
        g = O.mm(h2, L["w_gate"]).astype(np.float64)
        u = O.mm(h2, L["w_up"]).astype(np.float64)
        a = (g / (1.0 + np.exp(-g)) * u).astype(np.float32)
        x = x + allreduce(a.astype(np.float64) @ L["w_down"].astype(np.float64)).astype(np.float32)
    hf = O.rmsnorm(x[-1:], sw["final_norm"], c.rms_eps)
    return O.mm(hf, sw["embed"].T)[0]


def _reference_logits(tokens, mask):
    ocfg = _oracle()
    om = O.OracleModel(ocfg)
    oad = O.oracle_adapter("adapter0", ocfg, 4, seed=1, invocation_tokens=(90, 91, 92))
    kv = om.new_pool(-(-len(tokens) // 16), 16)
    span = O.OracleSpan("r", tokens, 0, list(range(kv.shape[0])), oad, mask)
    return om.forward_one(span, kv)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = ModelConfig(**DIMS)
        scfg = shard_config(full, world)
        w = O.oracle_weights(_oracle())
        sw = _from_base(shard_weights(_to_base(w), full, world, rank))
        sad = shard_adapter(_adapter(_oracle()), full, world, rank)
        rng = np.random.default_rng(7)
        tokens = np.concatenate([rng.integers(0, 88, 40), [90, 91, 92], rng.integers(0, 88, 5)])
        mask = np.arange(len(tokens)) < 40  # rows before the invocation take the base path exactly

        def allreduce(p):
            t = torch.from_numpy(np.ascontiguousarray(p))
            dist.all_reduce(t)
            return t.numpy()

        ocfg_s = O.OracleConfig(**{**DIMS, "n_heads": scfg.n_heads, "n_kv_heads": scfg.kv_heads,
                                   "ffn_dim": scfg.ffn}, numerics="fp64acc")
        got = tp_forward(ocfg_s, sw, sad, tokens, mask, allreduce)
        if rank == 0:
            want = _reference_logits(tokens, mask)
            q.put(float(np.max(np.abs(got - want))))
            q.put(int(np.argmax(got)) == int(np.argmax(want)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_config_and_weights_partition_the_model():
    full = ModelConfig(**DIMS)
    s2 = shard_config(full, 2)
    assert (s2.n_heads, s2.kv_heads, s2.ffn, s2.d_model) == (4, 2, 128, 64)
    assert shard_config(full, 1) is full
    with pytest.raises(ValueError):
        shard_config(full, 3)  # 8 heads do not split 3 ways
    with pytest.raises(ValueError):
        shard_config(ModelConfig(n_layers=1, n_heads=4, head_dim=16, d_model=64), 2)  # ref arch: no TP
    b = _to_base(O.oracle_weights(_oracle()))
    parts = [shard_weights(b, full, 2, r) for r in range(2)]
    L0 = b.layers[0]
    np.testing.assert_array_equal(np.concatenate([p.layers[0].wq for p in parts], axis=1), L0.wq)
    np.testing.assert_array_equal(np.concatenate([p.layers[0].wk for p in parts], axis=1), L0.wk)
    np.testing.assert_array_equal(np.concatenate([p.layers[0].wo for p in parts], axis=0), L0.wo)
    np.testing.assert_array_equal(np.concatenate([p.layers[0].w_in for p in parts], axis=1), L0.w_in)
    np.testing.assert_array_equal(np.concatenate([p.layers[0].w_out for p in parts], axis=0), L0.w_out)
    assert parts[1].embed is b.embed and parts[1].layers[0].attn_norm is L0.attn_norm  # replicated
    ad = _adapter(_oracle())
    sads = [shard_adapter(ad, full, 2, r) for r in range(2)]
    for t in ad.targets:
        assert sads[0].down[t] is ad.down[t]  # A replicated
        np.testing.assert_array_equal(np.concatenate([s.up[t] for s in sads], axis=1), ad.up[t])  # B sharded


@pytest.mark.timeout(300)
def test_tp2_gloo_forward_matches_unsharded_oracle():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    err = q.get()
    same_argmax = q.get()
    assert err < 1e-5, err
    assert same_argmax
