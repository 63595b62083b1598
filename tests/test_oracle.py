"""The oracle is pinned to the reference's own outputs before anything is checked against it.

Every fixture in tests/golden/ was produced by the reference package
(oracle/gen_golden.py). CPU only.
"""

import hashlib

import numpy as np
import pytest

from conftest import C1, dense_reference_attention, golden_json, golden_npz, row_projection_oracle
import oracle
from oracle import (OracleAdapter, OracleConfig, OracleModel, OracleSpan, bf16_round, chain_digests,
                    compute_block_keys, hash_block, oracle_adapter, oracle_weights, paged_attention,
                    project_qkv_masked)


def test_survey_known_answers():
    # SURVEY.md §8(c) table
    d1 = hash_block(None, [1, 2, 3], "", 3)
    assert d1.hex() == "cd6be95bcd95f1b55f63550e61534745"
    assert hash_block(d1, [4, 5, 6], "", 3).hex() == "8761716004a7d48ad5860f38f70de7f2"
    assert hash_block(None, [1, 2, 3], "adapter0", 3).hex() == "7a754e2b867f6a8450defdbdd26ae47e"
    assert hash_block(None, range(16), "", 16).hex() == "6eaeacca54ca17bf8e9087566a8b92cc"
    assert hash_block(None, [2**32 - 1], "", 1).hex() == "7d5cd7100b6c60d7bab50071f260cb71"


def test_hash_kats_and_chains_match_reference():
    g = golden_json("hash_kat.json")
    for row in g["kats"]:
        parent = None if row["parent"] is None else bytes.fromhex(row["parent"])
        assert hash_block(parent, row["tokens"], row["key"], row["block_size"]).hex() == row["digest"]
    for ch in g["chains"]:
        keys = compute_block_keys(ch["tokens"], ch["block_size"], **ch["keys_kw"])
        assert keys == ch["keys"]
        assert [d.hex() for d in chain_digests(ch["tokens"], keys, ch["block_size"])] == ch["digests"]


def test_hash_errors():
    with pytest.raises(ValueError):
        hash_block(None, [1, 2], "", 3)
    with pytest.raises(ValueError):
        hash_block(b"short", [1, 2, 3], "", 3)
    with pytest.raises(ValueError):
        hash_block(None, [2**32], "", 1)
    with pytest.raises(ValueError):
        compute_block_keys([1, 2], 2, inv_start=1)
    with pytest.raises(ValueError):
        compute_block_keys([1, 2], 2, adapter_id="a", inv_start=5)


def test_weights_fingerprint_matches_reference():
    fp = golden_json("weights_sha256.json")
    for tag, dims in (("d64", {}), ("c1", C1)):
        w = oracle_weights(OracleConfig(**dims))
        h = hashlib.sha256()
        for L in w["layers"]:
            for k in ("wq", "wk", "wv", "wo", "w_in", "w_out"):
                h.update(L[k].tobytes())
        h.update(w["embed"].tobytes())
        h.update(w["unembed"].tobytes())
        assert h.hexdigest() == fp[tag], tag
    ad = oracle_adapter("adapter0", OracleConfig(**C1), 8, seed=0, invocation_tokens=(1, 2, 3))
    blob = b"".join(ad.down[t].tobytes() + ad.up[t].tobytes() for t in "qkv")
    assert hashlib.sha256(blob).hexdigest() == fp["adapter0_c1"]


def _proj_cases():
    g = golden_npz("projection.npz")
    menu = [("q", "k", "v"), ("q", "v"), ("k",), ("q",)]
    for tag, dims in (("d64", {}), ("c1", C1)):
        cfg = OracleConfig(**dims)
        layer = oracle_weights(cfg)["layers"][0]
        for i in range(24):
            p = f"{tag}_{i}_"
            rank, aidx, seed, _ = g[p + "meta"]
            ad = oracle_adapter(f"a{aidx}", cfg, int(rank), seed=int(seed), targets=menu[i % 4],
                                invocation_tokens=(224, 225, 226))
            use_mask = bool(g[p + "use_mask"])
            yield cfg, layer, ad, g[p + "x"], g[p + "mask"], use_mask, (g[p + "q"], g[p + "k"], g[p + "v"])


def test_projection_bitwise_vs_reference():
    n = 0
    for cfg, layer, ad, x, mask, use_mask, want in _proj_cases():
        got = project_qkv_masked(x, layer["wq"], layer["wk"], layer["wv"], ad, mask if use_mask else None)
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)
        if use_mask:
            for t, mat, a in zip("qkv", (layer["wq"], layer["wk"], layer["wv"]), got):
                np.testing.assert_array_equal(a, row_projection_oracle(x, mat, ad, t, mask))
        n += 1
    assert n == 48


def test_attention_vs_reference_and_dense():
    g = golden_npz("attention.npz")
    i = 0
    while f"a{i}_meta" in g:
        B, total, start, nbp = (int(v) for v in g[f"a{i}_meta"])
        ids = [int(v) for v in g[f"a{i}_ids"]]
        k, v, q = g[f"a{i}_k"], g[f"a{i}_v"], g[f"a{i}_q"]
        kv = np.zeros((nbp, 1, 2, B, 64), np.float32)
        oracle.write_kv(kv, 0, ids, 0, k[:start], v[:start])
        out = paged_attention(q, kv, 0, ids, k[start:], v[start:], start, 4)
        np.testing.assert_array_equal(out, g[f"a{i}_o"])
        np.testing.assert_allclose(out, dense_reference_attention(q, k, v, 4, start), rtol=1e-5, atol=1e-6)
        i += 1
    assert i == 35


def test_gqa_attention_matches_dense():
    rng = np.random.default_rng(0)
    for B in (4, 16):
        total, start, H, Hkv, D = 45, 30, 8, 2, 16
        k = rng.standard_normal((total, Hkv * D)).astype(np.float32)
        v = rng.standard_normal((total, Hkv * D)).astype(np.float32)
        q = rng.standard_normal((total - start, H * D)).astype(np.float32)
        nb = -(-total // B)
        kv = np.zeros((nb, 1, 2, B, Hkv * D), np.float32)
        ids = list(range(nb))
        oracle.write_kv(kv, 0, ids, 0, k[:start], v[:start])
        out = paged_attention(q, kv, 0, ids, k[start:], v[start:], start, H, Hkv)
        np.testing.assert_allclose(out, dense_reference_attention(q, k, v, H, start, Hkv), rtol=1e-5, atol=1e-6)


def test_forward_bitwise_vs_reference():
    g = golden_npz("forward.npz")
    cfg = OracleConfig(**C1)
    model = OracleModel(cfg)
    ad = oracle_adapter("adapter0", cfg, 8, seed=0, invocation_tokens=(224, 225, 226))
    for i in range(6):
        toks = g[f"f{i}_tokens"]
        split, with_ad, inv = (int(v) for v in g[f"f{i}_meta"])
        ids = [int(v) for v in g[f"f{i}_ids"]]
        kv = model.new_pool(max(ids) + 1, 16)
        logits = []
        for s, e in ((0, split), (split, len(toks))):
            mask = (np.arange(s, e) < inv) if with_ad else None
            span = OracleSpan("r", toks[s:e], s, ids, ad if with_ad else None, mask)
            logits.append(model.forward_step([span], kv)["r"])
        np.testing.assert_array_equal(np.stack(logits), g[f"f{i}_logits"])
        np.testing.assert_array_equal(kv[ids], g[f"f{i}_kv"])


def test_bf16_round():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e38, 1e-40], np.float32)
    r = bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0078125)
    assert r[3] == -2.5
    import torch
    t = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(r, t)


def test_llama_oracle_chunked_equals_whole_and_gqa_shapes():
    cfg = OracleConfig(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=16, d_model=96,
                       ffn_dim=160, vocab_size=300, numerics="bf16")
    m = OracleModel(cfg)
    rng = np.random.default_rng(3)
    toks = rng.integers(0, 290, 23)
    kv1 = m.new_pool(8, 4)
    whole = m.forward_step([OracleSpan("r", toks, 0, list(range(6)))], kv1)["r"]
    kv2 = m.new_pool(8, 4)
    m.forward_step([OracleSpan("r", toks[:10], 0, list(range(6)))], kv2)
    part = m.forward_step([OracleSpan("r", toks[10:], 10, list(range(6)))], kv2)["r"]
    # the oracle accumulates in fp64 per row: chunking changes nothing beyond fp64 noise
    np.testing.assert_allclose(part, whole, rtol=1e-5, atol=1e-5)
    np.testing.assert_array_equal(kv1[:6, :, :, :, :], kv2[:6])
    assert kv1.shape[-1] == 32


def test_oracle_gqa_attention_matches_per_head_dense():
    """The oracle's batched GQA attention (llama mode) equals the per-head dense fp64 reference."""
    from conftest import dense_reference_attention
    rng = np.random.default_rng(5)
    H, Hkv, D, B, start, n = 8, 2, 16, 4, 13, 6
    total = start + n
    nb = -(-total // B)
    kv = rng.standard_normal((nb + 2, 1, 2, B, Hkv * D)).astype(np.float32)
    ids = list(rng.permutation(nb + 2)[:nb])
    k = rng.standard_normal((n, Hkv * D)).astype(np.float32)
    v = rng.standard_normal((n, Hkv * D)).astype(np.float32)
    q = rng.standard_normal((n, H * D)).astype(np.float32)
    import oracle as O
    got = O.paged_attention(q, kv, 0, ids, k, v, start, H, Hkv)
    pos = np.arange(start)
    kc = np.concatenate([kv[np.asarray(ids)[pos // B], 0, 0, pos % B], k])
    vc = np.concatenate([kv[np.asarray(ids)[pos // B], 0, 1, pos % B], v])
    want = dense_reference_attention(q, kc, vc, H, start, Hkv)
    assert np.max(np.abs(got - want)) < 1e-6
