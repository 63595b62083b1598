"""GPU parity, fp32 tier (fp32 storage, fp64 accumulation = the reference's numerics).

Against the reference's own outputs (tests/golden, made by aloraserve) and
the oracle, through the C ABI. Stated tolerances: logits and
KV within 1e-5 abs; hashes, hit block ids and greedy ids bit-exact. The
GPU-vs-GPU invariance properties the reference pins bitwise
(test_model.py:125-225) are asserted bitwise here too.
"""

import numpy as np
import pytest

from conftest import C1, dense_reference_attention, golden_json, golden_npz, row_projection_oracle
import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2512_17910_b200")


def _frac_equal(a, b):
    return float(np.mean(np.asarray(a) == np.asarray(b)))


def test_projection_vs_reference():
    g = golden_npz("projection.npz")
    menu = [("q", "k", "v"), ("q", "v"), ("k",), ("q",)]
    worst, eq = 0.0, []
    for tag, dims in (("d64", {}), ("c1", C1)):
        cfg = P.ModelConfig(**dims)
        layer = P.generate_weights(cfg).layers[0]
        for i in range(24):
            p = f"{tag}_{i}_"
            rank, aidx, seed, _ = (int(v) for v in g[p + "meta"])
            ad = P.generate_adapter(f"a{aidx}", cfg.d_model, rank, seed=seed, targets=menu[i % 4],
                                    invocation_tokens=(224, 225, 226))
            mask = g[p + "mask"] if bool(g[p + "use_mask"]) else None
            got = P.project_qkv_masked(g[p + "x"], layer, ad, mask)
            for a, b in zip(got, (g[p + "q"], g[p + "k"], g[p + "v"])):
                worst = max(worst, float(np.max(np.abs(a - b) / (np.abs(b) + 1e-6))))
                eq.append(_frac_equal(a, b))
            if mask is not None:  # masked rows are exactly the base projection: row select, not blend
                base = P.project_qkv_masked(g[p + "x"], layer)
                for a, b, t in zip(got, base, "qkv"):
                    np.testing.assert_array_equal(a[mask], b[mask])
                    if t not in ad.targets:
                        np.testing.assert_array_equal(a, b)
    print(f"[parity] projection: max rel err {worst:.3g}, bitwise-equal fraction {np.mean(eq):.6f}")
    assert worst <= 1e-6 and np.mean(eq) >= 0.999


def test_paged_attention_vs_reference_and_dense():
    g = golden_npz("attention.npz")
    worst = 0.0
    i = 0
    while f"a{i}_meta" in g:
        B, total, start, nbp = (int(v) for v in g[f"a{i}_meta"])
        ids = [int(v) for v in g[f"a{i}_ids"]]
        k, v, q = g[f"a{i}_k"], g[f"a{i}_v"], g[f"a{i}_q"]
        kv = np.zeros((nbp, 1, 2, B, 64), np.float32)
        O.write_kv(kv, 0, ids, 0, k[:start], v[:start])
        out = P.paged_attention(q, kv, 0, ids, k[start:], v[start:], start, 4)
        ref = g[f"a{i}_o"]
        worst = max(worst, float(np.max(np.abs(out - ref) / (np.abs(ref) + 1e-7))))
        np.testing.assert_allclose(out, dense_reference_attention(q, k, v, 4, start), rtol=1e-5, atol=1e-6)
        i += 1
    print(f"[parity] paged attention: max rel err vs reference {worst:.3g} over {i} cases")
    assert worst <= 1e-5


def test_paged_attention_short_table_raises():
    q = np.zeros((2, 64), np.float32)
    with pytest.raises(ValueError):
        P.paged_attention(q, np.zeros((4, 1, 2, 4, 64), np.float32), 0, [0], q, q, 4, 4)


def test_kv_write_bitwise():
    import torch
    rng = np.random.default_rng(3)
    for dtype, tdt in (("fp32", torch.float32), ("bf16", torch.bfloat16)):
        pool = P.BlockPool(12, 5, 3, 48, dtype=dtype)
        ref = np.zeros((12, 3, 2, 5, 48), np.float32)
        ids = [7, 2, 9, 0, 11]
        k = rng.standard_normal((17, 48)).astype(np.float32)
        v = rng.standard_normal((17, 48)).astype(np.float32)
        if dtype == "bf16":
            k, v = O.bf16_round(k), O.bf16_round(v)
        P.write_kv(pool.kv, 1, ids, 3, k, v)
        O.write_kv(ref, 1, ids, 3, k, v)
        np.testing.assert_array_equal(pool.kv.float().cpu().numpy(), ref)


def test_forward_vs_reference():
    g = golden_npz("forward.npz")
    cfg = P.ModelConfig(**C1)
    model = P.Model(cfg)
    ad = P.generate_adapter("adapter0", 256, 8, invocation_tokens=(224, 225, 226))
    worst_l = worst_kv = 0.0
    eq = []
    for i in range(6):
        toks = g[f"f{i}_tokens"]
        split, with_ad, inv = (int(v) for v in g[f"f{i}_meta"])
        ids = [int(v) for v in g[f"f{i}_ids"]]
        pool = P.BlockPool(max(ids) + 1, 16, 2, 256)
        logits = []
        for s, e in ((0, split), (split, len(toks))):
            mask = (np.arange(s, e) < inv) if with_ad else None
            logits.append(model.forward_step([P.SeqInput("r", toks[s:e], s, ids, ad if with_ad else None, mask)],
                                             pool.kv)["r"])
        kv = pool.kv[ids].cpu().numpy()
        worst_l = max(worst_l, float(np.max(np.abs(np.stack(logits) - g[f"f{i}_logits"]))))
        worst_kv = max(worst_kv, float(np.max(np.abs(kv - g[f"f{i}_kv"]))))
        eq.append(_frac_equal(kv, g[f"f{i}_kv"]))
    print(f"[parity] forward: max |dlogit| {worst_l:.3g}, max |dKV| {worst_kv:.3g}, KV bitwise fraction {np.mean(eq):.6f}")
    assert worst_l <= 1e-5 and worst_kv <= 1e-5


def _gpu_engine(g):
    spec = P.PipelineSpec(**g["spec"])
    return spec, P.build_engine(spec, model=P.ModelConfig(**g["model"]), **g["engine"])


@pytest.mark.parametrize("name", ["c1_bab_alora", "c1_bab_lora", "d64_multi_alora", "d64_adapter_base_alora",
                                  "d64_ba_lora", "d64_bab_alora_b8"])
def test_pipeline_parity_with_reference(name):
    g = golden_json("pipelines.json")[name]
    logits = golden_npz("pipeline_logits.npz")[name]
    spec, eng = _gpu_engine(g)
    sink = {}
    eng.on_logits = lambda rid, pos, row: sink.__setitem__(f"{rid}@{pos}", np.array(row, copy=True))
    tables = {}
    orig = eng.scheduler._lookup_done

    def spy(req, hits):
        orig(req, hits)
        tables[req.request_id] = {"block_ids": [int(b) for b in hits], "reused": [True] * len(hits)}

    eng.scheduler._lookup_done = spy
    rows = P.run_sync_pipeline(spec, eng)
    n_tok = 0
    for rid, r in g["requests"].items():
        mine = eng.finished[rid]
        assert list(map(int, mine.generated)) == r["generated"], rid  # greedy ids bit-exact
        assert (mine.hit_tokens, mine.computed_tokens) == (r["hit_tokens"], r["computed_tokens"]), rid
        n_tok += len(r["generated"])
    assert tables == g["first_tables"]  # cache-hit block indices bit-exact
    assert eng.pool.dump_state() == g["pool_dump"]  # block digests bit-exact
    assert P.render_csv(rows) == g["metrics_csv"]  # virtual-clock metrics byte-identical
    assert eng.trace == g["trace"]
    got = np.stack([sink[k] for k in sorted(sink)])
    assert sorted(sink) == g["logit_keys"]
    err = float(np.max(np.abs(got - logits)))
    print(f"[parity] pipeline {name}: {len(g['requests'])} requests, {n_tok} greedy ids exact, "
          f"max |dlogit| {err:.3g}, logits bitwise fraction {_frac_equal(got, logits):.6f}")
    assert err <= 1e-5


# --------------------------------------------- GPU-vs-GPU invariances (bitwise)
def _run(model, pool, rid, toks, adapter=None, mask=None, start=0, ids=None):
    ids = ids if ids is not None else pool.allocate(rid, -(-len(toks) // pool.block_size))
    out = model.forward_step([P.SeqInput(rid, toks, start, ids, adapter, mask)], pool.kv)[rid]
    return ids, out


@pytest.mark.parametrize("dtype", ["fp32"])
def test_batch_independence_and_chunking_bitwise(dtype):
    model = P.Model(P.ModelConfig(dtype=dtype))
    rng = np.random.default_rng(11)
    toks = [rng.integers(0, 200, n) for n in (5, 9, 13)]
    pool = P.BlockPool(32, 4, 2, 64, dtype=dtype)
    seqs = [P.SeqInput(f"r{i}", t, 0, pool.allocate(f"r{i}", -(-len(t) // 4))) for i, t in enumerate(toks)]
    batch = model.forward_step(seqs, pool.kv)
    for i, t in enumerate(toks):
        solo_pool = P.BlockPool(32, 4, 2, 64, dtype=dtype)
        _, solo = _run(model, solo_pool, "s", t)
        np.testing.assert_array_equal(batch[f"r{i}"], solo)
    t = rng.integers(0, 200, 11)
    pw = P.BlockPool(16, 4, 2, 64, dtype=dtype)
    ids_w, whole = _run(model, pw, "w", t)
    pc = P.BlockPool(16, 4, 2, 64, dtype=dtype)
    ids_c = pc.allocate("c", 3)
    for s, e in ((0, 4), (4, 8), (8, 11)):
        _, out = _run(model, pc, "c", t[s:e], start=s, ids=ids_c)
    np.testing.assert_array_equal(out, whole)
    np.testing.assert_array_equal(pw.kv[ids_w].cpu().numpy(), pc.kv[ids_c].cpu().numpy())


def test_placement_invariance_bitwise():
    model = P.Model(P.ModelConfig())
    rng = np.random.default_rng(9)
    t = rng.integers(0, 200, 13)
    outs = []
    for ids in ([0, 1, 2, 3], [7, 2, 5, 0]):
        pool = P.BlockPool(8, 4, 2, 64)
        _, o = _run(model, pool, "r", t[:10], ids=ids)
        _, o = _run(model, pool, "r", t[10:], start=10, ids=ids)
        outs.append(o)
    np.testing.assert_array_equal(outs[0], outs[1])


def test_pre_invocation_kv_identical_to_base():
    model = P.Model(P.ModelConfig())
    rng = np.random.default_rng(13)
    inv_start = 9
    toks = np.concatenate([rng.integers(0, 200, inv_start), [224, 225, 226], rng.integers(0, 200, 4)])
    ad = P.generate_adapter("a", 64, 8, invocation_tokens=(224, 225, 226))
    mask = np.arange(len(toks)) < inv_start
    pb = P.BlockPool(16, 4, 2, 64)
    ids_b, _ = _run(model, pb, "b", toks)
    pa = P.BlockPool(16, 4, 2, 64)
    ids_a, _ = _run(model, pa, "a", toks, ad, mask)
    kb, ka = pb.kv.cpu().numpy(), pa.kv.cpu().numpy()
    for pos in range(len(toks)):
        rb, ra = kb[ids_b[pos // 4], :, :, pos % 4], ka[ids_a[pos // 4], :, :, pos % 4]
        if pos < inv_start:
            np.testing.assert_array_equal(ra, rb)
        else:
            assert not np.array_equal(ra, rb)


def test_missing_mask_and_bad_pool_raise():
    model = P.Model(P.ModelConfig())
    ad = P.generate_adapter("a", 64, 8, invocation_tokens=(1, 2))
    pool = P.BlockPool(8, 4, 2, 64)
    ids = pool.allocate("r", 1)
    with pytest.raises(ValueError):
        model.forward_step([P.SeqInput("r", np.arange(3), 0, ids, ad, None)], pool.kv)
    with pytest.raises(ValueError):
        model.forward_step([P.SeqInput("r", np.arange(5), 0, ids)], pool.kv)  # short block table
    with pytest.raises(ValueError):
        model.forward_step([P.SeqInput("r", np.zeros(0, int), 0, ids)], pool.kv)


def test_greedy_next_token_device():
    assert P.greedy_next_token(np.array([0.0, 2.0, 1.0])) == 1
    assert P.greedy_next_token(np.array([3.0, 3.0, 1.0])) == 0
    with pytest.raises(ValueError):
        P.greedy_next_token(np.zeros((2, 2)))


def test_caching_on_off_identical_logits():
    """test_acceptance.py:234-280 on the GPU: prefix caching changes no sampled logit (bitwise here)."""
    rng = np.random.default_rng(5)
    for i in range(4):
        kind = ("base_adapter", "adapter_base", "base_adapter_base", "multi_adapter")[i]
        spec = P.PipelineSpec(pipeline=kind, mode="alora" if i % 3 else "lora", prompt_len=int(rng.integers(4, 28)),
                              gen_len=int(rng.integers(2, 12)), adapter_gen_len=int(rng.integers(1, 6)),
                              n_adapters=2 if kind == "multi_adapter" else 1, batch=1 + i % 2, seed=i)
        sinks = []
        for caching in (True, False):
            eng = P.build_engine(spec, pool_blocks=256, block_size=(1, 3, 4, 8)[i], token_budget=16 if i % 2 else 64,
                                 prefix_caching=caching)
            sink = {}
            eng.on_logits = lambda rid, pos, row, sink=sink: sink.__setitem__((rid, pos), np.array(row, copy=True))
            P.run_sync_pipeline(spec, eng)
            sinks.append(sink)
        assert sinks[0].keys() == sinks[1].keys()
        for k in sinks[0]:
            np.testing.assert_array_equal(sinks[0][k], sinks[1][k])
