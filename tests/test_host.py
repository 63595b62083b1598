"""Host-side logic of the drop-in, on CPU: native hashing, BlockPool, scheduler, engine.

The engine is driven with the CPU oracle model (tests only) and a host
storage pool, and must reproduce the reference's own pipeline runs
(tests/golden/pipelines.json, produced by aloraserve) exactly: generated ids,
cache hits, first block tables, virtual-clock metrics CSV, step trace, pool
digests and every sampled logits row.
"""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_json, golden_npz
import oracle as O
import paper_2512_17910_b200 as P
from paper_2512_17910_b200 import _native


# ------------------------------------------------------------------ C ABI ---
def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "alora_sm100a.h")).read()
    declared = set(re.findall(r"\b(alora_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    for name in declared:
        assert hasattr(_native.lib, name)
    assert "sm_100a" in P.native_version()


def test_tp_symmetric_buffer_layout():
    # flags + epochs, two partial slots, and two (call-parity) sets of reduced x (fp32) / h (bf16) rows
    for T, d in ((16, 64), (300, 4096), (8192, 8192)):
        total = _native.lib.alora_tp_buffer_bytes(T, d)
        p0, p1 = (_native.lib.alora_tp_partial_offset(T, d, s) for s in (0, 1))
        assert 0 < p0 < p1 and p1 - p0 >= T * d * 4
        assert _native.lib.alora_tp_partial_offset(T, d, 2) == p0  # slots alternate by call parity
        assert total - (p1 + T * d * 4) >= 2 * (T * d * 4 + T * d * 2)
    assert _native.lib.alora_tp_buffer_bytes(0, 64) == _native.ALORA_EINVAL


def test_native_hash_matches_reference_kats_and_chains():
    g = golden_json("hash_kat.json")
    for row in g["kats"]:
        parent = None if row["parent"] is None else bytes.fromhex(row["parent"])
        assert P.hash_block(parent, row["tokens"], row["key"], row["block_size"]).hex() == row["digest"]
    for ch in g["chains"]:
        keys = P.compute_block_keys(ch["tokens"], ch["block_size"], **ch["keys_kw"])
        assert keys == ch["keys"]
        n = len(ch["tokens"]) // ch["block_size"]
        assert [d.hex() for d in P.hash_chain(ch["tokens"], n, ch["block_size"], keys)] == ch["digests"]


def test_native_hash_long_keys_and_multiblock_messages():
    rng = np.random.default_rng(5)
    for B in (1, 7, 16, 31, 32, 33, 64, 100):  # messages straddling 128-byte compression blocks
        for key in ("", "k", "x" * 200, "adapter-ü"):
            toks = rng.integers(0, 2**32, B, dtype=np.uint64).tolist()
            parent = bytes(rng.integers(0, 256, 16, dtype=np.uint8))
            for p in (None, parent):
                assert P.hash_block(p, toks, key, B) == O.hash_block(p, toks, key, B)


def test_batched_chains_and_commit_digest_reuse_match_oracle():
    from paper_2512_17910_b200 import kv_cache as K

    rng = np.random.default_rng(11)
    B = 16
    chains = []
    for n_tok, split in ((4096, 100), (17, 0), (15, 0), (700, 30), (2052, 128)):
        toks = rng.integers(0, 2**32, n_tok, dtype=np.uint64).astype(np.int64)
        nb = -(-n_tok // B)
        chains.append((toks, n_tok // B, [""] * split + ["adapter0"] * (nb - split)))
    got = K.hash_chains(chains, B, n_threads=4)
    for (toks, n, keys), dg in zip(chains, got):
        want, parent = [], None
        for i in range(n):
            parent = O.hash_block(parent, toks[i * B:(i + 1) * B].tolist(), keys[i], B)
            want.append(parent)
        assert dg == want
    # the scheduler's batched admission hashing (two-run keys) equals the per-request chain
    items, want = [], []
    for n_tok, adapter, inv in ((2052, None, None), (33, "std", None), (2052, "act", 2040), (48, "act", 32),
                                (47, "act", 0), (17, "act", 17), (5, None, None)):
        toks = rng.integers(0, 2**32, n_tok, dtype=np.uint64).astype(np.int64)
        keys = P.compute_block_keys(toks, B, adapter_id=adapter, inv_start=inv)
        n = max(0, (n_tok - 1) // B)
        n_base = n if adapter is None else (0 if inv is None else min(-(-n_tok // B), inv // B))
        items.append((toks, n, n_base, adapter or ""))
        want.append(b"".join(P.hash_chain(toks, n, B, keys)))
    # requests sharing their base-key region (one conversation, several adapters) share its digests
    conv = rng.integers(0, 2**32, 200, dtype=np.uint64).astype(np.int64)
    for k, (tail, adapter, inv) in enumerate(((7, "act", 200), (9, "act2", 200), (7, "act", 193), (5, None, None),
                                              (12, "std", None), (7, "act", 200))):
        toks = np.concatenate([conv, rng.integers(0, 2**32, tail, dtype=np.uint64).astype(np.int64)])
        if k == 5:
            toks[3] += 1  # same n_base, different base tokens
        keys = P.compute_block_keys(toks, B, adapter_id=adapter if adapter != "std" else "std", inv_start=inv)
        n = max(0, (len(toks) - 1) // B)
        n_base = n if adapter is None else (0 if inv is None else min(-(-len(toks) // B), inv // B))
        items.append((toks, n, n_base, adapter or ""))
        want.append(b"".join(P.hash_chain(toks, n, B, keys)))
    assert K.hash_requests(items, B, n_threads=3) == want
    assert K.hash_requests(items, B, n_threads=1) == want
    with pytest.raises(ValueError):
        K.hash_requests([(np.array([-1] * 32), 2, 2, "")], B)
    # commit_and_free reuses the admission chain for the unchanged prefix and hashes the rest
    pool = P.BlockPool(64, B, 1, 8, storage="numpy")
    prompt = rng.integers(0, 1000, 70)
    keys = P.compute_block_keys(prompt, B)
    pool.find_cached_prefix("r", prompt, keys)
    pool.allocate("r", 5)
    seq = np.concatenate([prompt, rng.integers(0, 1000, 10)])
    pool.set_fill("r", len(seq))
    pool.commit_and_free("r", seq, P.compute_block_keys(seq, B))
    ref = P.hash_chain(seq, len(seq) // B, B, P.compute_block_keys(seq, B))
    assert [pool.blocks[pool._index[d]].hash for d in ref] == ref
    pool.check_conservation()


def test_hash_validation_errors():
    with pytest.raises(ValueError):
        P.hash_block(None, [1, 2], "", 3)
    with pytest.raises(ValueError):
        P.hash_block(b"short", [1, 2, 3], "", 3)
    with pytest.raises(ValueError):
        P.hash_block(None, [2**32], "", 1)
    with pytest.raises(ValueError):
        P.compute_block_keys([1, 2], 2, inv_start=1)
    with pytest.raises(ValueError):
        P.compute_block_keys([1, 2], 2, adapter_id="a", inv_start=5)


def test_block_keys_match_oracle_exhaustively():
    for B in (1, 2, 3, 4, 16):
        for n in range(0, 40):
            seq = list(range(n))
            assert P.compute_block_keys(seq, B) == O.compute_block_keys(seq, B)
            assert P.compute_block_keys(seq, B, adapter_id="a") == O.compute_block_keys(seq, B, adapter_id="a")
            for inv in range(0, n + 1):
                assert P.compute_block_keys(seq, B, "a", inv) == O.compute_block_keys(seq, B, "a", inv)


# -------------------------------------------------------------- BlockPool ---
def make_pool(total=16, B=4):
    return P.BlockPool(total, B, n_layers=1, d_model=8, storage="numpy")


def commit_seq(pool, rid, tokens, keys=None):
    B = pool.block_size
    keys = keys if keys is not None else [""] * (-(-len(tokens) // B))
    ids, hit = pool.find_cached_prefix(rid, tokens, keys)
    pool.allocate(rid, -(-len(tokens) // B) - len(ids))
    pool.set_fill(rid, len(tokens))
    pool.commit_and_free(rid, tokens, keys)
    return hit


def test_pool_reuse_law_and_last_token_rule():
    pool = make_pool()
    toks = list(range(10))
    assert commit_seq(pool, "a", toks) == 0
    assert commit_seq(pool, "b", toks) == 8
    pool2 = make_pool()
    commit_seq(pool2, "a", list(range(8)))
    ids, hit = pool2.find_cached_prefix("b", list(range(8)), ["", ""])
    assert hit == 4 and len(ids) == 1  # aligned prompt: last token always computed
    pool2.release("b")
    pool.check_conservation()
    pool2.check_conservation()


def test_pool_lru_eviction_tail_first_and_exhaustion():
    pool = make_pool(total=4, B=2)
    commit_seq(pool, "a", [1, 2, 3, 4, 5, 6])  # 3 blocks, released tail first
    order = list(pool._free)
    assert order[-1] == 0  # chain head released last = evicted last
    with pytest.raises(P.PoolExhaustedError):
        pool.allocate("x", 5)
    assert pool.num_free == 4  # atomic
    got = pool.allocate("x", 2)
    assert 0 not in got
    pool.release("x")
    pool.check_conservation()


def test_pool_last_writer_wins_and_refcount_pinning():
    pool = make_pool()
    commit_seq(pool, "a", list(range(9)))
    commit_seq(pool, "b", list(range(9)))  # same digests re-committed by b's fresh tail
    d = P.hash_block(None, [0, 1, 2, 3], "", 4)
    assert d in pool._index
    ids1, _ = pool.find_cached_prefix("r1", list(range(9)), ["", "", ""])
    ids2, _ = pool.find_cached_prefix("r2", list(range(9)), ["", "", ""])
    assert ids1 == ids2 and pool.blocks[ids1[0]].ref_count == 2
    pool.release("r1")
    pool.release("r2")
    pool.check_conservation()


def test_pool_random_walk_conservation():
    rng = np.random.default_rng(0)
    pool = make_pool(total=24, B=3)
    live = {}
    for step in range(300):
        if live and rng.random() < 0.5:
            rid = list(live)[int(rng.integers(len(live)))]
            toks = live.pop(rid)
            if rng.random() < 0.5:
                pool.set_fill(rid, len(toks))
                pool.commit_and_free(rid, toks, [""] * (-(-len(toks) // 3)))
            else:
                pool.release(rid)
        else:
            rid = f"r{step}"
            toks = rng.integers(0, 5, int(rng.integers(1, 12))).tolist()
            ids, _ = pool.find_cached_prefix(rid, toks, [""] * (-(-len(toks) // 3)))
            try:
                pool.allocate(rid, -(-len(toks) // 3) - len(ids))
                live[rid] = toks
            except P.PoolExhaustedError:
                pool.release(rid)
        pool.check_conservation()


# ----------------------------------------------------------------- engine ---
def detect_cases():
    assert P.detect_invocation([9, 8, 7, 1, 2, 3], [1, 2, 3]) == 3
    assert P.detect_invocation([1, 2, 3, 0, 1, 2, 3], [1, 2, 3]) == 4
    assert P.detect_invocation([4, 5], [4, 5]) == 0


def test_detect_invocation():
    detect_cases()
    with pytest.raises(P.InvocationNotFoundError):
        P.detect_invocation([1, 2, 3], [7, 8])
    with pytest.raises(P.InvocationNotFoundError):
        P.detect_invocation([1], [1, 2])
    with pytest.raises(ValueError):
        P.detect_invocation([1, 2], [])
    rng = np.random.default_rng(1)
    for i in range(400):
        # short prompts (one window) and long ones (> 512 tokens: the 256-token tail window, then the whole prompt)
        n = int(rng.integers(1, 20)) if i % 2 else int(rng.integers(500, 1200))
        p = rng.integers(-1, 3, n) if i % 3 == 0 else rng.integers(0, 3 if n < 20 else 6, n)
        inv = rng.integers(0, 3, int(rng.integers(1, 4 if n < 20 else 6)))
        try:
            want = O.detect_invocation(p, inv)
        except ValueError:
            with pytest.raises(P.InvocationNotFoundError):
                P.detect_invocation(p, inv)
            continue
        assert P.detect_invocation(p, inv) == want


def oracle_engine(dims, spec, block_size, token_budget, pool_blocks):
    model = O.OracleModel(O.OracleConfig(**dims))
    return P.build_engine(spec, model=P.ModelConfig(**dims), pool_blocks=pool_blocks, block_size=block_size,
                          token_budget=token_budget, engine_model=model, pool_storage="numpy")


def _run_golden(name):
    g = golden_json("pipelines.json")[name]
    logits = golden_npz("pipeline_logits.npz")[name]
    spec = P.PipelineSpec(**g["spec"])
    eng = oracle_engine(g["model"], spec, **g["engine"])
    sink = {}
    eng.on_logits = lambda rid, pos, row: sink.__setitem__(f"{rid}@{pos}", np.array(row, copy=True))
    tables = {}
    orig = eng.scheduler._lookup_done

    def spy(req, hits):
        orig(req, hits)
        tables[req.request_id] = {"block_ids": [int(b) for b in hits], "reused": [True] * len(hits)}

    eng.scheduler._lookup_done = spy
    rows = P.run_sync_pipeline(spec, eng)
    return g, logits, eng, rows, sink, tables


@pytest.mark.parametrize("name", ["d64_multi_alora", "d64_adapter_base_alora", "d64_ba_lora", "d64_bab_alora_b8",
                                  "c1_bab_alora"])
def test_engine_reproduces_reference_pipeline(name):
    g, logits, eng, rows, sink, tables = _run_golden(name)
    for rid, r in g["requests"].items():
        mine = eng.finished[rid]
        assert mine.prompt.tolist() == r["prompt"], rid
        assert list(map(int, mine.generated)) == r["generated"], rid
        assert (mine.hit_tokens, mine.computed_tokens) == (r["hit_tokens"], r["computed_tokens"]), rid
    assert tables == g["first_tables"]
    assert P.render_csv(rows) == g["metrics_csv"]
    assert eng.trace == g["trace"]
    assert eng.pool.dump_state() == g["pool_dump"]
    assert sorted(sink) == g["logit_keys"]
    np.testing.assert_array_equal(np.stack([sink[k] for k in sorted(sink)]), logits)


def test_submit_validation():
    spec = P.PipelineSpec()
    eng = oracle_engine({}, spec, 4, 64, 128)
    with pytest.raises(ValueError):
        eng.submit(np.zeros(0, dtype=np.int64))
    with pytest.raises(ValueError):
        eng.submit(np.zeros((2, 3), dtype=np.int64))
    with pytest.raises(ValueError):
        eng.submit([1, 2], max_new_tokens=0)
    with pytest.raises(ValueError, match=r"\[0, 256\), got \[1, 256\]"):
        eng.submit([1, 256])
    with pytest.raises(ValueError, match=r"got \[-1, 5\]"):  # negative ids wrap to >= 2**63 in the range check
        eng.submit([5, -1])
    with pytest.raises(ValueError):
        eng.submit(np.array([3, -(2 ** 63)], dtype=np.int64))
    # the native core reuses retired requests' token buffers: a shorter prompt after a longer one is intact
    a = eng.submit(list(range(1, 40)), max_new_tokens=1)
    eng.run_until_idle()
    b = eng.submit([7, 8, 9], max_new_tokens=1)
    eng.run_until_idle()
    assert list(eng.finished[a].prompt) == list(range(1, 40)) and list(eng.finished[b].prompt) == [7, 8, 9]
    with pytest.raises(ValueError):
        eng.submit([1] * 100, max_new_tokens=8093)
    with pytest.raises(ValueError):
        eng.submit([1, 2], adapter_id="nope")
    with pytest.raises(P.InvocationNotFoundError):
        eng.submit([1, 2, 3], adapter_id="adapter0")
    small = oracle_engine({}, spec, 4, 64, 2)
    with pytest.raises(ValueError, match="cannot ever fit"):
        small.submit([1] * 12, max_new_tokens=1)


def test_activation_mask_layout():
    spec = P.PipelineSpec()
    eng = oracle_engine({}, spec, 4, 64, 128)
    inv = list(eng.adapters["adapter0"].invocation_tokens)
    eng.submit(np.asarray([5, 6] + inv), adapter_id="adapter0", max_new_tokens=1, request_id="a")
    eng.submit(np.asarray([9, 9, 9]), max_new_tokens=1, request_id="b")
    ra, rb = eng.scheduler.requests["a"], eng.scheduler.requests["b"]
    mask = P.build_activation_mask([P.ScheduledSpan(ra, 0, 5, "prefill"), P.ScheduledSpan(rb, 1, 3, "prefill")])
    assert mask.values.tolist() == [True, True, False, False, False, True, True]
    assert mask.slices == {"a": slice(0, 5), "b": slice(5, 7)}
    assert mask.inv_start["b"] == rb.total_tokens
    assert P.build_activation_mask([ ]).values.shape == (0,)


def test_engine_config_json(tmp_path):
    import json
    p = tmp_path / "e.json"
    p.write_text(json.dumps({"model": {"n_layers": 1, "seed": 3}, "scheduler": {"token_budget": 32},
                             "pool_blocks": 64, "block_size": 8,
                             "adapters": [{"adapter_id": "x", "rank": 4, "seed": 0, "invocation_tokens": [250]}]}))
    cfg = P.load_engine_config(p)
    assert cfg.model.n_layers == 1 and cfg.scheduler.token_budget == 32 and cfg.block_size == 8
    p.write_text(json.dumps({"pool_block": 3}))
    with pytest.raises(ValueError, match="unknown engine config keys"):
        P.load_engine_config(p)


class _DeferredOracle:
    """Oracle model with the pipelined-decode interface (pack / launch_async / resolve): a decode step's input
    token may name the previous launch's greedy id of a span (-(j+1)), as on the device."""

    def __init__(self, oracle):
        self.o = oracle
        self.last_ids = np.zeros(0, dtype=np.int64)

    def _ids(self, seqs, out):
        return np.array([int(np.argmax(out[s.request_id])) for s in seqs], dtype=np.int64)

    def forward_step(self, seqs, kv):
        out = self.o.forward_step(seqs, kv)
        self.last_ids = self._ids(seqs, out)
        return out

    def pack(self, seqs, block_size, token_refs=False):
        res = []
        for s in seqs:
            t = np.asarray(s.tokens, dtype=np.int64)
            if (t < 0).any():
                assert token_refs and t.min() >= -len(self.last_ids)
                t = np.where(t < 0, self.last_ids[np.maximum(-t - 1, 0)], t)
            res.append(P.SeqInput(s.request_id, t, s.start_pos, list(s.block_ids), s.adapter, s.mask))
        return res

    def launch_async(self, seqs, kv):
        return self.forward_step(seqs, kv) and self.last_ids

    @staticmethod
    def resolve(handle):
        return handle


@pytest.mark.parametrize("name", ["d64_multi_alora", "d64_bab_alora_b8", "c1_bab_alora"])
def test_pipelined_decode_engine_matches_reference_pipeline(name):
    """Engine(pipelined_decode=True) bookkeeping (placeholder tokens, deferred retire, device token refs) must
    give the reference pipeline's ids, hits, first block tables, schedule and pool digests."""
    g = golden_json("pipelines.json")[name]
    spec = P.PipelineSpec(**g["spec"])
    model = _DeferredOracle(O.OracleModel(O.OracleConfig(**g["model"])))
    eng = P.build_engine(spec, model=P.ModelConfig(**g["model"]), engine_model=model, pool_storage="numpy",
                         pipelined_decode=True, **g["engine"])
    assert eng.pipelined_decode
    tables = {}
    orig = eng.scheduler._lookup_done

    def spy(req, hits):
        orig(req, hits)
        tables[req.request_id] = {"block_ids": [int(b) for b in hits], "reused": [True] * len(hits)}

    eng.scheduler._lookup_done = spy
    rows = P.run_sync_pipeline(spec, eng)
    for rid, r in g["requests"].items():
        mine = eng.finished[rid]
        assert list(map(int, mine.generated)) == r["generated"], rid
        assert (mine.hit_tokens, mine.computed_tokens) == (r["hit_tokens"], r["computed_tokens"]), rid
    assert tables == g["first_tables"]
    # virtual-clock stamps (finish = the launching step's stamp) give the reference's metrics CSV byte for byte
    assert P.render_csv(sorted(rows, key=lambda m: m.request_id)) == g["metrics_csv"] or \
        P.render_csv(rows) == g["metrics_csv"]
    strip = lambda tr: [{k: v for k, v in row.items() if k != "pool_free"} for row in tr]
    assert strip(eng.trace) == strip(g["trace"])
    assert sorted(r["digest"] for r in eng.pool.dump_state() if r["digest"]) == \
        sorted(r["digest"] for r in g["pool_dump"] if r["digest"])
    eng.pool.check_conservation()


def _pipelined_pair(pool_blocks, block_size=4, max_batch=8):
    cfg = O.OracleConfig(n_layers=1, n_heads=2, head_dim=16, d_model=32, vocab_size=64, seed=1)
    out = []
    for pipelined in (False, True):
        model = _DeferredOracle(O.OracleModel(cfg))
        ecfg = P.EngineConfig(model=P.ModelConfig(n_layers=1, n_heads=2, head_dim=16, d_model=32, vocab_size=64,
                                                  seed=1),
                              scheduler=P.SchedulerConfig(token_budget=64, max_batch_requests=max_batch),
                              pool_blocks=pool_blocks, block_size=block_size)
        out.append(P.Engine(ecfg, clock=P.VirtualClock(), model=model, pool_storage="numpy",
                            pipelined_decode=pipelined))
    return out


def test_pipelined_decode_commits_finished_request_before_next_admission():
    """A request waiting behind one that finishes in a pipelined decode step must see the finished request's
    published blocks (the synchronous engine commits before the next schedule_step)."""
    prompt = np.arange(32) % 50
    res = []
    for eng in _pipelined_pair(pool_blocks=64, max_batch=1):
        eng.submit(prompt, max_new_tokens=3, request_id="a")
        eng.submit(prompt, max_new_tokens=2, request_id="b")  # B waits for A's batch slot
        eng.run_until_idle()
        res.append((eng.finished["b"].hit_tokens, list(eng.finished["b"].generated), eng.finished["a"].finish,
                    eng.finished["b"].finish))
        eng.pool.check_conservation()
    assert res[0] == res[1]
    assert res[0][0] == 28  # ((32-1)//4)*4 once A's blocks are published


def test_pipelined_decode_tight_pool_matches_synchronous():
    """With a pool that only fits one request at a time, a pipelined engine must free a finished request's
    blocks before admitting the next (no spurious 'pool exhausted during decode')."""
    res = []
    for eng in _pipelined_pair(pool_blocks=10):
        for i, rid in enumerate("abc"):
            eng.submit((np.arange(30) + 7 * i) % 50, max_new_tokens=4, request_id=rid)
        eng.run_until_idle()
        res.append({rid: (r.failed, list(r.generated), r.hit_tokens, r.finish) for rid, r in eng.finished.items()})
        eng.pool.check_conservation()
    assert res[0] == res[1]
    assert all(v[0] is None for v in res[0].values())


def _fake_packer(vocab=384, graphs=False, last_S=0):
    import types
    cfg = P.ModelConfig(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512,
                        vocab_size=vocab, max_seq_len=4096, seed=4, dtype="bf16")
    slots = {None: -1, "a0": 0, "a1": 1}
    return types.SimpleNamespace(config=cfg, _max_seqs=64, _graphs=graphs, GRAPH_BLOCK_BUCKET=32, _last_S=last_S,
                                 _prefill_shapes={},
                                 _slot_for=lambda a: slots[None if a is None else a.adapter_id])


def test_step_packer_layout_and_token_refs():
    """Model.pack (the varlen step record the native forward reads), on CPU: positions, slot mapping, row
    adapter slots / apply flags, block tables, and the pipelined-decode token references."""
    from paper_2512_17910_b200.model import Model
    act = P.generate_adapter("a0", 256, 4, seed=1, invocation_tokens=(1, 2, 3))
    std = P.generate_adapter("a1", 256, 4, seed=2, mode="standard")
    B = 16
    seqs = [P.SeqInput("r0", np.array([5, 6, 7]), 30, [4, 9, 11], None, None),
            P.SeqInput("r1", np.array([8, 9]), 0, [3], act, np.array([True, False])),
            P.SeqInput("r2", np.array([10]), 17, [1, 2], std, None)]
    p = Model.pack(_fake_packer(), seqs, B)
    assert p["M"] == 6 and p["S"] == 3 and p["max_q"] == 3 and p["max_ctx"] == 33
    np.testing.assert_array_equal(p["positions"], [30, 31, 32, 0, 1, 17])
    np.testing.assert_array_equal(p["cu_q"], [0, 3, 5, 6])
    np.testing.assert_array_equal(p["last_row"], [2, 4, 5])
    np.testing.assert_array_equal(p["slot_mapping"], [9 * B + 14, 9 * B + 15, 11 * B, 3 * B, 3 * B + 1, 2 * B + 1])
    np.testing.assert_array_equal(p["row_slot"], [-1, -1, -1, 0, 0, 1])
    np.testing.assert_array_equal(p["row_apply"], [0, 0, 0, 0, 1, 1])  # masked activated row keeps the base
    np.testing.assert_array_equal(p["block_table"], [[4, 9, 11], [3, 0, 0], [1, 2, 0]])
    # token references: -(j+1) names span j of the previous launch; only with token_refs and j < last S
    ref = [P.SeqInput("r0", np.array([-2]), 33, [4, 9, 11], None, None)]
    with pytest.raises(ValueError):
        Model.pack(_fake_packer(last_S=3), ref, B)
    with pytest.raises(ValueError):
        Model.pack(_fake_packer(last_S=1), ref, B, token_refs=True)
    q = Model.pack(_fake_packer(last_S=3), ref, B, token_refs=True)
    assert q["tokens"].tolist() == [-2]
    with pytest.raises(ValueError):  # above the vocabulary is never a reference
        Model.pack(_fake_packer(last_S=3), [P.SeqInput("r0", np.array([384]), 0, [1], None, None)], B,
                   token_refs=True)
    # a recurring prefill shape is marked for graph capture on its second sighting; decode steps always are
    fk = _fake_packer(graphs=True)
    assert not Model.pack(fk, seqs, B)["graphable"] and Model.pack(fk, seqs, B)["graphable"]
    dec = Model.pack(fk, [P.SeqInput("r0", np.array([5]), 40, [4, 9, 11], None, None)], B)
    assert dec["graphable"] and dec["maxb"] == 32 and dec["max_ctx"] == 32 * B


def test_batched_hashing_after_fork():
    """The parked hashing helpers are per process: a fork()ed child that hashes after its parent used the
    helpers must not wait on threads that only exist in the parent."""
    import multiprocessing as mp
    chains = [(np.arange(256) % 97 + i, 16, [""] * 16) for i in range(4)]
    want = P.kv_cache.hash_chains(chains, 16, n_threads=4)  # parent starts its helpers

    def child(q):
        q.put(P.kv_cache.hash_chains(chains, 16, n_threads=4))

    ctx = mp.get_context("fork")
    q = ctx.Queue()
    pr = ctx.Process(target=child, args=(q,))
    pr.start()
    got = q.get(timeout=30)
    pr.join(timeout=30)
    assert pr.exitcode == 0 and got == want


def _plan(cu, starts, tables, B=16, H=32, Hkv=8, D=128, flags=1, cap=1 << 30):
    import ctypes  # noqa: F401
    S = len(starts)
    maxb = max(len(t) for t in tables)
    bt = np.zeros((S, maxb), np.int32)
    for i, t in enumerate(tables):
        bt[i, :len(t)] = t
    cu = np.asarray(cu, np.int32)
    st = np.asarray(starts, np.int32)
    out = np.empty(1 << 20, np.int32)
    n = P._native.lib.alora_plan_attention(S, cu.ctypes.data, st.ctypes.data, bt.ctypes.data, maxb, B, H, Hkv, D,
                                           flags, cap, out.ctypes.data, out.size)
    assert n > 0
    out = out[:n]
    ni, ns, nq = int(out[0]), int(out[1]), int(out[2])
    items = out[8:8 + 8 * ni].reshape(ni, 8)
    segs = out[8 + 8 * ni:8 + 8 * ni + 4 * ns].reshape(ns, 4)
    o = 8 + 8 * ni + 4 * ns
    sets = out[o:o + 2 * nq].reshape(nq, 2)
    M = int(cu[-1])
    set_tok = out[o + 2 * nq:o + 2 * nq + M]
    sp_np = out[o + 2 * nq + M:o + 2 * nq + M + S]
    return out, items, segs, sets, set_tok, sp_np, bt


@pytest.mark.parametrize("case", ["eval_groups", "decode_groups", "mixed", "long_prefill"])
def test_attention_plan_covers_every_key_once(case):
    """alora_plan_attention (host): for every (row, head) the plan's items x segments visit exactly the keys
    [0, pos] of the row's own sequence, each once, through block tables that map them to the row's own
    physical blocks; spans holding the same leading blocks are grouped (shared prefix read once)."""
    rng = np.random.default_rng(3)
    B, H, Hkv, G = 16, 32, 8, 4
    if case in ("eval_groups", "decode_groups"):
        n_conv, n_ad, cached = 3, 4, 1000 // 16 * 16
        lens = [1 if case == "decode_groups" else 20] * (n_conv * n_ad)
        starts, tables, nb = [], [], 0
        conv_blocks = [list(range(c * 200, c * 200 + cached // B)) for c in range(n_conv)]
        for c in range(n_conv):
            for k in range(n_ad):
                st = cached + (7 if case == "decode_groups" else 0) + k
                total = st + lens[len(starts)]
                own = list(range(5000 + len(starts) * 10, 5000 + len(starts) * 10 + 10))
                tables.append(conv_blocks[c] + own[:-(-total // B) - len(conv_blocks[c])])
                starts.append(st)
    elif case == "mixed":
        starts = [0, 300, 300, 40, 2000]
        lens = [70, 9, 9, 33, 1]
        shared = list(range(100, 120))
        tables = [list(range(0, 5)), shared + [900, 901, 902], shared + [910, 911], list(range(30, 35)),
                  list(range(40, 166))]
        tables[2] = tables[2] + [912]
    else:
        starts, lens = [0, 0], [700, 300]
        tables = [list(range(0, 44)), list(range(50, 69))]
    cu = np.concatenate([[0], np.cumsum(lens)])
    out, items, segs, sets, set_tok, sp_np, bt = _plan(cu, starts, tables, B, H, Hkv)
    M = int(cu[-1])
    row_span = np.repeat(np.arange(len(starts)), lens)
    pos = np.concatenate([np.arange(s, s + n) for s, n in zip(starts, lens)])
    seen = {}  # (row, head) -> list of physical (block, offset) keys
    for it in items:
        q, mt, sb, se, p_index = (int(x) for x in it[:5])
        off, n_tok = sets[q]
        QT = 128 * int(os.environ.get("ALORA_ATTN_MT", "2"))  # query rows per item (the kernel's tiles per CTA)
        for r in range(QT):
            pr = mt * QT + r
            if pr >= n_tok * G:
                break
            row = int(set_tok[off + pr // G])
            head = pr % G
            for tab, lo, hi, flt in segs[sb:se]:
                if flt >= 0 and flt != row_span[row]:
                    continue
                lim = min(pos[row], hi - 1)
                for k in range(lo, lim + 1):
                    seen.setdefault((row, head), []).append((int(bt[tab, k // B]), k % B))
    for row in range(M):
        want = [(tables[row_span[row]][k // B], k % B) for k in range(pos[row] + 1)]
        for head in range(G):
            assert sorted(seen[(row, head)]) == sorted(want), (case, row, head)
    assert sorted(set_tok.tolist()) == list(range(M))
    if case.endswith("groups"):
        assert int(out[2]) == 3  # one set per conversation
        assert int(out[5]) < sum(s + n for s, n in zip(starts, lens)) // 3  # distinct keys: prefixes counted once
    if case == "mixed":
        assert int(out[2]) == 4  # the two spans on the shared blocks form one set


def test_extension_targets_shapes_and_validation():
    """O / MLP adapter targets (extension of adapters.py:26): factor shapes per projection, unknown names rejected."""
    import paper_2512_17910_b200 as P
    ad = P.generate_adapter("x", 64, 4, targets=("o", "gate", "up", "down"), mode="standard", q_width=32,
                            kv_width=16, ffn_width=96)
    assert ad.down["o"].shape == (32, 4) and ad.up["o"].shape == (4, 64)
    assert ad.down["gate"].shape == (64, 4) and ad.up["up"].shape == (4, 96)
    assert ad.down["down"].shape == (96, 4) and ad.up["down"].shape == (4, 64)
    # the q/k/v factors are unchanged by the extension (same Philox streams as the reference)
    a1 = P.generate_adapter("y", 64, 4, targets=("q", "v"), mode="standard")
    a2 = P.generate_adapter("y", 64, 4, targets=("q", "v", "o"), mode="standard")
    np.testing.assert_array_equal(a1.down["q"], a2.down["q"])
    with pytest.raises(ValueError):
        P.generate_adapter("z", 64, 4, targets=("w_gate",), mode="standard")


def test_oracle_extension_targets_formula():
    """oracle._adapted at fp64acc is the reference's masked formula (model.py:141-145) at another projection."""
    import oracle as O
    from oracle.model_oracle import _adapted
    cfg = O.OracleConfig(n_layers=1, n_heads=2, head_dim=8, d_model=16, vocab_size=32)
    ad = O.oracle_adapter("o", cfg, 4, targets=("o",), mode="standard")
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 16)).astype(np.float32)
    w = rng.standard_normal((16, 16)).astype(np.float32)
    mask = np.array([True, False, True, False, False])
    got = _adapted(x, w, "o", ad, mask, False).astype(np.float32)
    base = O.mm(x, w)
    adapted = base + O.mm(O.mm(x, ad.down["o"]), ad.up["o"])
    np.testing.assert_array_equal(got, np.where(mask[:, None], base, adapted))
    np.testing.assert_array_equal(_adapted(x, w, "up", ad, None, False).astype(np.float32), base)
