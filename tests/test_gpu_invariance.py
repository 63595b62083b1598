"""Batch-invariant bf16 numerics (Model(batch_invariant=True)).

The reference computes every row in fp64 with one rounding (model.py:95-98), so a token's KV and logits do
not depend on how the engine batched or chunked it; its own tests pin exactly that (tests/test_model.py:
167-202 chunked == whole and batch independence; tests/test_acceptance.py:234-280 caching on/off). The fp32
tier reproduces it by construction; the bf16 tier does when batch_invariant is set: one weight-streaming GEMM
kernel and K range for every row (no M-dependent split-K, no swap-AB decode GEMM, 256-row launches for
larger steps), the segmented LoRA shrink for every row count, one tcgen05 attention kernel with a single KV
partition per row. These tests compute one aLoRA request's 300 tokens three ways -- one whole prefill, three
chunks co-batched with other requests, a prefill then 40 decode steps co-batched with other decode requests --
and require its KV (every layer) and its last-token logits to be bitwise identical.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")

SMALL = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512,
             vocab_size=320, seed=1)
C2W = dict(arch="llama", n_layers=2, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=8192,
           vocab_size=4096, seed=2)
C3W = dict(arch="llama", n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, ffn_dim=14336,
           vocab_size=4096, seed=3)
B = 16
N = 300


def _setup(dims):
    cfg = P.ModelConfig(**dims, max_seq_len=1024, dtype="bf16")
    V = cfg.vocab_size
    inv = P.invocation_for(V, 0)
    ad = P.generate_adapter("a0", cfg.d_model, 32, seed=4, invocation_tokens=inv, kv_width=cfg.kv_width,
                            q_width=cfg.q_width, ffn_width=cfg.ffn,
                            targets=("q", "k", "v", "o", "gate", "up", "down"))
    rng = np.random.default_rng(9)
    toks = np.concatenate([rng.integers(0, V - 32, 200), inv, rng.integers(0, V - 32, N - 203)]).astype(np.int64)
    others = [rng.integers(0, V - 32, 400).astype(np.int64) for _ in range(4)]
    return cfg, ad, toks, others


def _span(rid, toks, start, end, table, ad, inv_start=200):
    mask = np.arange(start, end) < inv_start
    return P.SeqInput(rid, toks[start:end], start, table, ad, mask)


def _kv_rows(pool, table, n):
    kv = pool.kv
    pos = np.arange(n)
    ids = torch.as_tensor(np.asarray(table)[pos // B], device=kv.device)
    rows = torch.as_tensor(pos % B, device=kv.device)
    return kv[ids, :, :, rows].float().cpu().numpy()  # [n, L, 2, kv_width]


@pytest.mark.parametrize("dims", [SMALL, C2W, C3W], ids=["small", "c2w", "c3w"])
def test_kv_and_logits_bitwise_whole_vs_chunked_vs_decode(dims):
    cfg, ad, toks, others = _setup(dims)
    model = P.Model(cfg, init="device", batch_invariant=True, max_tokens=1024)
    table = list(range(0, 20))  # the target request's blocks in every pool
    other_tables = [list(range(20 + 30 * i, 50 + 30 * i)) for i in range(4)]
    nb = 20 + 30 * 4 + 2

    def pool():
        return P.BlockPool(nb, B, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")

    # A: one whole prefill (M = 300 > 256: two row-chunk launches per GEMM), alone
    pa = pool()
    la = model.forward_step([_span("t", toks, 0, N, table, ad)], pa.kv)["t"]
    # B: three chunks, each co-batched with other requests' prefill spans of different lengths
    pb = pool()
    cuts, lens = [0, 128, 228, N], [37, 150, 5]
    for c in range(3):
        seqs = [P.SeqInput(f"o{c}", others[c][:lens[c]], 0, other_tables[c])]
        seqs.append(_span("t", toks, cuts[c], cuts[c + 1], table, ad))
        if c == 1:
            seqs.append(P.SeqInput("o3", others[3][:64], 0, other_tables[3]))
        lb = model.forward_step(seqs, pb.kv)["t"]
    # C: prefill 260 alone, then 40 decode steps with a changing set of co-batched decode requests
    pc = pool()
    model.forward_step([_span("t", toks, 0, 260, table, ad)], pc.kv)
    for i in range(4):
        model.forward_step([P.SeqInput(f"o{i}", others[i][:100], 0, other_tables[i])], pc.kv)
    for pos in range(260, N):
        seqs = [P.SeqInput(f"o{i}", others[i][100 + pos - 260:101 + pos - 260], 100 + pos - 260, other_tables[i])
                for i in range((pos % 4) + 1)]
        seqs.insert(pos % 3 if pos % 3 < len(seqs) else 0, _span("t", toks, pos, pos + 1, table, ad))
        lc = model.forward_step(seqs, pc.kv)["t"]
    ka, kb, kc = _kv_rows(pa, table, N), _kv_rows(pb, table, N), _kv_rows(pc, table, N)
    for name, other in (("chunked", kb), ("decode", kc)):
        bad = np.argwhere(np.any(ka != other, axis=(1, 2, 3)))
        assert len(bad) == 0, f"{name}: KV of {len(bad)} positions differs from the whole prefill, first {bad[:5].ravel()}"
    np.testing.assert_array_equal(la, lb)
    np.testing.assert_array_equal(la, lc)
    print(f"[parity] batch-invariant {cfg.d_model}: KV of {N} positions x {cfg.n_layers} layers and last logits "
          f"bitwise equal (whole / chunked+co-batched / prefill+40 decode steps)")


def test_invariant_mode_is_close_to_default_mode():
    """The invariant kernels compute the same function: logits within the bf16 tolerance of the default mode."""
    cfg, ad, toks, _ = _setup(SMALL)
    outs = []
    for inv in (False, True):
        m = P.Model(cfg, batch_invariant=inv)
        pool = P.BlockPool(24, B, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
        outs.append(m.forward_step([_span("t", toks, 0, N, list(range(20)), ad)], pool.kv)["t"])
    assert float(np.max(np.abs(outs[0] - outs[1]))) < 5e-2


def test_engine_batch_invariant_caching_on_off_identical():
    """The reference's caching on/off law (tests/test_acceptance.py:234-280) on the bf16 tier: with
    batch_invariant the same pipeline run with and without prefix caching emits identical greedy ids and
    identical logits, although with caching the eval turn computes only its suffix over reused blocks."""
    mc = P.ModelConfig(**SMALL, max_seq_len=1024, dtype="bf16")
    spec = P.PipelineSpec(pipeline="multi_adapter", mode="alora", prompt_len=150, gen_len=12, adapter_gen_len=8,
                          n_adapters=2, batch=2, seed=3)
    runs = []
    for caching in (True, False):
        eng = P.build_engine(spec, model=mc, block_size=B, prefix_caching=caching, batch_invariant=True,
                             token_budget=256)
        seen = []
        eng.on_logits = lambda rid, pos, lg, seen=seen: seen.append((rid, pos, np.array(lg, copy=True)))
        P.run_sync_pipeline(spec, eng)
        ids = {rid: list(r.generated) for rid, r in eng.finished.items()}
        hits = sum(r.hit_tokens for r in eng.finished.values())
        runs.append((ids, sorted(seen, key=lambda x: (x[0], x[1])), hits))
    (ids_a, lg_a, hits_a), (ids_b, lg_b, hits_b) = runs
    assert hits_a > 0 and hits_b == 0
    assert ids_a == ids_b
    assert [x[:2] for x in lg_a] == [x[:2] for x in lg_b]
    for a, b in zip(lg_a, lg_b):
        np.testing.assert_array_equal(a[2], b[2])
