"""bf16 tensor-core tier end to end on the B200, against the oracle's bf16 numerics.

The oracle (numerics="bf16") applies the same bf16 rounding points as the
GPU path (weights, GEMM inputs, q/k/v, KV cache, attention output) and
accumulates in fp64; the GPU accumulates in fp32 and rounds P to bf16 inside
attention. Stated tolerances: |Δlogit| <= 5e-2 abs,
KV rel-L2 <= 1e-2; cache-hit counts and block tables bit-exact; greedy ids
compared where the oracle's top-1/top-2 margin exceeds the bf16 error bound.
"""

import ctypes

import numpy as np
import pytest

from conftest import C1, dense_reference_attention, golden_json
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")
from paper_2512_17910_b200 import _native  # noqa: E402

LOGIT_TOL = 5e-2
KV_REL_L2 = 1e-2


def _attn_case(n_seqs, H, Hkv, D, B, starts, lens, seed):
    rng = np.random.default_rng(seed)
    kvw = Hkv * D
    totals = [s + n for s, n in zip(starts, lens)]
    nbs = [-(-t // B) for t in totals]
    NB = sum(nbs) + 3
    perm = rng.permutation(NB)
    pool = np.zeros((NB, 2, 2, B, kvw), np.float32)  # 2 layers, attend layer 1
    tables, ks, vs, qs = [], [], [], []
    off = 0
    for s in range(n_seqs):
        ids = [int(x) for x in perm[off:off + nbs[s]]]
        off += nbs[s]
        k = O.bf16_round(rng.standard_normal((totals[s], kvw)))
        v = O.bf16_round(rng.standard_normal((totals[s], kvw)))
        q = O.bf16_round(rng.standard_normal((lens[s], H * D)))
        for t in range(totals[s]):
            pool[ids[t // B], 1, 0, t % B] = k[t]
            pool[ids[t // B], 1, 1, t % B] = v[t]
        tables.append(ids)
        ks.append(k); vs.append(v); qs.append(q)
    return pool, tables, ks, vs, qs


@pytest.mark.parametrize("H,Hkv,D,B,starts,lens", [
    (32, 8, 64, 16, [0], [70]),
    (32, 8, 64, 16, [2000], [7]),                    # aLoRA suffix over a long cached prefix (split-KV)
    (8, 8, 128, 16, [100, 0, 517], [33, 1, 64]),    # MHA, D=128, mixed batch
    (8, 2, 64, 5, [13, 300], [40, 3]),              # odd block size
    (32, 8, 64, 16, [0, 0, 0, 0], [300, 257, 1, 64]),
    (32, 8, 64, 32, [100, 0, 1500], [40, 70, 9]),    # B=32: two pages per 64-key tile
    (8, 8, 128, 64, [300, 0], [20, 90]),             # B=64: one page per tile, D=128
    (8, 2, 64, 8, [40, 0], [30, 17]),                # B=8: eight pages per 64-key tile
    # decode steps (one query row per sequence): the split-KV decode kernel, every GQA group size it serves
    (32, 8, 64, 16, [2047, 5, 0, 130, 31, 32, 33], [1] * 7),
    (8, 8, 128, 16, [1000, 77], [1, 1]),             # G=1, D=128
    (32, 8, 128, 16, list(range(0, 1100, 100)), [1] * 11),  # D=128 with units >= 74: whole-context CTAs
    (16, 2, 64, 16, [511, 3], [1, 1]),               # G=8
    (8, 4, 64, 8, [300, 64, 7], [1, 1, 1]),          # G=2, B=8
    (32, 8, 64, 32, [4000, 100], [1, 1]),            # B=32: one page per 32-key chunk
    (32, 8, 64, 16, list(range(0, 1200, 50)), [1] * 24),   # many sequences: few partitions each
    (8, 2, 64, 5, [300, 12], [1, 1]),                # B=5: not a divisor of 32 -> tensor-core kernel
])
def test_paged_attention_bf16_vs_dense(H, Hkv, D, B, starts, lens):
    n = len(starts)
    pool, tables, ks, vs, qs = _attn_case(n, H, Hkv, D, B, starts, lens, seed=H + D + B)
    dev_pool = torch.as_tensor(pool).to("cuda", torch.bfloat16).contiguous()
    q = torch.as_tensor(np.concatenate(qs)).to("cuda", torch.bfloat16).contiguous()
    M = q.shape[0]
    out = torch.empty_like(q)
    maxb = max(len(t) for t in tables)
    bt = np.zeros((n, maxb), np.int32)
    for i, t in enumerate(tables):
        bt[i, :len(t)] = t
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    d_cu = torch.as_tensor(cu).cuda()
    d_sp = torch.as_tensor(np.asarray(starts, np.int32)).cuda()
    d_bt = torch.as_tensor(bt).cuda()
    max_q, max_ctx = max(lens), max(s + l for s, l in zip(starts, lens))
    wsb = _native.lib.alora_attn_workspace_bytes(_native.ALORA_BF16, M, n, max_q, max_ctx, H, Hkv, D)
    ws = torch.zeros(max(int(wsb), 1), dtype=torch.uint8, device="cuda")
    rc = _native.lib.alora_paged_prefill_attn(
        _native.ALORA_BF16, q.data_ptr(), q.shape[1], M, n, d_cu.data_ptr(), d_sp.data_ptr(), d_bt.data_ptr(), maxb,
        max_q, max_ctx, dev_pool.data_ptr(), dev_pool.shape[0], 2, 1, B, H, Hkv, D, out.data_ptr(), out.shape[1], ws.data_ptr(),
        ws.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc, "alora_paged_prefill_attn")
    got = out.float().cpu().numpy()
    worst = 0.0
    for s in range(n):
        want = dense_reference_attention(qs[s], ks[s], vs[s], H, starts[s], Hkv)
        worst = max(worst, float(np.max(np.abs(got[cu[s]:cu[s + 1]] - want))))
    print(f"[parity] bf16 paged attention H={H} Hkv={Hkv} D={D} B={B}: max |d| {worst:.3g} (split bytes {wsb})")
    assert worst < 3e-2


def _models(arch_dims, adapters):
    ocfg = O.OracleConfig(**arch_dims, numerics="bf16")
    om = O.OracleModel(ocfg)
    pcfg = P.ModelConfig(**arch_dims, dtype="bf16")
    pm = P.Model(pcfg)
    return om, pm, ocfg, pcfg


LLAMA = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512,
             vocab_size=320, seed=1)


@pytest.mark.parametrize("dims", [C1, LLAMA])
def test_forward_bf16_vs_oracle_with_adapters(dims):
    om, pm, ocfg, pcfg = _models(dims, None)
    V = dims["vocab_size"]
    inv = (V - 32, V - 31, V - 30)
    oa = O.oracle_adapter("a0", ocfg, 32, seed=2, invocation_tokens=inv)
    oa_std = O.oracle_adapter("a1", ocfg, 16, seed=3, targets=("q", "v"), mode="standard")
    pa = P.generate_adapter("a0", ocfg.d_model, 32, seed=2, invocation_tokens=inv, kv_width=ocfg.kv_width,
                            q_width=ocfg.q_width)
    pa_std = P.generate_adapter("a1", ocfg.d_model, 16, seed=3, targets=("q", "v"), mode="standard",
                                kv_width=ocfg.kv_width, q_width=ocfg.q_width)
    rng = np.random.default_rng(0)
    B = 16
    okv = om.new_pool(64, B)
    pool = P.BlockPool(64, B, dims["n_layers"], ocfg.d_model, kv_width=ocfg.kv_width, dtype="bf16")
    # three requests: base, activated adapter (prefix then masked suffix), standard LoRA
    toks = [rng.integers(0, V - 32, 150), np.concatenate([rng.integers(0, V - 32, 90), inv, rng.integers(0, V - 32, 4)]),
            rng.integers(0, V - 32, 40)]
    tables = [list(range(0, 12)), list(range(12, 24)), list(range(24, 30))]
    split = [100, 60, 0]
    worst = 0.0
    for phase in range(2):
        oseqs, pseqs = [], []
        for r in range(3):
            s, e = (0, split[r]) if phase == 0 else (split[r], len(toks[r]))
            if e <= s:
                continue
            if r == 1:
                mask = np.arange(s, e) < 90
                oseqs.append(O.OracleSpan(f"r{r}", toks[r][s:e], s, tables[r], oa, mask))
                pseqs.append(P.SeqInput(f"r{r}", toks[r][s:e], s, tables[r], pa, mask))
            elif r == 2:
                oseqs.append(O.OracleSpan(f"r{r}", toks[r][s:e], s, tables[r], oa_std, None))
                pseqs.append(P.SeqInput(f"r{r}", toks[r][s:e], s, tables[r], pa_std, None))
            else:
                oseqs.append(O.OracleSpan(f"r{r}", toks[r][s:e], s, tables[r]))
                pseqs.append(P.SeqInput(f"r{r}", toks[r][s:e], s, tables[r]))
        want = om.forward_step(oseqs, okv)
        got = pm.forward_step(pseqs, pool.kv)
        for k in want:
            err = float(np.max(np.abs(got[k] - want[k])))
            worst = max(worst, err)
            margin = np.sort(want[k])[-1] - np.sort(want[k])[-2]
            if margin > 2 * LOGIT_TOL:
                assert int(np.argmax(got[k])) == int(np.argmax(want[k])), k
    # two decode steps (M = 3 rows: the swap-AB decode GEMM path, LoRA expand as extra K, deferred RoPE /
    # LoRA select / residual consumers); every request feeds the oracle's greedy token of the previous step
    nxt = {k: int(np.argmax(want[k])) for k in want}
    lens = [len(t) for t in toks]
    for step in range(2):
        oseqs, pseqs = [], []
        for r in range(3):
            tk, pos = np.array([nxt[f"r{r}"]]), lens[r] + step
            if r == 1:
                oseqs.append(O.OracleSpan(f"r{r}", tk, pos, tables[r], oa, np.array([False])))
                pseqs.append(P.SeqInput(f"r{r}", tk, pos, tables[r], pa, np.array([False])))
            elif r == 2:
                oseqs.append(O.OracleSpan(f"r{r}", tk, pos, tables[r], oa_std, None))
                pseqs.append(P.SeqInput(f"r{r}", tk, pos, tables[r], pa_std, None))
            else:
                oseqs.append(O.OracleSpan(f"r{r}", tk, pos, tables[r]))
                pseqs.append(P.SeqInput(f"r{r}", tk, pos, tables[r]))
        want = om.forward_step(oseqs, okv)
        got = pm.forward_step(pseqs, pool.kv)
        for k in want:
            worst = max(worst, float(np.max(np.abs(got[k] - want[k]))))
            nxt[k] = int(np.argmax(want[k]))
    kv = pool.kv.float().cpu().numpy()
    rel = float(np.linalg.norm(kv - okv) / np.linalg.norm(okv))
    print(f"[parity] bf16 forward {dims.get('arch', 'ref')}: max |dlogit| {worst:.3g}, KV rel-L2 {rel:.3g}, "
          f"launches/step {pm.last_launches}")
    assert worst <= LOGIT_TOL and rel <= KV_REL_L2


def test_bf16_pre_invocation_kv_bitwise_identical_to_base():
    pm = P.Model(P.ModelConfig(**LLAMA, dtype="bf16"))
    cfg = pm.config
    V = cfg.vocab_size
    inv = (V - 32, V - 31, V - 30)
    ad = P.generate_adapter("a", cfg.d_model, 32, invocation_tokens=inv, kv_width=cfg.kv_width, q_width=cfg.q_width)
    rng = np.random.default_rng(13)
    toks = np.concatenate([rng.integers(0, V - 32, 77), inv, rng.integers(0, V - 32, 9)])
    mask = np.arange(len(toks)) < 77
    pools = []
    for adapter in (None, ad):
        pool = P.BlockPool(8, 16, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
        ids = pool.allocate("r", 6)
        pm.forward_step([P.SeqInput("r", toks, 0, ids, adapter, mask if adapter else None)], pool.kv)
        pools.append(pool.kv.float().cpu().numpy())
    for pos in range(len(toks)):
        a, b = pools[0][pos // 16, :, :, pos % 16], pools[1][pos // 16, :, :, pos % 16]
        if pos < 77:
            np.testing.assert_array_equal(a, b)
        else:
            assert not np.array_equal(a, b)


def test_bf16_c1_pipeline_hits_and_tables_exact():
    g = golden_json("pipelines.json")["c1_bab_alora"]
    spec = P.PipelineSpec(**g["spec"])
    eng = P.build_engine(spec, model=P.ModelConfig(**g["model"], dtype="bf16"), **g["engine"])
    seen = []  # (request id, end position, device logits) of every emitted token
    eng.on_logits = lambda rid, end, lg: seen.append((rid, end, np.array(lg)))
    rows = P.run_sync_pipeline(spec, eng)
    same = total = 0
    for rid, r in g["requests"].items():
        mine = eng.finished[rid]
        assert (mine.hit_tokens, mine.computed_tokens) == (r["hit_tokens"], r["computed_tokens"]), rid
        same += sum(int(a == b) for a, b in zip(mine.generated, r["generated"]))
        total += len(r["generated"])
    assert len(rows) == len(g["requests"])
    # margin-aware greedy parity: every emitted id, teacher-forced on the device's own token history, against
    # the bf16 oracle's logits for that context; ids must agree wherever the oracle's top-2 margin decides them
    ocfg = O.OracleConfig(**g["model"], numerics="bf16")
    om = O.OracleModel(ocfg)
    oads = {}
    for k, a in eng.adapters.items():
        oads[k] = O.oracle_adapter(k, ocfg, a.rank, seed=spec.seed, invocation_tokens=a.invocation_tokens)
    decided = agree = worst = 0
    for rid, end, lg in seen:
        req = eng.finished[rid]
        toks = req.tokens_slice(0, end)
        ad = None if req.adapter is None else oads[req.adapter.adapter_id]
        mask = None if ad is None else np.arange(end) < req.inv_start
        kv = om.new_pool(-(-end // 16), 16)
        want = om.forward_one(O.OracleSpan(rid, toks, 0, list(range(kv.shape[0])), ad, mask), kv)
        worst = max(worst, float(np.max(np.abs(lg - want))))
        top2 = np.partition(want, -2)[-2:]
        if top2[1] - top2[0] > 2 * LOGIT_TOL:
            decided += 1
            agree += int(np.argmax(lg)) == int(np.argmax(want))
    print(f"[parity] bf16 C1 pipeline: {len(seen)} emitted ids, max |dlogit| {worst:.3g}; margin-decided "
          f"{decided}, agreeing {agree}; free-running ids equal to the fp64 reference {same}/{total}")
    assert worst <= LOGIT_TOL
    assert agree == decided and decided >= 0.8 * len(seen)


@pytest.mark.parametrize("B", [16, 32])
def test_paged_attention_split_repeated_no_race(B):
    """The split-KV sequence of the mixed case, launched 150 times on one stream: every launch within tolerance
    (a stale-phase wait on a 2-deep PV barrier once let the O rescale / final read race a running PV, ~2% of
    launches at B=32)."""
    H, Hkv, D, starts, lens = 32, 8, 64, [100, 0, 1500], [40, 70, 9]
    n = len(starts)
    pool, tables, ks, vs, qs = _attn_case(n, H, Hkv, D, B, starts, lens, seed=H + D + B)
    want = [dense_reference_attention(qs[s], ks[s], vs[s], H, starts[s], Hkv) for s in range(n)]
    dev_pool = torch.as_tensor(pool).to("cuda", torch.bfloat16).contiguous()
    q = torch.as_tensor(np.concatenate(qs)).to("cuda", torch.bfloat16).contiguous()
    M = q.shape[0]
    maxb = max(len(t) for t in tables)
    bt = np.zeros((n, maxb), np.int32)
    for i, t in enumerate(tables):
        bt[i, :len(t)] = t
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    d_cu, d_sp, d_bt = (torch.as_tensor(a).cuda() for a in (cu, np.asarray(starts, np.int32), bt))
    max_q, max_ctx = max(lens), max(s + l for s, l in zip(starts, lens))
    wsb = _native.lib.alora_attn_workspace_bytes(_native.ALORA_BF16, M, n, max_q, max_ctx, H, Hkv, D)
    ws = torch.zeros(max(int(wsb), 1), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(150):
        out = torch.empty_like(q)
        _native.check(_native.lib.alora_paged_prefill_attn(
            _native.ALORA_BF16, q.data_ptr(), q.shape[1], M, n, d_cu.data_ptr(), d_sp.data_ptr(), d_bt.data_ptr(), maxb,
            max_q, max_ctx, dev_pool.data_ptr(), dev_pool.shape[0], 2, 1, B, H, Hkv, D, out.data_ptr(), out.shape[1],
            ws.data_ptr(), ws.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "attn")
        outs.append(out)
    got = torch.stack(outs).float().cpu().numpy()
    s = 2
    worst = float(np.max(np.abs(got[:, cu[s]:cu[s + 1]] - want[s][None])))
    assert worst < 3e-2, worst
    assert (got == got[0][None]).all()  # and bitwise identical launch to launch
