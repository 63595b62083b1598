"""Shared-prefix paged attention (alora_plan_attention + alora_paged_prefix_attn) on the B200 against the dense
fp64 per-head reference (reference tests/conftest.py:15-35 generalised to GQA; model.py:149-187 semantics).

Requests of one conversation evaluated on different adapters hold the same physical prefix blocks
(base-aligned reuse, reference kv_cache.py:72-96); the planner groups them so the prefix KV is streamed once
for all of their query rows, and each request's own keys (its private blocks, causal) are folded into the same
online softmax. Cases: eval-turn suffixes (20 rows over a 2k / 4k cached prefix), decode steps, a mix of
grouped and ungrouped spans (one split into KV partitions), long causal prefill, D 64 / 128, B 16 / 32.
"""

import ctypes

import numpy as np
import pytest

from conftest import dense_reference_attention
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")
from paper_2512_17910_b200 import _native  # noqa: E402


def _case(kind, B, D, H, Hkv, seed):
    rng = np.random.default_rng(seed)
    if kind in ("eval", "decode"):
        n_conv, n_ad = 3, 4
        cached = (2048 if D == 64 else 4096) // B * B
        starts, lens, tables, nb = [], [], [], 0
        conv = []
        for c in range(n_conv):
            conv.append(list(range(nb, nb + cached // B)))
            nb += cached // B
        for c in range(n_conv):
            for k in range(n_ad):
                st = cached if kind == "eval" else cached + 20 + k
                n = 20 if kind == "eval" else 1
                tail = -(-(st + n) // B) - len(conv[c])
                tables.append(conv[c] + list(range(nb, nb + tail)))
                nb += tail
                starts.append(st)
                lens.append(n)
    elif kind == "mixed":
        starts, lens = [0, 640, 640, 640, 3000, 17], [90, 12, 12, 12, 1, 40]
        tables, nb = [], 0
        shared = list(range(0, 640 // B))
        nb = len(shared)
        for s, n in zip(starts, lens):
            need = -(-(s + n) // B)
            if s == 640:
                own = list(range(nb, nb + need - len(shared)))
                tables.append(shared + own)
            else:
                own = list(range(nb, nb + need))
                tables.append(own)
            nb += len(own)
    else:  # long causal prefill
        starts, lens = [0, 128], [1500, 300]
        tables, nb = [], 0
        for s, n in zip(starts, lens):
            need = -(-(s + n) // B)
            tables.append(list(range(nb, nb + need)))
            nb += need
    perm = rng.permutation(nb + 5)  # scatter the logical blocks over the pool
    tables = [[int(perm[b]) for b in t] for t in tables]
    kvw = Hkv * D
    pool = np.zeros((nb + 5, 2, 2, B, kvw), np.float32)  # 2 layers, attend layer 1
    vals = O.bf16_round(rng.standard_normal((nb + 5, 2, B, kvw)).astype(np.float32))
    pool[:, 1] = vals
    qs, ks, vs = [], [], []
    for s, (st, n) in enumerate(zip(starts, lens)):
        p = np.arange(st + n)
        tb = np.asarray(tables[s])
        ks.append(pool[tb[p // B], 1, 0, p % B])
        vs.append(pool[tb[p // B], 1, 1, p % B])
        qs.append(O.bf16_round(rng.standard_normal((n, H * D)).astype(np.float32)))
    return starts, lens, tables, pool, qs, ks, vs


@pytest.mark.parametrize("kind,B,D,H,Hkv", [
    ("eval", 16, 128, 32, 8), ("eval", 16, 64, 32, 8), ("eval", 32, 128, 32, 8),
    ("decode", 16, 128, 32, 8), ("decode", 16, 64, 32, 8),
    ("mixed", 16, 128, 32, 8), ("mixed", 16, 64, 16, 2),
    ("long", 16, 128, 32, 8), ("long", 16, 64, 8, 8),
    # B = 4 runs the TMA page-box producer (the cp.async producer needs 8-row swizzle groups per page)
    ("eval", 4, 128, 32, 8), ("mixed", 4, 64, 16, 2), ("eval", 8, 128, 32, 8),
])
def test_shared_prefix_attention_vs_dense(kind, B, D, H, Hkv):
    starts, lens, tables, pool, qs, ks, vs = _case(kind, B, D, H, Hkv, seed=B + D + H)
    S = len(starts)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    M = int(cu[-1])
    maxb = max(len(t) for t in tables)
    bt = np.zeros((S, maxb), np.int32)
    for i, t in enumerate(tables):
        bt[i, :len(t)] = t
    st = np.asarray(starts, np.int32)
    cap = int(_native.lib.alora_attn_partial_capacity(H, D))
    out_plan = np.empty(1 << 20, np.int32)
    n = _native.lib.alora_plan_attention(S, cu.ctypes.data, st.ctypes.data, bt.ctypes.data, maxb, B, H, Hkv, D, 1,
                                         cap, out_plan.ctypes.data, out_plan.size)
    assert n > 0
    plan = out_plan[:n]
    n_items, n_segs, n_sets, max_np = (int(x) for x in plan[:4])
    if kind in ("eval", "decode"):
        assert n_sets == 3
    dev_pool = torch.as_tensor(pool).to("cuda", torch.bfloat16).contiguous()
    q = torch.as_tensor(np.concatenate(qs)).to("cuda", torch.bfloat16).contiguous()
    out = torch.empty_like(q)
    pos = torch.as_tensor(np.concatenate([np.arange(s, s + l) for s, l in zip(starts, lens)]).astype(np.int32)).cuda()
    row_seq = torch.as_tensor(np.repeat(np.arange(S), lens).astype(np.int32)).cuda()
    d_bt = torch.as_tensor(bt).cuda()
    d_plan = torch.as_tensor(plan).cuda()
    ws = torch.zeros(max(1, max_np * M * H * (D + 2) * 4), dtype=torch.uint8, device="cuda")
    rc = _native.lib.alora_paged_prefix_attn(
        q.data_ptr(), q.shape[1], M, S, pos.data_ptr(), row_seq.data_ptr(), d_bt.data_ptr(), maxb, d_plan.data_ptr(),
        n_items, n_segs, n_sets, max_np, dev_pool.data_ptr(), dev_pool.shape[0], 2, 1, B, H, Hkv, D, out.data_ptr(),
        out.shape[1], ws.data_ptr(), ws.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc, "alora_paged_prefix_attn")
    got = out.float().cpu().numpy()
    worst = 0.0
    for s in range(S):
        want = dense_reference_attention(qs[s], ks[s], vs[s], H, starts[s], Hkv)
        worst = max(worst, float(np.max(np.abs(got[cu[s]:cu[s + 1]] - want))))
    print(f"[parity] shared-prefix attention {kind} B={B} D={D} H={H}/{Hkv}: max |d| {worst:.3g} "
          f"(sets {n_sets} of {S} spans, items {n_items}, partitions {max_np})")
    assert worst < 3e-2


def test_shared_prefix_forward_matches_per_span_forward():
    """Model.forward_step with the shared-prefix plan vs the per-span kernels on the same step (C2-like widths,
    4 layers): logits within bf16 tolerance, written KV of the first layer identical (computed before attention),
    greedy ids equal where the margin decides."""
    dims = dict(arch="llama", n_layers=4, n_heads=32, n_kv_heads=8, head_dim=64, d_model=2048, ffn_dim=1024,
                vocab_size=2048, seed=3, max_seq_len=4096)
    cfg = P.ModelConfig(**dims, dtype="bf16")
    B, cached, suffix, n_conv, n_ad = 16, 2032, 20, 2, 3
    res = []
    for shared in (False, True):
        # "always": at these C2-like shapes the cost estimate alone would keep the per-span kernels
        model = P.Model(cfg, max_tokens=512, max_seqs=64, shared_prefix="always" if shared else False)
        nb = n_conv * (cached // B) + n_conv * n_ad * 2 + 4
        pool = P.BlockPool(nb, B, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
        g = torch.Generator(device="cuda").manual_seed(1)
        pool.kv.copy_(torch.randn(pool.kv.shape, generator=g, device="cuda").to(torch.bfloat16))
        rng = np.random.default_rng(0)
        seqs = []
        for c in range(n_conv):
            for k in range(n_ad):
                ad = P.generate_adapter(f"a{k}", cfg.d_model, 16, seed=k, invocation_tokens=(2016 + 3 * k, 2017 + 3 * k, 2018 + 3 * k),
                                        kv_width=cfg.kv_width, q_width=cfg.q_width)
                i = len(seqs)
                table = list(range(c * 127, (c + 1) * 127)) + [n_conv * 127 + 2 * i, n_conv * 127 + 2 * i + 1]
                toks = rng.integers(0, 2000, suffix)
                mask = np.arange(cached, cached + suffix) < cached + suffix - 3
                seqs.append(P.SeqInput(f"r{i}", toks, cached, table, ad, mask))
        p = model.pack(seqs, B)
        assert (p["attn_plan"] is not None) == shared
        out = model.forward_step(seqs, pool.kv)
        res.append((out, pool.kv[:, 0].float().cpu().numpy()))
    worst = max(float(np.max(np.abs(res[0][0][k] - res[1][0][k]))) for k in res[0][0])
    print(f"[parity] shared-prefix vs per-span forward: max |dlogit| {worst:.3g}")
    assert worst < 5e-2
    np.testing.assert_array_equal(res[0][1], res[1][1])
