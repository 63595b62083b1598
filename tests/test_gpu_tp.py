"""Tensor-parallel native forward on one B200: two TPModel ranks (threads, own CUDA streams) vs unsharded.

The ranks run the sm_100a executor on their shards (half the q/kv heads, half the FFN) and meet in
alora_model_forward's tp_allreduce hook after the row-parallel O-projection and MLP-down
(tp.ThreadGroup: a device-side sum in rank order). Logits, greedy ids and each rank's slice of the
paged KV cache must match the unsharded bf16 model within the bf16 tolerance of SURVEY.md §8(c).
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")

CFG = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=4, head_dim=64, d_model=512, ffn_dim=1024,
           vocab_size=512, max_seq_len=512, seed=0, dtype="bf16")


def _spans(cfg, adapter):
    rng = np.random.default_rng(5)
    inv = adapter.invocation_tokens
    toks = np.concatenate([rng.integers(0, 480, 45), inv, rng.integers(0, 480, 6)])
    n = len(toks)
    pre = P.SeqInput("r0", toks[:33], 0, list(range(4)))  # base prefix (adapter off)
    mask = np.arange(33, n) < 45  # activated after the invocation
    suf = P.SeqInput("r0", toks[33:], 33, list(range(4)), adapter, mask)
    return pre, suf


def test_tp2_threaded_ranks_match_unsharded_model():
    cfg = P.ModelConfig(**CFG)
    ad = P.generate_adapter("adapter0", cfg.d_model, 8, seed=1, invocation_tokens=(500, 501, 502),
                            kv_width=cfg.kv_width, q_width=cfg.q_width)
    full = P.Model(cfg)
    pool = P.BlockPool(8, 16, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
    pre, suf = _spans(cfg, ad)
    full.forward_step([pre], pool.kv)
    want = full.forward_step([suf], pool.kv)["r0"]

    group = P.ThreadGroup(2)
    ranks = [P.TPModel(cfg, group.rank_view(r)) for r in range(2)]
    pools = [P.BlockPool(8, 16, cfg.n_layers, cfg.d_model, kv_width=m.pool_kv_width, dtype="bf16") for m in ranks]
    out, errs = [None, None], []

    def run(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                ranks[r].forward_step([pre], pools[r].kv)
                out[r] = ranks[r].forward_step([suf], pools[r].kv)["r0"]
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    assert all(t is not None for t in out)
    np.testing.assert_array_equal(out[0], out[1])  # every rank ends with the same (all-reduced) logits
    err = float(np.max(np.abs(out[0] - want)))
    assert err < 5e-2, err
    assert int(np.argmax(out[0])) == int(np.argmax(want))
    # each rank caches exactly its kv heads: [.., kv_width] = [rank0 heads | rank1 heads]
    full_kv = pool.kv[:4].float().cpu().numpy()
    w = ranks[0].pool_kv_width
    for r in range(2):
        got = pools[r].kv[:4].float().cpu().numpy()
        ref = full_kv[..., r * w:(r + 1) * w]
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-2, (r, rel)
