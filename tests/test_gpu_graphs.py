"""Decode steps replay a captured CUDA graph of the whole native forward (alora_model_forward_graph).

Graph replay (bucketed block table, one capture per bucket) must give the same greedy tokens as the
eager executor and logits within the bf16 tolerance (the bucketed context bound changes the attention's
split-KV partitioning, hence the fp32 summation order), over decode steps that cross block boundaries,
with an activated adapter, a standard LoRA and a base request in the same batch.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")

LLAMA = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512,
             vocab_size=384, seed=4, dtype="bf16")


def _run(graphs: bool, steps: int = 24):
    cfg = P.ModelConfig(**LLAMA)
    model = P.Model(cfg, graphs=graphs)
    V = cfg.vocab_size
    inv = (V - 32, V - 31, V - 30)
    act = P.generate_adapter("a0", cfg.d_model, 16, seed=1, invocation_tokens=inv, kv_width=cfg.kv_width,
                             q_width=cfg.q_width)
    std = P.generate_adapter("a1", cfg.d_model, 8, seed=2, mode="standard", kv_width=cfg.kv_width,
                             q_width=cfg.q_width)
    pool = P.BlockPool(64, 16, cfg.n_layers, cfg.d_model, kv_width=cfg.kv_width, dtype="bf16")
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, V - 32, 37), np.concatenate([rng.integers(0, V - 32, 20), inv, [5, 6]]),
               rng.integers(0, V - 32, 29)]
    adapters = [None, act, std]
    tables = [list(range(0, 8)), list(range(8, 16)), list(range(16, 24))]

    def span(r, toks, start):
        a = adapters[r]
        mask = None
        if a is act:
            mask = np.arange(start, start + len(toks)) < 20
        return P.SeqInput(f"r{r}", toks, start, tables[r], a, mask)

    out = model.forward_step([span(r, prompts[r], 0) for r in range(3)], pool.kv)
    lens = [len(p) for p in prompts]
    nxt = {k: int(np.argmax(v)) for k, v in out.items()}
    ids, logits = [], []
    for t in range(steps):
        out = model.forward_step([span(r, np.array([nxt[f"r{r}"]]), lens[r] + t) for r in range(3)], pool.kv)
        nxt = {k: int(np.argmax(v)) for k, v in out.items()}
        ids.append([nxt[f"r{r}"] for r in range(3)])
        logits.append(np.stack([out[f"r{r}"] for r in range(3)]))
    torch.cuda.synchronize()
    return np.array(ids), np.stack(logits), model.last_launches


def test_decode_graph_replay_matches_eager():
    ids_g, lg_g, n_g = _run(True)
    ids_e, lg_e, n_e = _run(False)
    assert n_g == n_e > 0  # the replayed graph holds the same launches
    np.testing.assert_array_equal(ids_g, ids_e)
    assert float(np.max(np.abs(lg_g - lg_e))) < 5e-2
