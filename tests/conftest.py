"""Shared test setup.

Markers: `gpu` tests need a B200 (run with -m gpu on the GPU box); everything
else runs on CPU. Golden fixtures in tests/golden/ were produced by importing
the reference (oracle/gen_golden.py); nothing here reads /root/reference.
"""

import json
import os
import sys

# Tensor-parallel tests run several ranks as threads of one process on one GPU, each with its own streams,
# spinning in the fused all-reduce until every peer arrives. With the default 8 hardware work queues, 8 ranks'
# 16 streams share queues and a rank's kernels can sit behind a peer's spinning kernel (a false dependency
# that deadlocks until the barrier timeout). Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name))


C1 = dict(n_layers=2, n_heads=4, head_dim=64, d_model=256, vocab_size=256, seed=0)


def dense_reference_attention(q, k, v, n_heads, start_pos, n_kv_heads=None):
    """Per-head O(n^2) fp64 causal attention over a dense context (reference tests/conftest.py:15-35,
    generalised to GQA)."""
    n, dq = q.shape
    hkv = n_heads if n_kv_heads is None else n_kv_heads
    hd = dq // n_heads
    g = n_heads // hkv
    out = np.zeros((n, dq), dtype=np.float64)
    for h in range(n_heads):
        kh_i = h // g
        qh = q[:, h * hd:(h + 1) * hd].astype(np.float64)
        kh = k[:, kh_i * hd:(kh_i + 1) * hd].astype(np.float64)
        vh = v[:, kh_i * hd:(kh_i + 1) * hd].astype(np.float64)
        s = qh @ kh.T / np.sqrt(hd)
        for i in range(n):
            s[i, start_pos + i + 1:] = -np.inf
        e = np.exp(s - s.max(axis=1, keepdims=True))
        out[:, h * hd:(h + 1) * hd] = (e / e.sum(axis=1, keepdims=True)) @ vh
    return out.astype(np.float32)


def row_projection_oracle(x, w_mat, adapter, target, mask):
    """Row i of the masked projection computed on its own (reference tests/conftest.py:38-51)."""
    rows = []
    for i in range(len(x)):
        xi = x[i:i + 1].astype(np.float64)
        base = (xi @ w_mat.astype(np.float64)).astype(np.float32)
        if mask[i] or target not in adapter.targets:
            rows.append(base[0])
        else:
            down = adapter.down[target].astype(np.float64)
            up = adapter.up[target].astype(np.float64)
            delta = ((xi @ down).astype(np.float32).astype(np.float64) @ up).astype(np.float32)
            rows.append(base[0] + delta[0])
    return np.stack(rows)
