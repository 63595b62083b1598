"""Repeat the B=32 paged-attention case and report any run whose error exceeds the tolerance (race hunt)."""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import dense_reference_attention
import test_gpu_bf16_model as T
from paper_2512_17910_b200 import _native
H, Hkv, D, B, starts, lens = 32, 8, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 32, [100, 0, 1500], [40, 70, 9]
n = len(starts)
pool, tables, ks, vs, qs = T._attn_case(n, H, Hkv, D, B, starts, lens, seed=H + D + B)
want = [dense_reference_attention(qs[s], ks[s], vs[s], H, starts[s], Hkv) for s in range(n)]
dev_pool = torch.as_tensor(pool).to("cuda", torch.bfloat16).contiguous()
q = torch.as_tensor(np.concatenate(qs)).to("cuda", torch.bfloat16).contiguous()
M = q.shape[0]
maxb = max(len(t) for t in tables)
bt = np.zeros((n, maxb), np.int32)
for i, t in enumerate(tables): bt[i, :len(t)] = t
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
d_cu, d_sp, d_bt = (torch.as_tensor(a).cuda() for a in (cu, np.asarray(starts, np.int32), bt))
max_q, max_ctx = max(lens), max(s + l for s, l in zip(starts, lens))
wsb = _native.lib.alora_attn_workspace_bytes(_native.ALORA_BF16, M, n, max_q, max_ctx, H, Hkv, D)
ws = torch.zeros(max(int(wsb), 1), dtype=torch.uint8, device="cuda")
bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 300):
    out = torch.full_like(q, float("nan"))
    rc = _native.lib.alora_paged_prefill_attn(_native.ALORA_BF16, q.data_ptr(), q.shape[1], M, n, d_cu.data_ptr(),
        d_sp.data_ptr(), d_bt.data_ptr(), maxb, max_q, max_ctx, dev_pool.data_ptr(), dev_pool.shape[0], 2, 1, B, H, Hkv,
        D, out.data_ptr(), out.shape[1], ws.data_ptr(), ws.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc, "attn")
    got = out.float().cpu().numpy()
    for s in range(n):
        err = np.abs(got[cu[s]:cu[s + 1]] - want[s])
        e = float(np.nanmax(err)) if not np.isnan(err).any() else float("inf")
        if e > 3e-2:
            bad += 1
            r, c = np.unravel_index(np.nanargmax(np.where(np.isnan(err), np.inf, err)), err.shape)
            print(f"iter {it}: seq {s} err {e:.4f} at token {r} head {c // D} dim {c % D}", flush=True)
print(f"B={B}: {bad} bad of {it + 1}")
