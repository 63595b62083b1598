"""Debug: shared-prefix attention case from tests/test_gpu_shared_prefix.py with split on/off, per-row errors."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_gpu_shared_prefix import _case
from conftest import dense_reference_attention
import paper_2512_17910_b200 as P
from paper_2512_17910_b200 import _native
kind, B, D, H, Hkv = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
for flags in (1, 3):
    starts, lens, tables, pool, qs, ks, vs = _case(kind, B, D, H, Hkv, seed=B + D + H)
    S = len(starts); cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32); M = int(cu[-1])
    maxb = max(len(t) for t in tables); bt = np.zeros((S, maxb), np.int32)
    for i, t in enumerate(tables): bt[i, :len(t)] = t
    st = np.asarray(starts, np.int32)
    out_plan = np.empty(1 << 20, np.int32)
    n = _native.lib.alora_plan_attention(S, cu.ctypes.data, st.ctypes.data, bt.ctypes.data, maxb, B, H, Hkv, D, flags,
                                         1 << 30, out_plan.ctypes.data, out_plan.size)
    plan = out_plan[:n]; n_items, n_segs, n_sets, max_np = (int(x) for x in plan[:4])
    dev_pool = torch.as_tensor(pool).to("cuda", torch.bfloat16).contiguous()
    q = torch.as_tensor(np.concatenate(qs)).to("cuda", torch.bfloat16).contiguous(); out = torch.empty_like(q)
    pos = torch.as_tensor(np.concatenate([np.arange(s, s + l) for s, l in zip(starts, lens)]).astype(np.int32)).cuda()
    row_seq = torch.as_tensor(np.repeat(np.arange(S), lens).astype(np.int32)).cuda()
    d_bt = torch.as_tensor(bt).cuda(); d_plan = torch.as_tensor(plan).cuda()
    ws = torch.zeros(max(1, max_np * M * H * (D + 2) * 4), dtype=torch.uint8, device="cuda")
    _native.check(_native.lib.alora_paged_prefix_attn(q.data_ptr(), q.shape[1], M, S, pos.data_ptr(), row_seq.data_ptr(), d_bt.data_ptr(), maxb, d_plan.data_ptr(),
        n_items, n_segs, n_sets, max_np, dev_pool.data_ptr(), dev_pool.shape[0], 2, 1, B, H, Hkv, D, out.data_ptr(),
        out.shape[1], ws.data_ptr(), ws.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "x")
    got = out.float().cpu().numpy()
    print(f"flags {flags}: items {n_items} sets {n_sets} parts {max_np}")
    for s in range(S):
        want = dense_reference_attention(qs[s], ks[s], vs[s], H, starts[s], Hkv)
        e = np.abs(got[cu[s]:cu[s + 1]] - want).reshape(lens[s], H, D).max(axis=(0, 2))
        print(f"  span {s} start {starts[s]} |want| {np.abs(want).max():.3g} err per head max {e.max():.3g} worst heads {np.argsort(-e)[:4]}")
