import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ws = torch.zeros(lib.alora_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")


def run(M, N, K, ms, epi=0, reps=15, label="", cold=True):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: lib.alora_gemm_bf16(epi, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, ws.data_ptr() if ms > 1 else None, ws.numel() if ms > 1 else 0, st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    by = 2 * N * K
    print(f"{label:8s} M={M:4d} N={N:5d} K={K:5d} max_splits={ms} cold={int(cold)}: {t*1e6:7.2f} us  weights {by/t/1e9:7.1f} GB/s")


for cold in (True,):
    for ms in (1, 8):
        run(240, 2048, 2048, ms, label="o", cold=cold)
for ms in (1, 8):
    run(12, 2048, 8192, ms, label="dec_out")
for ms in (1, 8):
    run(128, 2048, 8192, ms, label="m128out")
for ms in (1, 8):
    run(240, 3072, 2048, ms, label="qkv")
    run(240, 16384, 2048, ms, label="mlp_in")
    run(240, 2048, 8192, ms, label="mlp_out")
    run(12, 3072, 2048, ms, label="dec_qkv")
    run(12, 16384, 2048, ms, label="dec_in")
