import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ws = torch.zeros(lib.alora_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
def run(M, N, K, split, epi=0, reps=20, label=""):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: lib.alora_gemm_bf16(epi, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, ws.data_ptr() if split else None, ws.numel() if split else 0, st)
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()  # cold L2: weights come from HBM as in the forward
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    by = 2 * (M * K + N * K) + 2 * M * N
    print(f"{label:10s} M={M:5d} N={N:6d} K={K:5d} split={int(split)}: {t*1e6:8.2f} us  {by/t/1e9:8.1f} GB/s  {2*M*N*K/t/1e12:7.1f} TFLOP/s")
for split in (False, True):
    run(240, 3072, 2048, split, label="qkv")
    run(240, 2048, 2048, split, label="o")
    run(240, 16384, 2048, split, label="mlp_in")
    run(240, 2048, 8192, split, label="mlp_out")
    run(12, 2048, 8192, split, label="dec_out")
    run(12, 128256, 2048, split, label="lm_head")
run(8192, 3072, 2048, False, label="big_qkv")
run(8192, 16384, 2048, False, label="big_in")
run(8192, 2048, 8192, False, label="big_out")
