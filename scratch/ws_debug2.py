import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
M, N, K = [int(x) for x in sys.argv[1:4]]
reps = int(sys.argv[4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
ref = A.double() @ B.double().T
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
bad = 0
for i in range(reps):
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    rc = lib.alora_gemm_bf16(16, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 0, st)
    torch.cuda.synchronize()
    err = (C.double() - ref).abs().max().item()
    if not err < 1e-3:
        bad += 1
print(f"M={M} N={N} K={K}: {bad}/{reps} bad", flush=True)
