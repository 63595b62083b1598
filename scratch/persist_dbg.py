import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
M, N, K, epi = [int(x) for x in sys.argv[1:5]]
A = (torch.randn(M, K, device="cuda") * 0.1).to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
out_cols = N // 2 if epi == 3 else N
C = torch.empty(M, out_cols, device="cuda", dtype=torch.float32 if epi == 16 else torch.bfloat16)
ws = torch.zeros(lib.alora_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
rc = lib.alora_gemm_bf16(epi, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), out_cols, M, N, K, None, 0,
                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("rc", rc, "ok")
