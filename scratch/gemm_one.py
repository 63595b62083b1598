import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
M, N, K = (int(a) for a in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    lib.alora_gemm_bf16(0, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 0, st)
torch.cuda.synchronize()
