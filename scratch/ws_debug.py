import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
M, N, K = [int(x) for x in sys.argv[1:4]]
epi = int(sys.argv[4]) if len(sys.argv) > 4 else 16
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (1, 16) else torch.bfloat16)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
rc = lib.alora_gemm_bf16(epi, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 0, st)
torch.cuda.synchronize()
ref = A.double() @ B.double().T
print("rc", rc, "maxerr", (C.double() - ref).abs().max().item())
