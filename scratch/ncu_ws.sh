#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2512_17910_b200 import _native
lib = _native.lib
M, N, K = 240, 2048, 8192
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    lib.alora_gemm_bf16(1, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 0, st)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_ws -s 1 -c 1 -o gpurun_out/prof_ws -f python /tmp/one.py > gpurun_out/ncu_ws.log 2>&1
tail -3 gpurun_out/ncu_ws.log
