import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2512_17910_b200 as P
from paper_2512_17910_b200 import kv_cache as K
toks=[np.random.randint(0,100000,2052).astype(np.int64) for _ in range(12)]
items=[(t,128,127,"adapter1") for t in toks]
def T(f, n=300):
    for _ in range(10): f()
    ts=[]
    for _ in range(n):
        t=time.perf_counter(); f(); ts.append(time.perf_counter()-t)
    return sorted(ts)[n//2]*1e6
for nt in (1,2,3,4,6,8):
    print("hash_requests threads", nt, round(T(lambda: K.hash_requests(items,16,nt)),1), "us")
import torch
print("after torch import (cuda init)")
torch.zeros(1, device="cuda")
for nt in (1,2,4):
    print("hash_requests threads", nt, round(T(lambda: K.hash_requests(items,16,nt)),1), "us")
