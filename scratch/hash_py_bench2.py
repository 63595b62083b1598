import time, numpy as np, sys, os
sys.path.insert(0, '.')
from paper_2512_17910_b200 import kv_cache as K
hist=[np.random.randint(0,100000,2048) for _ in range(4)]
items=[(np.concatenate([hist[i//3],[1,2,3,4]]).astype(np.int64),128,128,f"adapter{i%3}") for i in range(12)]
def T(f,n=200, gap=0):
    for _ in range(10): f()
    ts=[]
    for _ in range(n):
        if gap: time.sleep(gap)
        t=time.perf_counter(); f(); ts.append(time.perf_counter()-t)
    return round(sorted(ts)[n//2]*1e6,1)
for nt in (1,4):
    print("threads", nt, "tight", T(lambda: K.hash_requests(items,16,nt)), "us; with 20ms gaps", T(lambda: K.hash_requests(items,16,nt), n=50, gap=0.02), "us")
