"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel count/mean/total (us)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi or "alora" not in r[ki] and "gemm_" not in r[ki] and "attn" not in r[ki] and "kernel" not in r[ki]:
        continue
    name = re.sub(r"\(.*", "", r[ki].replace("void ", "").replace("(anonymous namespace)::", ""))
    name = name.replace("alora::<unnamed>::", "").replace("alora::", "").replace("unnamed>::", "")[:44]
    v = float(r[vi].replace(",", ""))
    unit = r[ui].lower()
    v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    agg.setdefault(name, []).append(v)
    tot += v
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:46s} n={len(v):4d} mean={sum(v) / len(v):8.2f} us total={sum(v):9.1f} us")
print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
