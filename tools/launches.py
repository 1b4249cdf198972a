"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
total / count / mean per kernel (cold-cache, serialised: compare shares)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) > iv:
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[iu], 1.0)
        d[r[ik][:100]].append(v)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v) / 1e3:9.3f} ms {100 * sum(v) / tot:5.1f}%  n={len(v):4d}  mean={sum(v) / len(v):9.1f} us  {k}")
print(f"total {tot / 1e3:.3f} ms")
