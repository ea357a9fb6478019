"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
bi = hdr.index("Block Size") if "Block Size" in hdr else None
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in data:
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("hkd::", "")
    name = name.replace("unnamed>::", "")[:44]
    key = f"{name} g={r[gi]}" + (f" b={r[bi]}" if bi is not None else "")
    v = float(r[vi].replace(",", ""))
    agg[key][0] += 1
    agg[key][1] += v
    tot += v
print(f"launches {len(data)}  total {tot / 1e6:.3f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / tot * 100:5.1f}%  n={n:4d}  avg={t / n / 1e3:8.2f} us  {k}")
