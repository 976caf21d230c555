"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
st = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[st]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[st + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}[r[ui]]
    k = r[ki].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total us':>10s} {'share':>6s} {'avg us':>9s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{k[:60]:60s} {n:5d} {t:10.1f} {100 * t / tot:5.1f}% {t / n:9.1f}")
print(f"total {tot:.1f} us")
