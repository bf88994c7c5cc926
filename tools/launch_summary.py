"""Summarise an ncu launch-list CSV (gpu__time_duration.sum): total and per-kernel time."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:60]
    ns = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += ns
    tot += ns
print(f"{len(rows) - 1} launches, {tot / 1e6:.3f} ms total kernel time")
for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ns / 1e6:9.3f} ms {100 * ns / tot:5.1f}%  x{n:5d}  {k}")
