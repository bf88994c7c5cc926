"""Per-kernel split of an ncu launch list with time and DRAM bytes (one GMRES solve)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")[:48]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot = sum(a[1] for a in agg.values())
print(f"{len(per)} launches, kernel time {tot / 1e6:.3f} ms total, {tot / 1e3 / iters:.1f} us per iteration ({iters} its)")
print(f"{'kernel':50s} {'launches':>8s} {'ms':>8s} {'share':>6s} {'us/it':>8s} {'DRAM GB':>8s} {'GB/s':>8s}")
for k, (n, ns, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {n:8d} {ns / 1e6:8.3f} {100 * ns / tot:5.1f}% {ns / 1e3 / iters:8.1f} {b / 1e9:8.3f} {b / ns if ns else 0:8.1f}")
