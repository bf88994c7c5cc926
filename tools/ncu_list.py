"""Print an ncu launch-list CSV (gpu__time_duration.sum) as 'us grid kernel' lines
(python tools/ncu_list.py file.csv [substring filter] [last N])."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
flt = sys.argv[2] if len(sys.argv) > 2 else ""
last = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = [r for r in rows[1:] if flt in r[ki]]
for r in out[-last:]:
    print(f"{float(r[vi].replace(',', '')) / 1e3:8.1f} {r[gi] if gi is not None else '':>14} {r[ki][:90]}")
