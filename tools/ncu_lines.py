"""Summarise an ncu source page (cuda,sass CSV) per CUDA line: samples, top stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(k for k, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
data = rows[hi + 1:]
wi = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
stall_cols = [k for k, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = 0.0
out = []
for r in data:
    if r and r[0] != "" and len(r) > wi:
        try:
            smp = float(r[wi])
        except ValueError:
            continue
        tot += smp
        st = sorted(((float(r[k] or 0), h[k][6:]) for k in stall_cols), reverse=True)[:3]
        out.append((r[0], smp, r[ie], r[1], st))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
print("total samples", tot)
for ln, smp, ie_, src, st in out:
    if smp / tot * 100 >= thr:
        print(f"{ln:>5} {smp / tot * 100:5.1f}% {ie_:>9}  {src.strip()[:70]:70s} " +
              " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0))
