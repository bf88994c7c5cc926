"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    h, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            data.append(dict(zip(h, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:60]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1.0)
    tot = sum(x[1] for x in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:60s} {c:8d} {t:12.1f} {t / c:10.2f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
