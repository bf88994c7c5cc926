"""Per-CTA timeline of the one-band source-major K1 (FWI_KKT_KM_TRACE): when each CTA starts,
enters and leaves its source loop and ends, by globaltimer, on which SM. Diagnostics only.
usage: python tools/k1_timeline.py [c128|c64] [out.json]"""
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.join(tempfile.gettempdir(), "fwi_km_trace.txt")
os.environ["FWI_KKT_KM_TRACE"] = path
from paper_2204_06489_b200 import _abi  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c2_problem, random_kkt  # noqa: E402

c64 = len(sys.argv) > 1 and sys.argv[1] == "c64"
p = c2_problem()
st = fw.GnState(p, exact=False, c64=c64)
prec = _abi.FWI_C64 if c64 else _abi.FWI_C128
xs = [fw.KktVector.from_host(st, random_kkt(p, 1 + i).astype("float32" if c64 else "float64"), prec) for i in range(2)]
ys = [fw.KktVector(st, prec) for _ in range(2)]
runs = []
for i in range(12):
    fw.kkt_apply(st, xs[i & 1], ys[i & 1])
    st.synchronize()
    if i >= 4:
        runs.append(np.loadtxt(path, dtype=np.int64))
out = {"kernel": st.kkt_kernel(prec).split(" (")[0], "launches": []}
for t in runs:
    t0 = t[:, 1].min()
    start, loop0, loop1, end = (t[:, j] - t0 for j in (1, 2, 3, 4))
    span = float(end.max())
    life = end - start
    out["launches"].append({
        "span_us": span / 1e3,
        "start_skew_us": float(start.max()) / 1e3,
        "prologue_us_mean": float((loop0 - start).mean()) / 1e3,
        "loop_us": {"min": float((loop1 - loop0).min()) / 1e3, "mean": float((loop1 - loop0).mean()) / 1e3,
                    "max": float((loop1 - loop0).max()) / 1e3},
        "end_us": {"min": float(end.min()) / 1e3, "p10": float(np.percentile(end, 10)) / 1e3,
                   "median": float(np.median(end)) / 1e3, "p90": float(np.percentile(end, 90)) / 1e3,
                   "max": span / 1e3},
        "mean_lifetime_over_span": float(life.mean()) / span,
        "ctas": int(len(t)), "sms_used": int(len(set(t[:, 5].tolist()))),
    })
last = runs[-1]
t0 = last[:, 1].min()
out["last_launch_ctas"] = [{"cta": int(r[0]), "sm": int(r[5]), "start": int(r[1] - t0), "loop0": int(r[2] - t0),
                            "loop1": int(r[3] - t0), "end": int(r[4] - t0)} for r in last]
js = json.dumps(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(js)
for l in out["launches"]:
    print(json.dumps(l))
