"""North-star residual-history gate on config 1 (VERDICT r1 "next" #1).

For the exact, ILU(4) and ILU(21) preconditioners: tol = 0, maxit = 50,
restart = 30 (the restart at j = 30 is crossed), ecg_stride = 0. Records the
reference's history (oracle/_ref), the reference's history with b perturbed by
1e-15 relative (its own rounding-noise yardstick: the residual r, from which
kkt_rhs builds b, scaled elementwise by 1 + 1e-15 N(0,1)) and the device
history, all 51 entries, with no floor.

    python tools/history_gate.py [out.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import pyoracle as po  # noqa: E402
from paper_2204_06489_b200 import api as fw  # noqa: E402
from paper_2204_06489_b200.problem import c1_problem  # noqa: E402


def main():
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    base = po.Ref(p, full=True, exact=True, ilu_level=4)
    u, r = base.u(), base.residual()
    out = {}
    for name, mode, level in (("exact", fw.PrecondMode.exact, 4), ("ilu4", fw.PrecondMode.ilu, 4),
                              ("ilu21", fw.PrecondMode.ilu, 21)):
        q = c1_problem()
        q.u, q.r = u, r
        ref = po.Ref(q, full=False, exact=True, ilu_level=level)
        qp = c1_problem()
        rng = np.random.default_rng(77)
        qp.u, qp.r = u, r * (1.0 + 1e-15 * rng.standard_normal(r.shape))
        refp = po.Ref(qp, full=False, exact=True, ilu_level=level)
        dev = fw.GnState(q, exact=True, ilu_level=level)
        opts = dict(restart=30, tol=0.0, maxit=50, ecg_stride=0)
        _, lr = ref.fsgn(int(mode), 30, 0.0, 50, 0)
        _, lp = refp.fsgn(int(mode), 30, 0.0, 50, 0)
        _, ld = fw.fsgn_gmres_step(dev, fw.FsgnOptions(mode=mode, **opts))
        hr, hp, hd = (np.array(x.residuals()) for x in (lr, lp, ld))
        dd = np.abs(hd - hr) / hr
        dp = np.abs(hp - hr) / hr
        out[name] = {"entries": len(hr), "ref": hr.tolist(), "ref_perturbed": hp.tolist(), "dev": hd.tolist(),
                     "dev_dev": dd.tolist(), "ref_drift": dp.tolist(), "max_dev": float(dd.max()),
                     "argmax_dev": int(dd.argmax()), "max_ref_drift": float(dp.max())}
        print(name, "entries", len(hr), "max dev", dd.max(), "at", dd.argmax(), "ref drift", dp.max(),
              flush=True)
        print("  dev  per it:", " ".join(f"{x:.1e}" for x in dd))
        print("  drift per it:", " ".join(f"{x:.1e}" for x in dp))
        dev.close()
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "history_gate.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
