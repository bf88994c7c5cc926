import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2204_06489_b200 import _abi, api as fw
from paper_2204_06489_b200.problem import c2_problem, small_problem, random_kkt
which, variant, prec = sys.argv[1], sys.argv[2], sys.argv[3]
p = {"small": lambda: small_problem(), "c2k5": lambda: c2_problem(K=5, R=17), "c2": lambda: c2_problem()}[which]()
os.environ["FWI_KKT_KERNEL"] = variant
st = fw.GnState(p, exact=False, c64=True)
x = random_kkt(p, 1)
if prec == "64":
    y = fw.kkt_apply(st, fw.KktVector.from_host(st, x)).to_host()
else:
    y = fw.kkt_apply(st, fw.KktVector.from_host(st, x.astype(np.float32), _abi.FWI_C64)).to_host()
st.synchronize()
print(which, variant, prec, os.environ.get("FWI_KKT_STAGES"), "ok", float(np.linalg.norm(y)))
