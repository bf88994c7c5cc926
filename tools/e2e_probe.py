import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c2_problem, random_kkt
p = c2_problem(); st = fw.GnState(p, exact=False)
hin = [np.ascontiguousarray(random_kkt(p, 31 + i)) for i in range(2)]; hout = np.empty(st.vec_len)
for a in hin + [hout]: fw.host_register(a)
fw.kkt_apply_host(st, hin[0], hout)
t0 = time.perf_counter()
for i in range(10): fw.kkt_apply_host(st, hin[i & 1], hout)
t = (time.perf_counter() - t0) / 10
print(f"e2e {1/t:.1f} applies/s  {t*1e3:.2f} ms/step  {2*st.vec_len*8/t/1e9:.1f} GB/s H2D+D2H")
# raw copy rates
import ctypes as C
L = fw.lib(); d = fw.KktVector(st)
t0 = time.perf_counter()
for i in range(5): d.upload(hin[0])
t = (time.perf_counter() - t0) / 5; print(f"H2D {st.vec_len*8/t/1e9:.1f} GB/s")
t0 = time.perf_counter()
for i in range(5): d.to_host(hout)
t = (time.perf_counter() - t0) / 5; print(f"D2H {st.vec_len*8/t/1e9:.1f} GB/s")
