"""Host-buffer KKT apply (fwi_dev_kkt_apply_host, config 2) against the number of source chunks it
pipelines through H2D / apply / D2H (FWI_HOST_CHUNKS; page-locked buffers from fwi_host_alloc, as
the bench). python tools/e2e_chunks.py"""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import time
    from paper_2204_06489_b200 import api as fw
    from paper_2204_06489_b200.problem import c2_problem, random_kkt
    p = c2_problem()
    st = fw.GnState(p, exact=False)
    hin = []
    for i in range(2):
        a = fw.host_empty(st.vec_len)
        a[:] = random_kkt(p, 31 + i)
        hin.append(a)
    hout = fw.host_empty(st.vec_len)
    fw.kkt_apply_host(st, hin[0], hout)
    best = 0.0
    for rep in range(3):
        t0 = time.perf_counter()
        for i in range(10):
            fw.kkt_apply_host(st, hin[i & 1], hout)
        best = max(best, 10 / (time.perf_counter() - t0))
    print(f"chunks {sys.argv[1]}: {best:.1f} applies/s")
else:
    for ch in (16, 32, 64, 8):
        subprocess.run([sys.executable, __file__, str(ch)], env={**os.environ, "FWI_HOST_CHUNKS": str(ch)})
