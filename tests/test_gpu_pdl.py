"""Programmatic dependent launch (csrc/common.cuh launch_pdl / pdl_enter) changes scheduling only:
the same GMRES solves (exact with cyclic reduction and with the Schur sweeps, ILU) and KKT applies
give bit-identical results with FWI_PDL=0 (plain stream launches) and with it on (the default).
The switch is read once per process, so each setting runs in its own subprocess."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2204_06489_b200 import api as fw
from paper_2204_06489_b200.problem import c1_problem, c2_problem, random_kkt, small_problem
h = hashlib.sha256()
q = c1_problem()
q.d_obs = fw.simulate(q)
st = fw.GnState(q, exact=True, ilu_level=4)
for mode in (fw.PrecondMode.exact, fw.PrecondMode.ilu):
    ds, log = fw.fsgn_gmres_step(st, fw.FsgnOptions(mode=mode, tol=0.0, maxit=35, restart=30, ecg_stride=0))
    h.update(np.asarray(ds).tobytes()); h.update(np.array(log.residuals()).tobytes())
st.close()
os.environ["FWI_EXACT_BCR"] = "1"
p = small_problem(nx=40, nz=26, n_pml=4, K=3, R=5)
s2 = fw.GnState(p, exact=True)
ds, log = fw.fsgn_gmres_step(s2, fw.FsgnOptions(tol=1e-8, maxit=20, ecg_stride=0))
h.update(np.asarray(ds).tobytes()); h.update(np.array(log.residuals()).tobytes())
c = c2_problem(K=8, R=17)
s3 = fw.GnState(c, exact=False)
h.update(fw.kkt_apply(s3, fw.KktVector.from_host(s3, random_kkt(c, 5))).to_host().tobytes())
print("HASH", h.hexdigest())
""" % ROOT


def run(pdl):
    env = {**os.environ, "FWI_PDL": pdl}
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.startswith("HASH")][0]


def test_dependent_launch_bit_identical_to_plain_launch():
    assert run("1") == run("0")
