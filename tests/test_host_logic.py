"""CPU: host-side logic — synthetic configurations, PML profile, survey
validity, and the multi-rank (replicas) timing logic of bench.py on gloo."""
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_06489_b200 import _abi  # noqa: E402
from paper_2204_06489_b200.problem import (Grid, c1_problem, c2_problem, omega_of, pml_sigma_max,  # noqa: E402
                                           random_kkt, small_problem)


def test_pml_profile_formula():
    """make_pml_profile (src/grid.cpp:21-33)."""
    g = Grid(128, 64, 25.0, 10)
    assert pml_sigma_max(g, 2000.0) == 3.0 * 2000.0 * math.log(1e3) / (2.0 * 10 * 25.0)
    assert pml_sigma_max(Grid(8, 8, 1.0, 0), 1.0) == 0.0
    with pytest.raises(ValueError):
        pml_sigma_max(g, 0.0)


@pytest.mark.parametrize("mk", [c1_problem, c2_problem, small_problem])
def test_surveys_sit_on_usable_nodes(mk):
    """Survey::validate (src/forward.cpp:23-41): core, off the Dirichlet ring."""
    p = mk()
    g, sv = p.grid, p.survey
    g.validate()
    for k in range(sv.num_sources):
        assert g.usable_node(int(sv.src_ix[k]), int(sv.src_iz[k]))
        for j in range(sv.recv_offset[k], sv.recv_offset[k + 1]):
            assert g.usable_node(int(sv.recv_ix[j]), int(sv.recv_iz[j]))
    assert np.all(p.s > 0) and np.all(np.isfinite(p.s))


def test_baseline_config_shapes():
    p1, p2 = c1_problem(), c2_problem()
    assert (p1.grid.nx, p1.grid.nz, p1.grid.n_pml, p1.K, p1.survey.num_data // p1.K) == (128, 64, 10, 8, 64)
    assert (p2.grid.nx, p2.grid.nz, p2.grid.n_pml, p2.K, p2.survey.num_data // p2.K) == (512, 256, 20, 64, 256)
    assert p1.freq_hz == 5.0 and p2.freq_hz == 8.0
    assert p2.vec_len == 4 * 64 * 512 * 256 + 512 * 256
    assert omega_of(5.0) == 2.0 * math.pi * 5.0
    # seeded: reproducible inputs
    assert np.array_equal(random_kkt(p2, 3)[:100], random_kkt(p2, 3)[:100])


def test_offset_weights_formula():
    """build_weights offset mode (src/forward.cpp:43-62)."""
    p = small_problem(weight_mode=_abi.FWI_WEIGHT_OFFSET)
    w = p.survey.weights()
    assert w.max() == 1.0 and np.all(w > 0)


def _replica_worker(rank, ws, port, q):
    import time

    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bench
    import pyoracle as po
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    p = small_problem(seed=rank)  # each replica owns an independent instance
    o = po.Orc(p, exact=False)
    x = random_kkt(p, 9)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(3 + rank):  # uneven work: the max over ranks must win
        o.kkt_apply(x)
    t = time.perf_counter() - t0
    tmax = bench.barrier_max_cpu(t, ws)
    q.put((rank, t, tmax))
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29517
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    ts = {r: t for r, t, _ in res}
    for _, _, tmax in res:
        assert tmax == pytest.approx(max(ts.values()))


def test_host_alloc_symbols_declared():
    """fwi_host_alloc/free are part of the C ABI (page-locked buffers for the host apply)."""
    import re
    hdr = open(os.path.join(ROOT, "include", "fwi_b200.h")).read()
    assert re.search(r"int fwi_host_alloc\(void\*\* out, int64_t bytes\);", hdr)
    assert re.search(r"int fwi_host_free\(void\* host\);", hdr)
