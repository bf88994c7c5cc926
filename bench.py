#!/usr/bin/env python3
"""bench.py — throughput of the B200 KKT/Krylov hot path (BASELINE.json metric).

Default (N=1): BASELINE config 2 — the isolated, source-batched KKT operator
apply on a 512x256 grid (20-cell PML), K=64 sources, 256 receivers, complex128.
One step = one fused KKT apply over all sources with inputs resident in HBM.
The JSON line also carries the complex64 apply, the Krylov iteration
throughput of BASELINE config 1 (exact, ILU(4) and ILU(21) preconditioners)
and config 3 (exact) with its algorithmic HBM fraction, the end-to-end number
through the C ABI with host buffers, and the reference's CPU baselines (its
kkt_apply on all host threads and its fsgn_gmres_step on config 1, serial),
timed on the same host in the same run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU kkt_apply (oracle/_ref, the
unmodified reference core) on the same config with all host threads.
Multi-GPU: replicas only (the north star fixes one GPU).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KKT applies/sec and Krylov iters/sec at 1 B200; achieved HBM GB/s vs peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML while running."""
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def timed_events(stream_ptr, fn, steps):
    """CUDA-event time of `steps` calls of fn() on the library's own stream."""
    import torch
    s = torch.cuda.ExternalStream(stream_ptr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for i in range(steps):
        fn(i)
    e1.record(s)
    e1.synchronize()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def barrier_max(t, ws):
    if ws == 1:
        return t
    import torch
    import torch.distributed as dist
    x = torch.tensor([t], dtype=torch.float64, device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


def barrier_max_cpu(t, ws):
    """Max over ranks of a host time on an initialised (gloo) process group."""
    if ws == 1:
        return t
    import torch
    import torch.distributed as dist
    x = torch.tensor([t], dtype=torch.float64)
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def bench_config(ws, n):
    """The config dict both arms print (identical keys and values)."""
    return {"workload": "C2: isolated batched KKT apply, 512x256 grid, 20-cell PML, "
                        "K=64 sources, R=256 receivers, complex128",
            "nx": 512, "nz": 256, "K": 64, "R": 256, "n": n,
            "l2": "inputs larger than L2 (2 alternating 270 MB input vectors + 134 MB u "
                  "+ 2 outputs per step pair)",
            "parallelism": f"replicas x{ws}"}


def krylov_alg_bytes(st, log, restart, mode):
    """Algorithmic HBM bytes of one fsgn_gmres_step solve: per iteration j
    (0-based in its restart cycle) 2 KKT applies + 1 preconditioner apply + (5j + 11) KKT
    vectors (fused MGS 4(j+1), norm/scale 3, x_cand j+3, b for the true residual 1); per
    cycle one apply + preconditioner + 3 vectors; once the preconditioned b. Preconditioner
    = factor bytes read once per batched sweep (exact: 2 sweeps x 2 solves over the block
    factor; ILU: the 4 stored sweeps L, U, U^T, L^T once) + 64 K n (RHS and solution of both
    solves) + 16 n (the ds row)."""
    n, K = st.n, st.K
    V = st.vec_len * 8
    A = 80 * K * n + 24 * n
    F = 4 * st.exact_factor_bytes if mode == "exact" else st.ilu_factor_bytes
    P = F + 64 * K * n + 16 * n
    N = log.iterations()
    total = P + V
    total += math.ceil(N / restart) * (A + P + 3 * V)
    for k in range(N):
        j = k % restart
        total += 2 * A + P + (5 * j + 11) * V
    return total


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2204_06489_b200 import _abi
    from paper_2204_06489_b200 import api as fw
    from paper_2204_06489_b200.problem import c1_problem, c2_problem, c3_problem, random_kkt

    peak, peak_src = peaks()
    p = c2_problem()
    st = fw.GnState(p, exact=False, c64=True)
    n, K = p.n, p.K
    alg_bytes = 80 * K * n + 24 * n            # complex128 per apply
    alg_bytes32 = 40 * K * n + 12 * n
    xs = [fw.KktVector.from_host(st, random_kkt(p, 11 + i)) for i in range(2)]
    ys = [fw.KktVector(st) for _ in range(2)]
    L = fw.lib()
    sp = st.stream_ptr()

    def step(i):
        fw._check(L.fwi_dev_kkt_apply(st.h, xs[i & 1].h, ys[i & 1].h))

    for i in range(args.warmup):
        step(i)
    st.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        t = timed_events(sp, step, args.steps)
    t = barrier_max(t, ws)
    per = t / args.steps
    kname = st.kkt_kernel(_abi.FWI_C128)
    value = ws * args.steps / t
    achieved = alg_bytes / per / 1e9

    # complex64 apply (reported separately)
    xs32 = [fw.KktVector.from_host(st, random_kkt(p, 21 + i).astype(np.float32), _abi.FWI_C64)
            for i in range(2)]
    ys32 = [fw.KktVector(st, _abi.FWI_C64) for _ in range(2)]

    def step32(i):
        fw._check(L.fwi_dev_kkt_apply(st.h, xs32[i & 1].h, ys32[i & 1].h))

    for i in range(args.warmup):
        step32(i)
    t32 = barrier_max(timed_events(sp, step32, args.steps), ws)
    per32 = t32 / args.steps
    kname32 = st.kkt_kernel(_abi.FWI_C64)

    # end to end through the C ABI on host buffers (the reference's value-in /
    # value-out kkt_apply): pinned host in -> device -> host out, every step
    e2e_steps = max(3, min(args.steps, 20))
    hin = []
    for i in range(2):  # page-locked host buffers (cudaHostAlloc through the C ABI)
        a = fw.host_empty(st.vec_len)
        a[:] = random_kkt(p, 31 + i)
        hin.append(a)
    hout = fw.host_empty(st.vec_len)

    def e2e_step(i):
        fw.kkt_apply_host(st, hin[i & 1], hout)

    e2e_step(0)
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e_step(i)
    te = barrier_max(time.perf_counter() - t0, ws)
    del hin, hout
    vec_bytes = st.vec_len * 8

    # Krylov iterations/s on BASELINE config 1 (exact, ILU(4) and ILU(21) preconditioners) and
    # config 3 (exact), with the algorithmic HBM bytes of each solve against the peak
    krylov = {}
    if not args.skip_krylov:
        def time_solve(state, mode, label, cfg):
            o = fw.FsgnOptions(mode=mode, restart=30, tol=1e-3, maxit=60, ecg_stride=0)
            for _ in range(2):  # warm-up with the timed options (workspace, plans, clocks)
                fw.fsgn_gmres_step(state, o)
            runs = []
            for _ in range(5):
                t0 = time.perf_counter()
                ds, log = fw.fsgn_gmres_step(state, o)
                runs.append((log.entries[-1].wall_time, time.perf_counter() - t0, log))
            runs.sort(key=lambda r: r[0])
            wt, tw, log = runs[2]
            it = log.iterations()
            byt = krylov_alg_bytes(state, log, 30, "exact" if mode == fw.PrecondMode.exact else "ilu")
            krylov[label] = {"config": cfg, "iterations": it, "converged": log.converged,
                             "final_residual": log.final_residual(), "iters_per_s": it / wt,
                             "ms_per_iter": wt / it * 1e3, "solve_wall_s": wt, "step_wall_s": tw,
                             "alg_bytes_per_solve": byt, "achieved_gbs": byt / wt / 1e9,
                             "hbm_frac": byt / wt / 1e9 / peak,
                             "timing": "median of 5 solves after 2 warm-up solves, ConvergenceLog wall time; "
                                       "bytes: SURVEY 8(d) per-iteration formula (krylov_alg_bytes)"}

        q = c1_problem()
        q.d_obs = fw.simulate(q)
        c1cfg = "C1 128x64, K=8, 5 Hz, eps=1e10, tol 1e-3, restart 30, maxit 60"
        s1 = fw.GnState(q, exact=True, ilu_level=4)
        time_solve(s1, fw.PrecondMode.exact, "exact", c1cfg)
        time_solve(s1, fw.PrecondMode.ilu, "ilu", c1cfg + ", ILU(4)")
        s1.close()
        s21 = fw.GnState(q, exact=True, ilu_level=21)
        time_solve(s21, fw.PrecondMode.ilu, "ilu21", c1cfg + ", ILU(21)")
        s21.close()
        # config 3 (384x128, K=48, 3 Hz, exact preconditioner, eps = 1e-2 ||J^H J|| = 2.8e10)
        q3 = c3_problem(freq_hz=3.0)
        q3.d_obs = fw.simulate(q3)
        q3.epsilon = 2.8e10
        s3 = fw.GnState(q3, exact=True)
        time_solve(s3, fw.PrecondMode.exact, "c3_exact",
                   "C3 384x128, K=48, 3 Hz, eps=2.8e10, tol 1e-3, restart 30, maxit 60")
        s3.close()

    cpu = None
    if rank == 0 and not args.skip_cpu:
        cpu = cpu_baseline_apply(p, sample_applies=None)
        if not args.skip_krylov:
            cpu["krylov"] = cpu_baseline_krylov()

    if rank == 0:
        tr = load_traffic().get("kkt_apply_c128_c2")
        line = {
            "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded; BASELINE config 2 shapes and distributions)",
            "config": bench_config(ws, n),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "frac_of_datasheet_8000gbs": achieved / 8000.0,
                         "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                         "traffic_source": (f"{tr.get('source')}; not measured in this run") if tr else None,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel": kname},
            "c64": {"applies_per_s": ws / per32, "ms_per_apply": per32 * 1e3,
                    "achieved_gbs": alg_bytes32 / per32 / 1e9,
                    "frac": alg_bytes32 / per32 / 1e9 / peak, "kernel": kname32},
            "krylov": krylov,
            "e2e": {"value": ws * e2e_steps / te, "unit": "applies/s", "h2d_bytes_per_step": vec_bytes,
                    "d2h_bytes_per_step": vec_bytes,
                    "path": "fwi_dev_kkt_apply_host (page-locked host buffers from fwi_host_alloc; source chunks stream H2D, "
                            "are applied as they land and stream back D2H)"},
            "gpu_launches": args.steps,
            "clocks": clk.result(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref: the unmodified reference core, all threads)
# ---------------------------------------------------------------------------
def ref_threads(p):
    n_cpu = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            avail_kb = int([l for l in f if l.startswith("MemAvailable")][0].split()[1])
    except Exception:
        avail_kb = 16 << 20
    per_apply = 3 * p.vec_len * 8  # output + temporaries of one serial kkt_apply
    by_mem = max(1, int(avail_kb * 1024 * 0.5 // per_apply))
    return max(1, min(n_cpu, by_mem))


def cpu_baseline_apply(p, sample_applies=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_2204_06489_b200.problem import random_kkt
    ref = po.Ref(p, full=False, exact=False)
    x = random_kkt(p, 11)
    th = ref_threads(p)
    na = sample_applies or max(th, 2 * th)
    sec = ref.bench_kkt_apply(x, th, na)
    return {"value": na / sec, "unit": "applies/s", "cores": th, "kind": "reference",
            "sample": f"{na} reference kkt_apply calls (C2, complex128) over {th} host threads, "
                      f"{sec:.1f} s wall; {os.cpu_count()} host CPUs"}


def cpu_baseline_krylov():
    """The reference's fsgn_gmres_step (oracle/_ref, unmodified reference core; serial, so 1
    core) on BASELINE config 1 with ecg_stride 0, same options as our krylov block."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_2204_06489_b200 import _abi
    from paper_2204_06489_b200.problem import c1_problem
    p = c1_problem()
    p.d_obs = po.ref_simulate(p)
    out = {}
    for label, mode, level in (("exact", _abi.FWI_PRECOND_EXACT, 4), ("ilu", _abi.FWI_PRECOND_ILU, 4),
                               ("ilu21", _abi.FWI_PRECOND_ILU, 21)):
        ref = po.Ref(p, full=True, exact=True, ilu_level=level)
        t0 = time.perf_counter()
        _, log = ref.fsgn(mode, 30, 1e-3, 60, 0)
        tw = time.perf_counter() - t0
        it = log.iterations()
        wt = log.entries[-1].wall_time
        out[label] = {"iters_per_s": it / wt, "iterations": it, "converged": log.converged,
                      "solve_wall_s": wt, "step_wall_s": tw, "cores": 1, "kind": "reference",
                      "sample": "one reference fsgn_gmres_step (C1, tol 1e-3, restart 30, maxit 60, "
                                f"ecg_stride 0{', ILU(%d)' % level if mode == _abi.FWI_PRECOND_ILU else ''}), "
                                "ConvergenceLog wall time, same host, same run"}
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2204_06489_b200.problem import c2_problem, random_kkt
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    p = c2_problem()
    ref = po.Ref(p, full=False, exact=False)
    x = random_kkt(p, 11)
    th = ref_threads(p)
    per_step = th
    for _ in range(args.warmup):
        ref.bench_kkt_apply(x, th, th)
    tot = 0.0
    for _ in range(args.steps):
        tot += ref.bench_kkt_apply(x, th, per_step)
    value = args.steps * per_step / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded; BASELINE config 2 shapes and distributions)",
        "config": bench_config(ws, p.n),
        "cpu_baseline": {"value": value, "unit": "applies/s", "cores": th, "kind": "reference",
                         "sample": f"each step = {per_step} serial reference kkt_apply calls over {th} "
                                   f"host threads ({os.cpu_count()} CPUs)"},
        "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-krylov", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
