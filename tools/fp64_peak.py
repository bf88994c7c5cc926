"""FP64 roofline denominators on this B200 (tool only — cuBLAS through torch, never on the
product path): DGEMM (real FP64, tensor cores) and ZGEMM throughput, best of N, CUDA events.
Writes profiles/r02_fp64_peak.json; DESIGN.md §3.3 quotes the DMMA complex GEMM against it.

    python tools/fp64_peak.py [out.json]
"""
import json
import sys

import torch


def best(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    t = best(lambda: a @ b)
    out[f"dgemm_{n}_tflops"] = 2 * n ** 3 / t / 1e12
for n in (1024, 4096):
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    t = best(lambda: a @ b)
    out[f"zgemm_{n}_tflops_8mnk"] = 8 * n ** 3 / t / 1e12
out["device"] = torch.cuda.get_device_name()
out["how"] = "torch.matmul (cuBLAS) best of 10 after 3 warm-up, CUDA events; ZGEMM counted as 8MNK"
print(json.dumps(out, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
