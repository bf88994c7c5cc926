"""Raw PCIe rates on the box: H2D alone, D2H alone, both concurrently (pinned, 270 MB)."""
import time

import torch

n = 270 * 1024 * 1024 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = n * 8 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D alone {gb / t:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H alone {gb / t:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(both)
print(f"concurrent: {2 * gb / t:.1f} GB/s aggregate ({gb / t:.1f} each way)")

# chunked copies (16 chunks each way, the host-apply pipeline's granularity)
ch = 16
sz = n // ch


def both_chunked():
    for c in range(ch):
        with torch.cuda.stream(s1):
            d_a[c * sz:(c + 1) * sz].copy_(h_in[c * sz:(c + 1) * sz], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[c * sz:(c + 1) * sz].copy_(d_b[c * sz:(c + 1) * sz], non_blocking=True)


t = timed(both_chunked)
print(f"concurrent, {ch} chunks: {2 * gb / t:.1f} GB/s aggregate")

# registered (cudaHostRegister) numpy memory, as bench.py / the C ABI use
import numpy as np  # noqa: E402
import sys, os  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_06489_b200 import api as fw  # noqa: E402
a_in = np.ones(n)
a_out = np.empty(n)
fw.host_register(a_in)
fw.host_register(a_out)
r_in = torch.from_numpy(a_in)
r_out = torch.from_numpy(a_out)


def both_reg():
    with torch.cuda.stream(s1):
        d_a.copy_(r_in, non_blocking=True)
    with torch.cuda.stream(s2):
        r_out.copy_(d_b, non_blocking=True)


t = timed(both_reg)
print(f"concurrent, registered numpy: {2 * gb / t:.1f} GB/s aggregate")
