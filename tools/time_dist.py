#!/usr/bin/env python
"""Device-resident ms per call for a given n and distribution (CUDA events,
3 warm-up + 5 timed calls). Usage: python tools/time_dist.py n p_on p_dc seed"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import device  # noqa: E402

n, p_on, p_dc, seed = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
v = device.gen3_device(n, p_on, p_dc, seed)
r, cnt = device.dense_prime_ranks_device(v, n)
for _ in range(2):
    r, cnt = device.dense_prime_ranks_device(v, n, out=r)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r, cnt = device.dense_prime_ranks_device(v, n, out=r)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"n={n} p_on={p_on} p_dc={p_dc} seed={seed}: {cnt} primes, {ms:.2f} ms, {3**n / ms * 1e3:.3g} cells/s")
