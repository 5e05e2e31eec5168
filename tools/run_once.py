#!/usr/bin/env python
"""One device-resident engine call (for ncu captures): gen3 on device, then
dense_prime_ranks_device. Usage: python tools/run_once.py [n] [reps] [libdqmc variant .so]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import _lib, device  # noqa: E402

if len(sys.argv) > 3:  # a tools/build_variant.py build instead of the in-tree library
    _lib.LIB_PATH = os.path.abspath(sys.argv[3])

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
v = device.gen3_device(n, 0.75, 0.05, 3)
out = None
for _ in range(reps):
    r, cnt = device.dense_prime_ranks_device(v, n, out=out)
    out = r if out is None else out
torch.cuda.synchronize()
print(f"n={n} primes={cnt}")
