#!/usr/bin/env python
"""Per-pass CUDA-event times of n-variable config-4 calls for several builds of
libdqmc (tools/build_variant.py), interleaved in one process each, and a check
that every build returns the same primes. Usage: [P_ON=0.75 P_DC=0.05] python tools/ab_passes.py N LIB..."""
import hashlib
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, hashlib
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_2302_10083_b200 import _lib
_lib.LIB_PATH = sys.argv[2]
from paper_2302_10083_b200 import device
n = int(sys.argv[3])
v = device.gen3_device(n, float(sys.argv[4]), float(sys.argv[5]), 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.05) + 4096, dtype=torch.int64, device="cuda")
acc = {}
for i in range(7):
    r, c = device.dense_prime_ranks_device(v, n, out=out, timing=True)
    if i < 2:
        continue
    for k, ms, b in _lib.timings():
        acc.setdefault(k, []).append(ms)
h = hashlib.sha256(out[:c].cpu().numpy().tobytes()).hexdigest()[:16]
tot = sum(min(x) for x in acc.values())
print(f"{sys.argv[2].split('/')[-1]:28s} primes={c} sha={h} total={tot:.2f} " +
      " ".join(f"{k}={min(x):.2f}" for k, x in acc.items() if min(x) > 0.05), flush=True)
'''
n = sys.argv[1]
p_on, p_dc = os.environ.get("P_ON", "0.75"), os.environ.get("P_DC", "0.05")
for rep in range(2):
    for lib in sys.argv[2:]:
        subprocess.run([sys.executable, "-c", CHILD, REPO, os.path.abspath(lib), n, p_on, p_dc], timeout=300)
