#!/usr/bin/env python
"""Per-pass times of count-only n=24 calls (timing experiments whose results may be wrong).
Usage: python tools/time_count.py LIB.so [p_on] [gather_permille]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_10083_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2302_10083_b200 import device  # noqa: E402

p_on = float(sys.argv[2]) if len(sys.argv) > 2 else 0.75
if len(sys.argv) > 3:
    _lib.load().dqmc_gather_threshold(int(sys.argv[3]))
v = device.gen3_device(24, p_on, 0.05 if p_on == 0.75 else 0.0, 3)
acc = {}
for i in range(5):
    r, c = device.dense_prime_ranks_device(v, 24, count_only=True, timing=True)
    if i >= 2:
        for k, ms, b in _lib.timings():
            acc.setdefault(k, []).append(ms)
print(os.path.basename(sys.argv[1]), "count", c, " ".join(f"{k}={min(x):.2f}" for k, x in acc.items() if min(x) > 0.05))
