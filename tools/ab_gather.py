#!/usr/bin/env python
"""Pass D against the gather finish (dqmc_gather_threshold 0 / 1000) at n = 24 over input densities:
per-pass CUDA-event times, the nonzero-block share pass C counted, and equality of the rank lists.
Usage: python tools/ab_gather.py [LIB.so] [p_on ...]"""
import ctypes
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import _lib  # noqa: E402

args = sys.argv[1:]
if args and args[0].endswith(".so"):
    _lib.LIB_PATH = os.path.abspath(args.pop(0))
from paper_2302_10083_b200 import device  # noqa: E402

L = _lib.load()
n = 24
for p_on in [float(a) for a in args] or [0.75, 0.9, 0.95, 0.99]:
    v = device.gen3_device(n, p_on, 0.05 if p_on == 0.75 else 0.0, 3)
    r, c = device.dense_prime_ranks_device(v, n)
    out = torch.empty(int(c * 1.02) + 4096, dtype=torch.int64, device="cuda")
    del r
    res = {}
    for thr in (0, 1000):
        L.dqmc_gather_threshold(thr)
        acc = {}
        for i in range(5):
            r, c = device.dense_prime_ranks_device(v, n, out=out, timing=True)
            if i < 2:
                continue
            for k, ms, b in _lib.timings():
                acc.setdefault(k, []).append(ms)
        nzb, tot, g = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
        _lib.check(L.dqmc_last_gather(ctypes.byref(nzb), ctypes.byref(tot), ctypes.byref(g)))
        h = hashlib.sha256(out[:c].cpu().numpy().tobytes()).hexdigest()[:12]
        res[thr] = (sum(min(x) for x in acc.values()), h)
        print(f"p_on={p_on} thr={thr} gathered={g.value} nz_blocks={nzb.value / tot.value:.4f} primes={c} sha={h} "
              f"total={res[thr][0]:.2f} " + " ".join(f"{k.replace('k_strided','S').replace('k_c0_','')}={min(x):.2f}"
                                                     for k, x in acc.items() if min(x) > 0.05), flush=True)
    assert res[0][1] == res[1000][1]
    del out
    torch.cuda.empty_cache()
