"""One-off CPU measurement for bench.py's cpu_baseline.one_thread_n24: the
oracle port (C restatement of the reference's dense engine) on the full
BASELINE config-4 call (n=24) with ONE host thread — the reference's own
concurrency (single-threaded NumPy) — on the GPU box's host. Writes
gpurun_out/r2_cpu_n24.json (copied to profiles/ by hand)."""

import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
info = bench.cpu_info()
from oracle import gen as G  # noqa: E402

v = G.gen3(n, 0.75, 0.05, 3)
t0 = time.time()
dt, cnt, thr = bench.cpu_port_run(n, threads=1, values=v)
out = {"n": n, "seconds": dt, "primes": cnt, "threads": thr, "cells_per_s": 3**n / dt,
       "what": "oracle port (oracle/dqmc_oracle.c) dense_prime_ranks, BASELINE config 4, 1 host thread, one call",
       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), **info}
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", "r2_cpu_n24.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
