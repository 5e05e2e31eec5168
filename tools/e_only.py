"""Pass E alone at n=24 (timing flag): full, and count-only."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_10083_b200 import _lib, device
n = 24
v = device.gen3_device(n, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.05) + 4096, dtype=torch.int64, device="cuda")
for mode in ("full", "count"):
    for i in range(3):
        device.dense_prime_ranks_device(v, n, out=out, timing=True, count_only=(mode == "count"))
    print(mode, os.environ.get("DQMC_E_NOSTORE", ""), {k: round(ms, 2) for k, ms, b in _lib.timings() if k in ("k_c0_final", "k_reorder")})
