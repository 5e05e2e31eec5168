import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_10083_b200 import device, _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
v = device.gen3_device(n, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.02) + 1024, dtype=torch.int64, device="cuda")
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, c2 = device.dense_prime_ranks_device(v, n, out=out, timing=True)
    t1 = time.perf_counter()
    tl = _lib.timings()
    print(f"call {i}: wall {1e3*(t1-t0):.2f} ms, passes {sum(x[1] for x in tl):.2f} ms", flush=True)
