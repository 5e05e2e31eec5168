"""Per-call CUDA-event times of back-to-back device-resident calls (no per-pass timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_10083_b200 import device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 30
v = device.gen3_device(n, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.02) + 1024, dtype=torch.int64, device="cuda")
del r
for _ in range(3):
    device.dense_prime_ranks_device(v, n, out=out)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(calls + 1)]
torch.cuda.synchronize()
ev[0].record()
for i in range(calls):
    device.dense_prime_ranks_device(v, n, out=out)
    ev[i + 1].record()
torch.cuda.synchronize()
ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(calls)]
print(" ".join(f"{t:.1f}" for t in ts))
print(f"mean {sum(ts) / len(ts):.2f} min {min(ts):.2f} max {max(ts):.2f}")
