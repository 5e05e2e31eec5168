"""Per-call CUDA-event times of back-to-back device-resident calls.
usage: call_spread.py n calls [sync|async|graph]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_10083_b200 import device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 30
mode = sys.argv[3] if len(sys.argv) > 3 else "sync"
v = device.gen3_device(n, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.02) + 1024, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
del r
g = device.PrimesGraph(v, n) if mode == "graph" else None
for _ in range(3):
    device.dense_prime_ranks_device(v, n, out=out)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(calls + 1)]
torch.cuda.synchronize()
t0 = time.perf_counter()
host = []
ev[0].record()
for i in range(calls):
    h0 = time.perf_counter()
    if mode == "sync":
        device.dense_prime_ranks_device(v, n, out=out)
    elif mode == "async":
        device.enqueue_prime_ranks(v, n, out, cnt)
    else:
        g.replay()
    host.append(time.perf_counter() - h0)
    ev[i + 1].record()
t_enq = time.perf_counter() - t0
torch.cuda.synchronize()
ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(calls)]
print(mode, " ".join(f"{t:.1f}" for t in ts))
print(f"{mode}: mean {sum(ts) / len(ts):.2f} min {min(ts):.2f} max {max(ts):.2f}; host enqueue total {1e3 * t_enq:.1f} ms, "
      f"max host call {1e3 * max(host):.2f} ms")
