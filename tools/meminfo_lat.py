import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_10083_b200 import device
n = 24
v = device.gen3_device(n, 0.75, 0.05, 3)
g = device.PrimesGraph(v, n)
torch.cuda.synchronize()
for label, busy in (("idle", False), ("busy", True)):
    if busy:
        for _ in range(20):
            g.replay()
    lat = []
    for _ in range(200):
        t0 = time.perf_counter(); torch.cuda.mem_get_info(); lat.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    lat.sort()
    print(label, "mem_get_info ms: median %.3f p99 %.3f max %.3f" % (1e3*lat[100], 1e3*lat[197], 1e3*lat[-1]))
