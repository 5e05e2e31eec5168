import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_10083_b200 as P
from paper_2302_10083_b200 import device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
v = device.gen3_device(n, 0.75, 0.05, 3)
hv = torch.empty(1 << n, dtype=torch.uint8, pin_memory=True); hv.copy_(v.cpu()); hv = hv.numpy()
for mode in ("pipe", "plain", "pipe"):
    if mode == "plain": os.environ["DQMC_NO_PIPELINE"] = "1"
    else: os.environ.pop("DQMC_NO_PIPELINE", None)
    ts = []
    for i in range(5):
        t0 = time.perf_counter(); r = P.prime_ranks_from_values(hv); ts.append(time.perf_counter() - t0); del r
    print(mode, " ".join(f"{1e3*t:.1f}" for t in ts), flush=True)
# raw D2H bandwidth pinned
x = torch.empty(210_000_000, dtype=torch.int64, device="cuda"); h = torch.empty_like(x, device="cpu").pin_memory()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"D2H {x.numel()*8/dt/1e9:.1f} GB/s ({1e3*dt:.1f} ms)")
