"""A/B: does in-process NVML sampling perturb the device-resident timing loop?"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv
import torch
from paper_2302_10083_b200 import device

nv.nvmlInit()
H = nv.nvmlDeviceGetHandleByIndex(0)
QUERIES = {
    "none": [],
    "clock": [lambda: nv.nvmlDeviceGetClockInfo(H, nv.NVML_CLOCK_SM)],
    "maxclock": [lambda: nv.nvmlDeviceGetMaxClockInfo(H, nv.NVML_CLOCK_SM)],
    "reasons": [lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(H)],
}
n = 24
v = device.gen3_device(n, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, n)
out = torch.empty(int(c * 1.02) + 1024, dtype=torch.int64, device="cuda")
del r
for _ in range(3):
    device.dense_prime_ranks_device(v, n, out=out)
for rep in range(2):
    for name, qs in QUERIES.items():
        stop = threading.Event()
        cnt = [0, 0.0]

        def run():
            while not stop.is_set():
                t0 = time.perf_counter()
                for q in qs:
                    q()
                cnt[0] += 1
                cnt[1] += time.perf_counter() - t0
                stop.wait(0.05)

        th = threading.Thread(target=run, daemon=True)
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            device.dense_prime_ranks_device(v, n, out=out)
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        print(f"{name:9s} {e0.elapsed_time(e1) / 10:.2f} ms/step  samples {cnt[0]} host {1e3 * cnt[1] / max(1, cnt[0]):.2f} ms/sample",
              flush=True)
