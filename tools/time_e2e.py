"""Host-to-host timing of the n=24 config-4 call: the synchronous drop-in call and the job
stream (three in flight), for several sizes of the host widening pool (packed rank transfer).
usage: [DQMC_LIB=variant.so] python tools/time_e2e.py [n] [threads ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hashlib
import numpy as np
import torch
import paper_2302_10083_b200 as pkg
from paper_2302_10083_b200 import _lib
if os.environ.get("DQMC_LIB"):  # a tools/build_variant.py build
    _lib.LIB_PATH = os.path.abspath(os.environ["DQMC_LIB"])
from paper_2302_10083_b200 import device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
threads = [int(x) for x in sys.argv[2:]] or [0]
v = device.gen3_device(n, 0.75, 0.05, 3)
ref, c = device.dense_prime_ranks_device(v, n)
want = hashlib.sha256(ref.cpu().numpy().tobytes()).hexdigest()
del ref
hv_t = torch.empty(1 << n, dtype=torch.uint8, pin_memory=True)
hv_t.copy_(v.cpu())
hv = hv_t.numpy()
L = _lib.load()
for th in threads:
    L.dqmc_host_threads(th)
    for _ in range(3):
        r = pkg.prime_ranks_from_values(hv)
    assert hashlib.sha256(r.tobytes()).hexdigest() == want, "single-call ranks differ"
    del r
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = pkg.prime_ranks_from_values(hv)
        ts.append(time.perf_counter() - t0)
        del r
    for r in pkg.stream_prime_ranks([hv] * 3):
        last = r
    assert hashlib.sha256(last.tobytes()).hexdigest() == want, "stream ranks differ"
    del last, r
    torch.cuda.synchronize(); t0 = time.perf_counter()
    k = 0
    for r in pkg.stream_prime_ranks([hv] * 30):
        k += 1
        del r
    t_stream = (time.perf_counter() - t0) / k
    print(f"n={n} primes={c} pool={th}: single call {np.mean(ts)*1e3:.2f} ms (min {min(ts)*1e3:.2f}), "
          f"job stream {t_stream*1e3:.2f} ms/call", flush=True)
