"""Time the sharded schedule with all 2^k ranks emulated on one GPU (one
process, EmulatedComm): ms per call for n and k, against the single-GPU call.
Usage: python tools/shard_time.py [n] [reps] [libdqmc variant .so]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import _lib, device  # noqa: E402

if len(sys.argv) > 3:  # a tools/build_variant.py build instead of the in-tree library
    _lib.LIB_PATH = os.path.abspath(sys.argv[3])
from paper_2302_10083_b200 import sharded as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
v = device.gen3_device(n, 0.75, 0.05, 3)
r, cnt = device.dense_prime_ranks_device(v, n)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    device.dense_prime_ranks_device(v, n)
torch.cuda.synchronize()
out = {"n": n, "single_gpu_ms": (time.perf_counter() - t0) / reps * 1e3, "primes": cnt}
for k in (1, 2, 3):
    plan = S.ShardPlan(n, k)
    nl = n - k
    ops = S.GpuOps()
    comm = S.EmulatedComm(plan.world)
    inputs = {g: v[g << nl : (g + 1) << nl] for g in range(plan.world)}
    parts = S.run_schedule(plan, inputs, ops, comm)
    got = sum(c for _, c in parts.values())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ops.reset_output()
        S.run_schedule(plan, inputs, ops, comm)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    out[f"k{k}"] = {"m": plan.m, "super_blocks": len(plan.blocks), "emulated_ms_all_ranks": ms,
                    "per_rank_ms_if_parallel": ms / plan.world, "primes_ok": got == cnt}
    del ops
    torch.cuda.empty_cache()
print(json.dumps(out))
