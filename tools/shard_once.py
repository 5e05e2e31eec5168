#!/usr/bin/env python
"""One emulated sharded call (all 2^k ranks on this GPU) after a warm-up, for ncu
launch lists. Usage: python tools/shard_once.py [n] [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import device  # noqa: E402
from paper_2302_10083_b200 import sharded as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
v = device.gen3_device(n, 0.75, 0.05, 3)
plan = S.ShardPlan(n, k)
nl = n - k
ops = S.GpuOps()
comm = S.EmulatedComm(plan.world)
inputs = {g: v[g << nl : (g + 1) << nl] for g in range(plan.world)}
for _ in range(2):
    ops.reset_output()
    parts = S.run_schedule(plan, inputs, ops, comm)
torch.cuda.synchronize()
print(n, k, sum(c for _, c in parts.values()))
