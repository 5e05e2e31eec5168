#!/bin/bash
# per-pass ms of one n=24 call per env setting (results may be wrong for timing-only knobs)
for v in "$@"; do
  env $v timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import torch
from paper_2302_10083_b200 import device, _lib
v = device.gen3_device(24, 0.75, 0.05, 3)
r, c = device.dense_prime_ranks_device(v, 24)
out = torch.empty(int(c * 1.5) + 4096, dtype=torch.int64, device='cuda')
for i in range(4):
    device.dense_prime_ranks_device(v, 24, out=out, timing=True)
print('[$v]', {k: round(ms, 2) for k, ms, b in _lib.timings() if ms > 0.5})
" 2>&1 | tail -1
done
