"""Time the reduce-only strided kernel on the far group (3^13-block row stride,
1 in-block axis) and the near group (3^7, 4 axes) through the sharded path's
dqmc_reduce_extract_device at n=24 (timing flag, count only)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2302_10083_b200 import _lib, device
from paper_2302_10083_b200.dense import state_bytes

n = 24
L = _lib.load()
v = device.gen3_device(n, 0.75, 0.05, 3)
st = torch.empty(state_bytes(n, 5) // 4, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    _lib.check(L.dqmc_merge_device(v.data_ptr(), _lib.IN_U8, n, st.data_ptr(), s))
    cnt = ctypes.c_int64(0)
    _lib.check(L.dqmc_reduce_extract_device(st.data_ptr(), n, None, 0, None, 0, ctypes.byref(cnt), _lib.FLAG_TIMING, s))
    print(rep, cnt.value, [(k, round(ms, 2)) for k, ms, b in _lib.timings()])
