#!/usr/bin/env python
"""Sparsity of the merged implicant bitmap M at n (config-4 distribution by
default): fraction of nonzero 32-B blocks, 128-B pieces, D tiles (729 pieces
of one group-0 column) and C0 tiles. Usage: python tools/sparsity.py [n] [p_on] [p_dc]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_10083_b200 import _lib, device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
p_on = float(sys.argv[2]) if len(sys.argv) > 2 else 0.75
p_dc = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
L = _lib.load()
v = device.gen3_device(n, p_on, p_dc, 3)
H = n - 5
M = torch.empty(3**H * 8, dtype=torch.int32, device="cuda")
_lib.check(L.dqmc_merge_device(ctypes.c_void_p(v.data_ptr()), 1, n, ctypes.c_void_p(M.data_ptr()), None))
torch.cuda.synchronize()
blk = M.view(-1, 8).ne(0).any(1)  # 3^H blocks
print(f"n={n} p_on={p_on} p_dc={p_dc}")
print(f"blocks nonzero: {blk.float().mean().item():.4f}")
g = min(H, 7)
T = H - g
t = blk.view(3**T, 3**g)
print(f"C0 tiles nonzero: {t.any(1).float().mean().item():.4f}")
pad = (4 - 3**g % 4) % 4
tp = torch.cat([t, torch.zeros(3**T, pad, dtype=torch.bool, device='cuda')], 1) if pad else t
pieces = tp.view(3**T, -1, 4).any(2)  # [upper*q1][x]
print(f"128-B pieces nonzero: {pieces.float().mean().item():.4f}")
if T >= 6:
    r0 = 6
    pc = pieces.view(3**(T - r0), 3**r0, -1)  # [q2][q1][x]
    print(f"D tiles (q2, x over q1) nonzero: {pc.any(1).float().mean().item():.4f}")
    # C's tiles: (q1, x) over the upper digits
    print(f"C tiles (q1, x over upper) nonzero: {pc.any(0).float().mean().item():.4f}")
    # D-tile sub-blocks of g consecutive group-0 rows (the low log3(g) digits vary)
    for gsz in (3, 9, 27, 81, 243):
        sb = pc.permute(0, 2, 1).reshape(3**(T - r0), -1, 729 // gsz, gsz).any(3)
        print(f"D sub-blocks of {gsz} rows nonzero: {sb.float().mean().item():.4f}")
del M
