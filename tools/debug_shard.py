"""Emulated k-rank sharded call vs the single-GPU engine, with the super-blocks
that differ listed. Usage: python tools/debug_shard.py n k [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2302_10083_b200 as P  # noqa: E402
from paper_2302_10083_b200 import device, sharded as S  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
vd = device.gen3_device(n, 0.75, 0.05, 3)
want = P.prime_ranks_from_values(vd.cpu().numpy())
plan = S.ShardPlan(n, k)
for rep in range(reps):
    got = S.gpu_sharded_prime_ranks_emulated(vd, n, k)
    ok = np.array_equal(got, want)
    print("rep", rep, "ok", ok, len(got), len(want), flush=True)
    if not ok:
        for d in plan.blocks:
            lo, hi = plan.offset(d), plan.offset(d) + 3**plan.L
            g = got[(got >= lo) & (got < hi)]
            w = want[(want >= lo) & (want < hi)]
            if not np.array_equal(g, w):
                print("  super-block", d, "owner", plan.owner[d], "got", len(g), "want", len(w))
