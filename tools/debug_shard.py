import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_10083_b200 as P
from paper_2302_10083_b200 import device, sharded as S
n = int(sys.argv[1]); k = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
vd = device.gen3_device(n, 0.75, 0.05, 3)
want = P.prime_ranks_from_values(vd.cpu().numpy())
nl = n - k
for rep in range(reps):
    got = S.gpu_sharded_prime_ranks_emulated(vd, n, k)
    ok = np.array_equal(got, want)
    print("rep", rep, "ok", ok, len(got), len(want), flush=True)
    if not ok:
        for t in S.all_blocks(k):
            lo, hi = S.rho(t) * 3**nl, (S.rho(t) + 1) * 3**nl
            g = got[(got >= lo) & (got < hi)]; w = want[(want >= lo) & (want < hi)]
            if not np.array_equal(g, w):
                print("  block", t, "got", len(g), "want", len(w), "missing", len(np.setdiff1d(w, g)), "extra", len(np.setdiff1d(g, w)))
