#!/usr/bin/env python
"""Run one case with DQMC_DEBUG=1 (sync + report after every pass)."""
import os
import sys

os.environ.setdefault("DQMC_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2302_10083_b200 as P  # noqa: E402
from oracle import gen as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
pon = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
pdc = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
v = G.gen3(n, pon, pdc, 1)
r = P.prime_ranks_from_values(v)
o = O.dense_prime_ranks(G.values_to_words(v), n)
print(n, len(r), len(o), np.array_equal(r, o))
