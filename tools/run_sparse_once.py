#!/usr/bin/env python
"""One sparse-engine call (for ncu captures): a random function of given
density. Usage: python tools/run_sparse_once.py [n] [density]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10083_b200 as P  # noqa: E402
from oracle import gen as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
tt = P.TruthTable(n, G.random_words(n, d, 1))
r = P.sparse_prime_ranks(tt)
print(f"n={n} density={d} primes={len(r)}")
