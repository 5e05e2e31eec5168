import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_10083_b200 as P
from oracle import gen as G
for n in range(1, 16):
    P.dense_prime_ranks(P.TruthTable.full(n)); P.dense_prime_ranks(P.TruthTable.empty(n))
print("consts ok", flush=True)
v = G.config_values(1); P.prime_ranks_from_values(v); P.dense_prime_ranks(P.TruthTable(10, G.values_to_words(v)))
print("cfg1 ok", flush=True)
v = G.config_values(2); r = P.prime_ranks_from_values(v)
print("cfg2", len(r), flush=True)
