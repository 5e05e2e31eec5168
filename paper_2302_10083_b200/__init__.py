"""B200-native dense Quine-McCluskey prime-implicant engine (arXiv 2302.10083).

Drop-in for the reference's dense path (implicants.dense_prime_ranks /
find_primes_dense, /root/reference/pkg/src/implicants/dense.py:405-428): same
signature, int64 ascending ranks, same errors; the work runs in hand-written
sm_100a kernels behind the C ABI of include/dqmc.h (libdqmc.so).
"""

from .dense import (DEFAULT_SPLIT, MERGE, REDUCE, PrimeJob, block_bits_for, count_primes, dense_prime_ranks,
                    find_primes_dense, prime_bitmap, prime_ranks_from_values, state_bytes, stream_prime_ranks, submit)
from .engine import ENGINES, run_engine
from .errors import ImplicantsError, ParseError, ResourceLimitError
from .sparse import find_primes_sparse, sparse_prime_ranks
from .ternary import (MAX_N, SYMBOLS, TruthTable, index_to_rank, rank, rank_digits, rank_weights, ranks_to_text,
                      unrank, unrank_many)

__version__ = "0.1.0"

# the drop-in surface: the reference's names for this path, plus the device-side additions
__all__ = sorted(
    "DEFAULT_SPLIT ENGINES ImplicantsError MAX_N MERGE ParseError PrimeJob REDUCE ResourceLimitError SYMBOLS "
    "TruthTable block_bits_for count_primes dense_prime_ranks find_primes_dense find_primes_sparse index_to_rank "
    "prime_bitmap prime_ranks_from_values rank rank_digits rank_weights ranks_to_text run_engine "
    "stream_prime_ranks sparse_prime_ranks submit state_bytes unrank unrank_many".split()
)
