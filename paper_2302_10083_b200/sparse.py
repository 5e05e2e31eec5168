"""Sparse engine on the GPU — drop-in for the reference's
sparse_prime_ranks / find_primes_sparse (/root/reference/pkg/src/implicants/
sparse.py:288-314): same signature, int64 ascending ranks, same errors. The
level walk over packed cubes runs in csrc/dqmc_sparse.cu (device hash sets,
linear probing, tombstones, first-star generation rule). Its work scales with
the number of implicants, so it is the engine of choice at low density; the
dense engine wins once levels approach the full cube.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, errors
from .ternary import unrank_many

_MIN_TABLE = 64


def _table_slots(entries: int) -> int:
    size = _MIN_TABLE
    while size < 2 * entries:
        size *= 2
    return size


def sparse_prime_ranks(tt, mem_cap: int | None = None) -> np.ndarray:
    """Ranks of all prime implicants of ``tt``, int64, ascending (sparse.py:288-307).
    ``mem_cap`` bounds every level table in bytes (default: 75% of free device
    memory); a table over it raises ResourceLimitError before allocation."""
    n = int(tt.n)
    words = np.ascontiguousarray(tt.words, dtype=np.uint64)
    if words.shape != (max(1, (1 << n) // 64),):
        raise ValueError(f"expected {max(1, (1 << n) // 64)} words for n={n}, got shape {words.shape}")
    cap = 0
    if mem_cap is not None:
        cap = int(mem_cap)
        if cap <= 0:  # the level-0 table alone exceeds it (sparse.py:105-111)
            size = _table_slots(int(np.bitwise_count(words).sum()))
            raise errors.ResourceLimitError(
                f"sparse level table needs {size * 8} bytes ({size} slots), exceeding the cap of {cap} bytes"
            )
    L = _lib.load()
    res = _lib.DqmcResult()
    _lib.check(L.dqmc_sparse_primes_tt(words.ctypes.data, n, cap, ctypes.byref(res)))
    return _lib.result_to_array(res)


def find_primes_sparse(tt, mem_cap: int | None = None) -> set[str]:
    """All prime implicants as ternary strings (sparse.py:310-314)."""
    return set(unrank_many(sparse_prime_ranks(tt, mem_cap=mem_cap), tt.n))
