"""Dense prime-implicant engine on B200 — the drop-in for the reference path.

Public surface mirrors /root/reference/pkg/src/implicants/dense.py:
  dense_prime_ranks(tt, h=None, optimized=True, mem_cap=None)  dense.py:405-418
  find_primes_dense(tt, h=None, optimized=True, mem_cap=None)  dense.py:421-428
  state_bytes / block_bits_for / DEFAULT_SPLIT / MERGE / REDUCE dense.py:38-63
with the same argument meaning, dtype (int64, ascending, unique), empty-result
shape and error behaviour (ValueError for a bad split, ResourceLimitError
naming the needed bytes before anything is allocated).

All computation happens in libdqmc.so (csrc/dqmc.cu) on the GPU; this module
only validates arguments and moves buffers. ``h`` and ``optimized`` are
validated exactly as the reference does but do not change the result, which
the reference guarantees is independent of both (tests/test_dense.py:218-229);
the device always runs its own plan on the h=5 layout.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from . import errors
from .ternary import TruthTable, unrank_many

MERGE = "merge"
REDUCE = "reduce"
DEFAULT_SPLIT = 5


def block_bits_for(h: int) -> int:
    """Smallest power-of-two block holding 3^h bits, at least 64 (dense.py:56-58)."""
    return max(64, 1 << (3**h - 1).bit_length())


def state_bytes(n: int, h: int) -> int:
    """Dense state size blocks * block_bits / 8 (dense.py:61-63)."""
    return 3 ** (n - h) * block_bits_for(h) // 8


def _as_words(tt) -> tuple[int, np.ndarray]:
    n = int(tt.n)
    w = np.ascontiguousarray(tt.words, dtype=np.uint64)
    if w.shape != (max(1, (1 << n) // 64),):
        raise ValueError(f"expected {max(1, (1 << n) // 64)} words for n={n}, got shape {w.shape}")
    return n, w


def _validate(n: int, h: int | None) -> int:
    if h is None:
        return 0
    h = int(h)
    if not 1 <= h <= n:
        raise ValueError(f"split must be in 1..{n}, got {h}")
    return h


def _cap_arg(n: int, hh: int, mem_cap: int | None) -> int:
    """0 = library default (75% of free device memory); an explicit cap <= 0
    can never hold the state, so it fails here exactly as load() would
    (dense.py:358-364)."""
    if mem_cap is None:
        return 0
    cap = int(mem_cap)
    if cap <= 0:
        h = hh or min(n, DEFAULT_SPLIT)
        need = state_bytes(n, h)
        raise errors.ResourceLimitError(
            f"dense state needs {need} bytes ({3 ** (n - h)} blocks of "
            f"{block_bits_for(h)} bits), exceeding the cap of {cap} bytes"
        )
    return cap


def dense_prime_ranks(
    tt: TruthTable,
    h: int | None = None,
    optimized: bool = True,
    mem_cap: int | None = None,
) -> np.ndarray:
    """Ranks of all prime implicants of ``tt``, int64, ascending (dense.py:405-418)."""
    n, words = _as_words(tt)
    hh = _validate(n, h)
    L = _lib.load()
    res = _lib.DqmcResult()
    cap = _cap_arg(n, hh, mem_cap)
    rc = L.dqmc_primes_tt(words.ctypes.data, n, hh, cap, 0, ctypes.byref(res))
    _lib.check(rc)
    return _lib.result_to_array(res)


def prime_ranks_from_values(
    values: np.ndarray,
    h: int | None = None,
    mem_cap: int | None = None,
) -> np.ndarray:
    """Primes of a three-valued table (uint8 0 off / 1 on / 2 don't-care).

    Don't-care semantics are the only ones the reference can express:
    primes of TruthTable.from_bools(n, v != 0). The uint8
    table goes to the GPU as is and is packed there.
    """
    v = np.ascontiguousarray(values, dtype=np.uint8)
    n = int(len(v)).bit_length() - 1
    if len(v) != (1 << n) or not 1 <= n <= 31:
        raise ValueError(f"expected 2^n values, got {len(v)}")
    hh = _validate(n, h)
    L = _lib.load()
    res = _lib.DqmcResult()
    cap = _cap_arg(n, hh, mem_cap)
    rc = L.dqmc_primes_u8(v.ctypes.data, n, hh, cap, 0, ctypes.byref(res))
    _lib.check(rc)
    return _lib.result_to_array(res)


class PrimeJob:
    """A submitted call (dqmc_submit_*): ``result()`` waits for it and returns
    the int64 ranks. Keeps its input alive until collected. At most three jobs
    may be outstanding; they are collected in submission order."""

    def __init__(self, job_id: int, keep):
        self.id = job_id
        self._keep = keep
        self._done = None

    def result(self) -> np.ndarray:
        if self._done is None:
            res = _lib.DqmcResult()
            _lib.check(_lib.load().dqmc_collect(self.id, ctypes.byref(res)))
            self._done = _lib.result_to_array(res)
            self._keep = None
        return self._done


def submit(table) -> PrimeJob:
    """Queue one call: a TruthTable (or anything with .n/.words), or a uint8
    three-valued table (0 off / 1 on / 2 don't-care, 2^n entries)."""
    L = _lib.load()
    job = ctypes.c_int64(0)
    if isinstance(table, np.ndarray) and table.dtype == np.uint8:
        v = np.ascontiguousarray(table)
        n = int(len(v)).bit_length() - 1
        if len(v) != (1 << n) or not 1 <= n <= 31:
            raise ValueError(f"expected 2^n values, got {len(v)}")
        _lib.check(L.dqmc_submit_u8(v.ctypes.data, n, 0, ctypes.byref(job)))
        return PrimeJob(job.value, v)
    n, words = _as_words(table)
    _lib.check(L.dqmc_submit_tt(words.ctypes.data, n, 0, ctypes.byref(job)))
    return PrimeJob(job.value, words)


def stream_prime_ranks(tables):
    """Prime ranks of every table of an iterable, in order, with three calls in
    flight: call i's device-to-host copy overlaps call i+1's passes while call
    i+2 is already queued behind them (dqmc_submit_* / dqmc_collect)."""
    pending = []
    for t in tables:
        pending.append(submit(t))
        if len(pending) == 3:
            yield pending.pop(0).result()
    while pending:
        yield pending.pop(0).result()


def find_primes_dense(
    tt: TruthTable,
    h: int | None = None,
    optimized: bool = True,
    mem_cap: int | None = None,
) -> set[str]:
    """All prime implicants as ternary strings (dense.py:421-428)."""
    return set(unrank_many(dense_prime_ranks(tt, h, optimized, mem_cap), tt.n))


def count_primes(tt: TruthTable, mem_cap: int | None = None) -> int:
    """Number of prime implicants without materialising ranks (large n)."""
    n, words = _as_words(tt)
    L = _lib.load()
    res = _lib.DqmcResult()
    cap = _cap_arg(n, 0, mem_cap)
    rc = L.dqmc_primes_tt(words.ctypes.data, n, 0, cap, _lib.FLAG_COUNT_ONLY, ctypes.byref(res))
    _lib.check(rc)
    cnt = int(res.count)
    L.dqmc_free_result(ctypes.byref(res))
    return cnt


def prime_bitmap(tt: TruthTable) -> np.ndarray:
    """Final prime bitmap in DenseState.words layout (h=5 blocks, dense.py:127-170)
    as uint64 words, for bitmap-level parity checks. n >= 5."""
    n, words = _as_words(tt)
    if n < 5:
        raise ValueError("prime_bitmap needs n >= 5 (h=5 layout)")
    L = _lib.load()
    res = _lib.DqmcResult()
    rc = L.dqmc_primes_tt(words.ctypes.data, n, 0, 0, _lib.FLAG_KEEP_BITMAP | _lib.FLAG_COUNT_ONLY,
                          ctypes.byref(res))
    _lib.check(rc)
    L.dqmc_free_result(ctypes.byref(res))
    out = np.zeros(state_bytes(n, 5) // 8, dtype=np.uint64)
    _lib.check(L.dqmc_bitmap_download(out.ctypes.data, out.nbytes))
    return out
