"""CPU oracle for the dense prime-implicant path.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and --impl reference) as the checker / CPU baseline.
The product package (paper_2302_10083_b200) never imports it.

Three independent constructions, each pinned against the reference's own
golden vectors in tests/test_oracle_golden.py:

* ``dense_prime_ranks``   — ctypes binding to oracle/dqmc_oracle.c, a C
  restatement of the reference's dense engine (dense.py:340-418), OpenMP
  threaded. Used as the CPU baseline (kind "port") and the large-n checker.
* ``definition_prime_ranks`` — numpy restatement of the definition-level
  oracle (oracle.py:51-81): implicant tensor by AND over completions, prime =
  implicant with no implicant one-widening parent.
* ``naive_primes`` — pure-Python string enumeration (tests/conftest.py:26-43),
  tiny n only.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from itertools import product

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

MERGE, REDUCE = 0, 1
SYMBOLS = "01*"


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "dqmc_oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.oracle_block_bits.restype = i64
        L.oracle_block_bits.argtypes = [i32]
        L.oracle_state_bytes.restype = i64
        L.oracle_state_bytes.argtypes = [i32, i32]
        L.oracle_set_threads.restype = i32
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_load.restype = None
        L.oracle_load.argtypes = [vp, i32, i32, vp]
        L.oracle_run_pass.restype = i32
        L.oracle_run_pass.argtypes = [vp, i32, i32, i32, vp, i32, i32, vp]
        L.oracle_run_merge_reduce.restype = None
        L.oracle_run_merge_reduce.argtypes = [vp, i32, i32]
        L.oracle_extract.restype = i64
        L.oracle_extract.argtypes = [vp, i32, i32, vp]
        L.oracle_padding_bits_zero.restype = i32
        L.oracle_padding_bits_zero.argtypes = [vp, i32, i32]
        L.oracle_dense_prime_ranks.restype = i64
        L.oracle_dense_prime_ranks.argtypes = [vp, i32, i32, i32, ctypes.POINTER(ctypes.POINTER(ctypes.c_int64))]
        L.oracle_free.restype = None
        L.oracle_free.argtypes = [vp]
        _lib = L
    return _lib


def set_threads(t: int = 0) -> int:
    """Set (t > 0) and return the OpenMP thread count of the C oracle."""
    return int(lib().oracle_set_threads(int(t)))


def _words(tt_words, n: int) -> np.ndarray:
    w = np.ascontiguousarray(tt_words, dtype=np.uint64)
    if w.shape != (max(1, (1 << n) // 64),):
        raise ValueError(f"expected {max(1, (1 << n) // 64)} words for n={n}, got {w.shape}")
    return w


def block_bits_for(h: int) -> int:
    return int(lib().oracle_block_bits(h))


def state_bytes(n: int, h: int) -> int:
    return int(lib().oracle_state_bytes(n, h))


def dense_prime_ranks(tt_words, n: int, h: int | None = None, optimized: bool = True) -> np.ndarray:
    """Reference dense engine restated in C (dense.py:405-418); int64 ascending."""
    w = _words(tt_words, n)
    if h is None:
        h = min(n, 5)
    out = ctypes.POINTER(ctypes.c_int64)()
    cnt = lib().oracle_dense_prime_ranks(w.ctypes.data, n, h, int(bool(optimized)), ctypes.byref(out))
    if cnt == -1:
        raise ValueError(f"split must be in 1..{n}, got {h}")
    if cnt < 0:
        raise RuntimeError(f"oracle failed with code {cnt}")
    try:
        res = np.ctypeslib.as_array(out, shape=(max(1, cnt),))[:cnt].copy()
    finally:
        lib().oracle_free(out)
    return res.astype(np.int64)


class OracleState:
    """Reference-layout DenseState on the host (dense.py:127-170), C-backed."""

    def __init__(self, tt_words, n: int, h: int | None = None):
        self.n = n
        self.h = min(n, 5) if h is None else h
        if not 1 <= self.h <= n:
            raise ValueError(f"split must be in 1..{n}, got {self.h}")
        self.words = np.zeros(state_bytes(n, self.h) // 8, dtype=np.uint64)
        lib().oracle_load(_words(tt_words, n).ctypes.data, n, self.h, self.words.ctypes.data)

    @classmethod
    def from_words(cls, words: np.ndarray, n: int, h: int = 5) -> "OracleState":
        """Wrap an existing state array (uint64, DenseState.words layout)."""
        st = cls.__new__(cls)
        st.n, st.h = n, h
        st.words = np.ascontiguousarray(words, dtype=np.uint64)
        if st.words.shape != (state_bytes(n, h) // 8,):
            raise ValueError("state size does not match n, h")
        return st

    def run_pass(self, op: int, dims=None, optimized: bool = True) -> dict:
        if dims is None:
            dims = list(range(self.h + 1, self.n + 1)) + list(range(1, self.h + 1))
        d = np.asarray(dims, dtype=np.int32)
        counts = np.zeros(len(d), dtype=np.int64)
        rc = lib().oracle_run_pass(
            self.words.ctypes.data, self.n, self.h, int(op), d.ctypes.data, len(d), int(optimized), counts.ctypes.data
        )
        if rc != 0:
            raise ValueError("bad op or dimension")
        return {int(k): int(c) for k, c in zip(d, counts) if c >= 0}

    def run_merge_reduce(self) -> None:
        lib().oracle_run_merge_reduce(self.words.ctypes.data, self.n, self.h)

    def padding_bits_zero(self) -> bool:
        return bool(lib().oracle_padding_bits_zero(self.words.ctypes.data, self.n, self.h))

    def extract_ranks(self) -> np.ndarray:
        cnt = lib().oracle_extract(self.words.ctypes.data, self.n, self.h, None)
        if cnt < 0:
            raise AssertionError("padding bit set in dense state")
        out = np.zeros(max(1, cnt), dtype=np.int64)
        lib().oracle_extract(self.words.ctypes.data, self.n, self.h, out.ctypes.data)
        return out[:cnt]


# ---------------------------------------------------------------------------
# definition-level oracle (oracle.py:51-81), numpy


def tt_bools(tt_words, n: int) -> np.ndarray:
    bits = np.unpackbits(np.ascontiguousarray(tt_words, dtype=np.uint64).view(np.uint8), bitorder="little")
    return bits[: 1 << n].astype(bool)


def definition_prime_ranks(tt_words, n: int, max_n: int = 14) -> np.ndarray:
    """Ranks of all primes, ascending, straight from the definitions.

    Axis j of the (2,)*n reshaped table is variable n-j (C order), so the flat
    C-order index of a (3,)*n tensor equals the ternary rank (oracle.py:67-69).
    imp[..., d, ...] along an axis is the implicant indicator with that
    variable fixed to d (0/1) or free (2 = AND over both halves), applied on
    every axis; prime = implicant and no single fixed digit can be widened to
    an implicant (oracle.py:77-80).
    """
    if n > max_n:
        raise ValueError(f"definition oracle materialises 3^n tensors; refusing n={n} > {max_n}")
    imp = tt_bools(tt_words, n).reshape((2,) * n)
    for ax in range(n):
        lo = np.take(imp, 0, axis=ax)
        hi = np.take(imp, 1, axis=ax)
        imp = np.stack([lo, hi, lo & hi], axis=ax)
    prime = imp.copy()
    for ax in range(n):
        head = (slice(None),) * ax
        prime[head + (slice(0, 2),)] &= ~imp[head + (slice(2, 3),)]
    return np.flatnonzero(prime.ravel()).astype(np.int64)


def string_points(s: str) -> list[int]:
    """Truth-table indices covered by a ternary string (tests/conftest.py:17-23)."""
    options = [("0", "1") if ch == "*" else (ch,) for ch in s]
    return [sum((ch == "1") << i for i, ch in enumerate(combo)) for combo in product(*options)]


def naive_primes(tt_words, n: int) -> set[str]:
    """Definition-literal primes by string enumeration (tests/conftest.py:26-43)."""
    on = tt_bools(tt_words, n)
    support = {int(i) for i in np.flatnonzero(on)}
    implicants = set()
    for digits in product(SYMBOLS, repeat=n):
        s = "".join(digits)
        if all(p in support for p in string_points(s)):
            implicants.add(s)
    return {
        s
        for s in implicants
        if not any(s[:i] + "*" + s[i + 1 :] in implicants for i in range(n) if s[i] != "*")
    }


def unrank(r: int, n: int) -> str:
    out = []
    for _ in range(n):
        out.append(SYMBOLS[r % 3])
        r //= 3
    return "".join(out)


def rank(s: str) -> int:
    return sum(SYMBOLS.index(ch) * 3**i for i, ch in enumerate(s))


def is_prime_cube(r: int, n: int, on: np.ndarray) -> tuple[bool, bool]:
    """Independent (implicant, maximal) check of one cube against the on∪dc
    bitmap ``on`` (covered_indices semantics, oracle.py:23-37)."""
    s = unrank(int(r), n)

    def implicant(t: str) -> bool:
        return bool(on[np.asarray(string_points(t), dtype=np.int64)].all())

    imp = implicant(s)
    maximal = imp and not any(implicant(s[:i] + "*" + s[i + 1 :]) for i in range(n) if s[i] != "*")
    return imp, maximal
