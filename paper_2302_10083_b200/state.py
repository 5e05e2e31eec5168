"""Device-resident DenseState, any split h.

Mirrors /root/reference/pkg/src/implicants/dense.py:127-402:

  load(tt, h=None, mem_cap=None, optimized=True) -> DenseState      dense.py:340-373
  DenseState.run_pass(op, dims=None) -> {top dim: block-triple count} dense.py:296-315
  DenseState.run_merge_reduce()                                       dense.py:317-337
  DenseState.padding_bits_zero / copy / equal_state / blocks / words_per_block
  extract_ranks(state) / extract_strings(state)                       dense.py:376-402

The state lives on the GPU (libdqmc.so, csrc/dqmc_state.cu: one streaming
kernel per dimension, as the reference's layers). ``words`` is a host mirror
with the reference's layout and dtype: the reference's tests poke bits into it
(``state.words[i] |= bit``) and read it back, so every device operation first
uploads the mirror and afterwards refreshes it in place. Set ``mirror=False``
for large states to keep the data on the device only (``words`` then fetches
a copy on access).
"""

from __future__ import annotations

import ctypes
from collections.abc import Sequence

import numpy as np

from . import _lib
from .dense import DEFAULT_SPLIT, MERGE, REDUCE, block_bits_for, state_bytes
from . import errors
from .ternary import unrank_many

_OPS = {MERGE: 0, REDUCE: 1}


class DenseState:
    """Mutable dense pass state on the GPU. Create via load()."""

    def __init__(self, n: int, h: int, words: np.ndarray | None = None, optimized: bool = True,
                 mirror: bool = True, _handle=None):
        self.n = int(n)
        self.h = int(h)
        self.block_bits = block_bits_for(self.h)
        self.optimized = optimized  # both bottom-layer realizations give identical states; one kernel here
        self._mirror = mirror
        self._L = _lib.load()
        if _handle is None:
            h_ = ctypes.c_void_p()
            _lib.check(self._L.dqmc_state_create(self.n, self.h, 0, ctypes.byref(h_)))
            self._h = h_
        else:
            self._h = _handle
        nw = state_bytes(self.n, self.h) // 8
        self._words = np.zeros(nw, dtype=np.uint64) if mirror else None
        if words is not None:
            w = np.ascontiguousarray(words, dtype=np.uint64)
            if w.shape != (nw,):
                raise ValueError("state size does not match n, h")
            if mirror:
                self._words[:] = w
            _lib.check(self._L.dqmc_state_set_words(self._h, w.ctypes.data, nw))
        elif mirror and _handle is not None:
            self._pull()

    # -- layout helpers (dense.py:144-152)
    @property
    def blocks(self) -> int:
        return 3 ** (self.n - self.h)

    @property
    def words_per_block(self) -> int:
        return self.block_bits // 64

    @property
    def words(self) -> np.ndarray:
        if self._mirror:
            return self._words
        out = np.empty(state_bytes(self.n, self.h) // 8, dtype=np.uint64)
        _lib.check(self._L.dqmc_state_get_words(self._h, out.ctypes.data, len(out)))
        return out

    def _push(self) -> None:
        if self._mirror:
            _lib.check(self._L.dqmc_state_set_words(self._h, self._words.ctypes.data, len(self._words)))

    def _pull(self) -> None:
        if self._mirror:
            _lib.check(self._L.dqmc_state_get_words(self._h, self._words.ctypes.data, len(self._words)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._L.dqmc_state_free(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    # -- invariants (dense.py:154-170)
    def padding_bits_zero(self) -> bool:
        self._push()
        ok = ctypes.c_int(0)
        _lib.check(self._L.dqmc_state_padding_zero(self._h, ctypes.byref(ok)))
        return bool(ok.value)

    def copy(self) -> "DenseState":
        self._push()
        h_ = ctypes.c_void_p()
        _lib.check(self._L.dqmc_state_copy(self._h, ctypes.byref(h_)))
        return DenseState(self.n, self.h, optimized=self.optimized, mirror=self._mirror, _handle=h_)

    def equal_state(self, other: "DenseState") -> bool:
        if self.n != other.n or self.h != other.h:
            return False
        self._push()
        other._push()
        eq = ctypes.c_int(0)
        _lib.check(self._L.dqmc_state_equal(self._h, other._h, ctypes.byref(eq)))
        return bool(eq.value)

    # -- passes (dense.py:296-337)
    def run_pass(self, op: str, dims: Sequence[int] | None = None) -> dict[int, int]:
        if op not in (MERGE, REDUCE):
            raise ValueError(f"op must be {MERGE!r} or {REDUCE!r}")
        if dims is None:
            dims = list(range(self.h + 1, self.n + 1)) + list(range(1, self.h + 1))
        dims = [int(d) for d in dims]
        for d in dims:
            if not 1 <= d <= self.n:
                raise ValueError(f"dimension {d} out of range 1..{self.n}")
        self._push()
        arr = np.asarray(dims, dtype=np.int32)
        counts = np.zeros(max(1, len(arr)), dtype=np.int64)
        _lib.check(self._L.dqmc_state_run_pass(self._h, _OPS[op], arr.ctypes.data, len(arr), counts.ctypes.data))
        self._pull()
        return {d: int(c) for d, c in zip(dims, counts) if c >= 0}

    def run_merge_reduce(self) -> None:
        self._push()
        _lib.check(self._L.dqmc_state_run_merge_reduce(self._h))
        self._pull()


def load(tt, h: int | None = None, mem_cap: int | None = None, optimized: bool = True,
         mirror: bool = True) -> DenseState:
    """Dense state of a truth table on the GPU (dense.py:340-373): bit rank(x) set iff f(x)=1."""
    n = int(tt.n)
    if h is None:
        h = min(n, DEFAULT_SPLIT)
    if not 1 <= h <= n:
        raise ValueError(f"split must be in 1..{n}, got {h}")
    need = state_bytes(n, h)
    if mem_cap is not None and need > mem_cap:
        raise errors.ResourceLimitError(
            f"dense state needs {need} bytes ({3 ** (n - h)} blocks of "
            f"{block_bits_for(h)} bits), exceeding the cap of {mem_cap} bytes"
        )
    st = DenseState(n, h, optimized=optimized, mirror=mirror)
    words = np.ascontiguousarray(tt.words, dtype=np.uint64)
    _lib.check(st._L.dqmc_state_load_tt(st._h, words.ctypes.data))
    st._pull()
    return st


def extract_ranks(state: DenseState) -> np.ndarray:
    """Ranks of all set bits, ascending (dense.py:376-397); AssertionError on a padding bit."""
    state._push()
    L = state._L
    cnt = ctypes.c_int64(0)
    rc = L.dqmc_state_extract(state._h, None, 0, ctypes.byref(cnt))
    if rc == _lib.DQMC_ERR_INVALID and "padding" in _lib.last_error():
        raise AssertionError("padding bit set in dense state")
    _lib.check(rc)
    out = np.zeros(max(1, cnt.value), dtype=np.int64)
    _lib.check(L.dqmc_state_extract(state._h, out.ctypes.data, len(out), ctypes.byref(cnt)))
    return out[: cnt.value]


def extract_strings(state: DenseState) -> set[str]:
    """Set bits of the state as ternary strings (dense.py:400-402)."""
    return set(unrank_many(extract_ranks(state), state.n))
