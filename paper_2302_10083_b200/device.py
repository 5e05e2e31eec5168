"""Device-resident entry points (torch tensors in HBM), used by bench.py.

torch is plumbing here (allocation, streams, events); the work is the same
libdqmc.so plan as dense_prime_ranks, entered through dqmc_primes_device.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib


def gen3_device(n: int, p_on: float, p_dc: float, seed: int, device: int = 0) -> torch.Tensor:
    """2^n uint8 values from the frozen counter generator, built on the GPU
    (ttio.py:331-378 restated; SURVEY.md §8(d) three-way variant)."""
    out = torch.empty(1 << n, dtype=torch.uint8, device=f"cuda:{device}")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(_lib.load().dqmc_gen3_device(out.data_ptr(), n, float(p_on), float(p_dc), int(seed), stream))
    return out


def dense_prime_ranks_device(
    table: torch.Tensor,
    n: int,
    out: torch.Tensor | None = None,
    timing: bool = False,
    count_only: bool = False,
) -> tuple[torch.Tensor, int]:
    """Primes of a device-resident table: uint8 values (2^n) or uint64/int64
    words (TruthTable layout). Returns (ranks[:count] view of ``out``, count).
    ``out`` (int64, cuda) is grown and the pass rerun if it is too small."""
    if not table.is_cuda:
        raise ValueError("table must be a CUDA tensor")
    kind = _lib.IN_U8 if table.dtype == torch.uint8 else _lib.IN_WORDS
    if kind == _lib.IN_WORDS and table.dtype not in (torch.int64, torch.uint64):
        raise ValueError("word tables must be int64/uint64")
    L = _lib.load()
    flags = (_lib.FLAG_TIMING if timing else 0) | (_lib.FLAG_COUNT_ONLY if count_only else 0)
    stream = torch.cuda.current_stream(table.device).cuda_stream
    cnt = ctypes.c_int64(0)
    if count_only:
        _lib.check(L.dqmc_primes_device(table.data_ptr(), kind, n, None, 0, ctypes.byref(cnt), flags, stream))
        return torch.empty(0, dtype=torch.int64, device=table.device), int(cnt.value)
    if out is None:
        out = torch.empty(1 << 20, dtype=torch.int64, device=table.device)
    _lib.check(L.dqmc_primes_device(table.data_ptr(), kind, n, out.data_ptr(), out.numel(), ctypes.byref(cnt), flags, stream))
    if cnt.value > out.numel():
        out = torch.empty(int(cnt.value * 1.05) + 1024, dtype=torch.int64, device=table.device)
        _lib.check(
            L.dqmc_primes_device(table.data_ptr(), kind, n, out.data_ptr(), out.numel(), ctypes.byref(cnt), flags, stream)
        )
    return out[: cnt.value], int(cnt.value)
