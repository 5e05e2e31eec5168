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


def _kind(table: torch.Tensor) -> int:
    if not table.is_cuda:
        raise ValueError("table must be a CUDA tensor")
    if table.dtype == torch.uint8:
        return _lib.IN_U8
    if table.dtype not in (torch.int64, torch.uint64):
        raise ValueError("word tables must be int64/uint64")
    return _lib.IN_WORDS


def enqueue_prime_ranks(table: torch.Tensor, n: int, out: torch.Tensor, count: torch.Tensor) -> None:
    """Stream-ordered call (DQMC_FLAG_ASYNC): nothing synchronises, so calls
    queue back to back and can be captured into a CUDA graph. ``count`` (int64
    cuda, one element) receives the prime count, or -(count + 1) if ``out`` or
    the engine's rank scratch was too small (call dense_prime_ranks_device once
    first: it sizes the scratch for this n)."""
    if count.dtype != torch.int64 or not count.is_cuda or count.numel() < 1:
        raise ValueError("count must be a one-element int64 CUDA tensor")
    if out.dtype != torch.int64 or not out.is_cuda:
        raise ValueError("out must be an int64 CUDA tensor")
    stream = torch.cuda.current_stream(table.device).cuda_stream
    _lib.check(_lib.load().dqmc_primes_device(table.data_ptr(), _kind(table), n, out.data_ptr(), out.numel(),
                                              ctypes.cast(count.data_ptr(), ctypes.POINTER(ctypes.c_int64)),
                                              _lib.FLAG_ASYNC, stream))


class PrimesGraph:
    """One prime-implicant call on fixed device buffers, captured once as a
    CUDA graph and replayed (no per-call host work beyond one graph launch).
    ``table`` may be refilled in place between replays; ``ranks()`` reads the
    result of the last replay (synchronising)."""

    def __init__(self, table: torch.Tensor, n: int, headroom: float = 1.05):
        self.table, self.n = table, n
        r, cnt = dense_prime_ranks_device(table, n)  # sizes the engine's workspace for n
        del r
        self.out = torch.empty(int(cnt * headroom) + 1024, dtype=torch.int64, device=table.device)
        self.count = torch.zeros(1, dtype=torch.int64, device=table.device)
        s = torch.cuda.Stream(table.device)
        s.wait_stream(torch.cuda.current_stream(table.device))
        with torch.cuda.stream(s):
            enqueue_prime_ranks(table, n, self.out, self.count)  # warm-up on the capture stream
        torch.cuda.current_stream(table.device).wait_stream(s)
        torch.cuda.synchronize(table.device)
        self.graph = torch.cuda.CUDAGraph()
        L = _lib.load()
        with torch.cuda.graph(self.graph, stream=s):
            enqueue_prime_ranks(table, n, self.out, self.count)
        # the graph holds raw pointers into the engine workspace: valid until
        # the engine reallocates or releases a buffer (dqmc_engine_generation)
        self.generation = int(L.dqmc_engine_generation())

    def replay(self) -> None:
        """Launch the captured call on the current stream, ordered after every
        earlier use of the engine workspace and before every later one."""
        L = _lib.load()
        if int(L.dqmc_engine_generation()) != self.generation:
            raise RuntimeError("the engine workspace was reallocated or released since this graph was captured; "
                               "build a new PrimesGraph")
        stream = torch.cuda.current_stream(self.table.device).cuda_stream
        _lib.check(L.dqmc_engine_enter(stream))
        self.graph.replay()
        _lib.check(L.dqmc_engine_exit(stream))

    def ranks(self) -> torch.Tensor:
        c = int(self.count.item())
        if c < 0:
            raise RuntimeError(f"graph output too small for {-c - 1} primes; rebuild the PrimesGraph")
        return self.out[:c]
