"""Top-k-variable sharding of the dense path over 2^k ranks.

Rank g owns the binary assignment of the top k variables (bit j of g =
variable n-k+1+j) and the contiguous truth-table slice [g*2^(n-k), (g+1)*2^(n-k)).
With n' = n-k, the 3^k "top blocks" t in {0,1,*}^k each cover the contiguous
rank range [rho(t)*3^n', (rho(t)+1)*3^n') and hold 3^n' cells in the h=5
layout, so the global prime list is the concatenation of the blocks' lists in
rho order. The algorithm (composition verified on the reference, SURVEY.md
App. B.3):

1. local MERGE of the n' low dimensions on every binary block -> M_t;
2. star blocks, one round per top axis j: M_t = M_{t[j->0]} AND M_{t[j->1]}
   for the blocks whose highest star is j (block-level AND of dense.py:174-212);
3. kills: K_t = OR over the fixed top digits j of M_{t[j->*]} (pre-reduce M,
   as the oracle formula oracle.py:77-80 requires);
4. P_t = REDUCE_low(M_t) AND NOT K_t, compacted to ranks + rho(t)*3^n'.

Blocks are placed by a deterministic greedy balance (every rank computes the
same map); each block computed at its owner, inputs exchanged point-to-point.
NCCL has no bitwise-AND reduction (nccl.h ops: sum/prod/max/min/avg), so the
exchange is send/recv of whole blocks and the AND/OR runs in our kernels.

The same schedule runs over a real process group, or over all 2^k ranks inside
one process (``EmulatedComm``), which lets one GPU check k-GPU bit-exactness.
Transports for a process group:
  ``DistComm``  torch.distributed send/recv of whole blocks (NCCL on GPUs;
                gloo with host staging for CPU tests and GPU-sharing tests);
  ``IpcComm``   P2P: no transfer at all. Each rank exports CUDA IPC handles of
                the blocks peers need; the peer opens them and our AND / OR
                kernels read the owner's memory directly over NVLink (the
                survey's fused peer-load design). Host-side
                all_gather / barrier order the rounds; no kernel ever waits
                on another process.
Local compute is an ``ops`` object: ``GpuOps`` (libdqmc.so) in production;
tests may pass a CPU implementation to exercise the host logic under gloo.
"""

from __future__ import annotations

import itertools
from collections.abc import Iterable

import numpy as np


# ---------------------------------------------------------------------------
# schedule (pure host logic)


def rho(t: tuple[int, ...]) -> int:
    """Rank of a top-digit tuple (digit j has weight 3^j)."""
    return sum(d * 3**j for j, d in enumerate(t))


def all_blocks(k: int) -> list[tuple[int, ...]]:
    """Every top block, in rho (= global rank) order."""
    return sorted(itertools.product((0, 1, 2), repeat=k), key=rho)


def binary_block(g: int, k: int) -> tuple[int, ...]:
    return tuple((g >> j) & 1 for j in range(k))


def owner_map(k: int) -> dict[tuple[int, ...], int]:
    """Deterministic balanced placement: each block goes to the least loaded
    rank whose bits agree with the block's fixed digits (binary blocks to
    their own rank)."""
    load = [0] * (1 << k)
    own: dict[tuple[int, ...], int] = {}
    for t in sorted(all_blocks(k), key=lambda t: (sum(d == 2 for d in t), rho(t))):
        cands = [g for g in range(1 << k) if all(((g >> j) & 1) == d for j, d in enumerate(t) if d != 2)]
        best = min(cands, key=lambda g: (load[g], g))
        own[t] = best
        load[best] += 1
    return own


def highest_star(t: tuple[int, ...]) -> int:
    stars = [j for j, d in enumerate(t) if d == 2]
    return max(stars) if stars else -1


def children(t: tuple[int, ...], j: int) -> tuple[tuple[int, ...], tuple[int, ...]]:
    return tuple(0 if i == j else d for i, d in enumerate(t)), tuple(1 if i == j else d for i, d in enumerate(t))


def parents(t: tuple[int, ...]) -> list[tuple[int, ...]]:
    return [tuple(2 if i == j else d for i, d in enumerate(t)) for j, d in enumerate(t) if d != 2]


def star_rounds(k: int) -> list[list[tuple[tuple, tuple, tuple]]]:
    """Round j: (t, c0, c1) for every block whose highest star axis is j."""
    rounds = []
    for j in range(k):
        jobs = []
        for t in all_blocks(k):
            if highest_star(t) == j:
                c0, c1 = children(t, j)
                jobs.append((t, c0, c1))
        rounds.append(jobs)
    return rounds


def transfer_volume(k: int) -> dict[int, int]:
    """Blocks each rank receives over the whole schedule (for DESIGN notes / tests)."""
    own = owner_map(k)
    recv = {g: 0 for g in range(1 << k)}
    for jobs in star_rounds(k):
        seen = set()
        for t, c0, c1 in jobs:
            for c in (c0, c1):
                if own[c] != own[t] and (c, own[t]) not in seen:
                    seen.add((c, own[t]))
                    recv[own[t]] += 1
    seen = set()
    for t in all_blocks(k):
        for p in parents(t):
            if own[p] != own[t] and (p, own[t]) not in seen:
                seen.add((p, own[t]))
                recv[own[t]] += 1
    return recv


# ---------------------------------------------------------------------------
# communication


class EmulatedComm:
    """All 2^k ranks inside one process: a transfer is a reference."""

    def __init__(self, world: int):
        self.world = world

    def local_ranks(self) -> list[int]:
        return list(range(self.world))

    def is_local(self, r: int) -> bool:
        return True

    def exchange(self, transfers, held, ops):
        return {(dst, c): held[(src, c)] for c, src, dst in transfers}

    def done_reading(self, ops):
        pass

    def barrier(self):
        pass


class DistComm:
    """One rank of a torch.distributed process group (NCCL or gloo).

    staging=True moves device blocks through host memory (gloo cannot send
    CUDA tensors); it lets several processes share one GPU in tests, since no
    kernel ever waits on another process — only the host-side exchange does."""

    def __init__(self, group=None, staging: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.staging = staging
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def local_ranks(self) -> list[int]:
        return [self.rank]

    def is_local(self, r: int) -> bool:
        return r == self.rank

    def exchange(self, transfers, held, ops):
        """Point-to-point block moves, posted in the same global order on
        every rank so sends and receives pair up deterministically."""
        dist = self.dist
        ops.sync()  # blocks about to be sent must be complete
        reqs, out, staged = [], {}, []
        for c, src, dst in transfers:
            if src == self.rank:
                t = held[(src, c)]
                if self.staging and t.is_cuda:
                    t = t.cpu()
                    staged.append(t)
                reqs.append(dist.isend(t, dst, group=self.group))
            elif dst == self.rank:
                buf = ops.empty_block()
                if self.staging and buf.is_cuda:
                    host = buf.new_empty(buf.shape, device="cpu")
                    reqs.append(dist.irecv(host, src, group=self.group))
                    staged.append((buf, host))
                else:
                    reqs.append(dist.irecv(buf, src, group=self.group))
                out[(dst, c)] = buf
        for r in reqs:
            r.wait()
        for x in staged:
            if isinstance(x, tuple):
                x[0].copy_(x[1])
        ops.sync()
        return out

    def done_reading(self, ops):
        pass  # received blocks are private copies

    def barrier(self):
        self.dist.barrier(group=self.group)


class PeerBlock:
    """A block that lives in a peer process's device memory (opened via CUDA
    IPC): duck-types the two tensor methods the block ops use."""

    def __init__(self, ptr: int, numel: int):
        self._ptr, self._numel = ptr, numel

    def data_ptr(self) -> int:
        return self._ptr

    def numel(self) -> int:
        return self._numel


class IpcComm(DistComm):
    """P2P transport over CUDA IPC (see the module docstring). Round protocol:
    every rank finishes its stream, then all-gathers (block, owner, handle,
    offset) for the blocks others need; consumers open each peer allocation
    once and read it in place. ``done_reading`` (sync + barrier) fences the
    owners' in-place REDUCE behind the peers' last reads."""

    def __init__(self, group=None):
        super().__init__(group, staging=False)
        from . import _lib

        self._lib = _lib
        self._opened: dict = {}  # (owner rank, owner base address) -> local base pointer

    def exchange(self, transfers, held, ops):
        import ctypes

        L = self._lib.load()
        ops.sync()  # blocks peers will read are complete before anyone reads them
        mine = []
        for c, src, dst in transfers:
            if src == self.rank:
                t = held[(src, c)]
                h = ctypes.create_string_buffer(64)
                off = ctypes.c_uint64(0)
                self._lib.check(L.dqmc_ipc_get(t.data_ptr(), h, ctypes.byref(off)))
                mine.append((c, dst, h.raw, int(off.value), t.data_ptr() - int(off.value), int(t.numel())))
        allx = [None] * self.world
        self.dist.all_gather_object(allx, mine, group=self.group)
        out = {}
        for src, lst in enumerate(allx):
            for c, dst, hb, off, base_id, numel in lst:
                if dst != self.rank:
                    continue
                key = (src, base_id)
                if key not in self._opened:
                    p = ctypes.c_void_p()
                    self._lib.check(L.dqmc_ipc_open(hb, ctypes.byref(p)))
                    self._opened[key] = int(p.value)
                out[(dst, c)] = PeerBlock(self._opened[key] + off, numel)
        return out

    def done_reading(self, ops):
        ops.sync()
        self.dist.barrier(group=self.group)
        L = self._lib.load()
        for base in self._opened.values():
            self._lib.check(L.dqmc_ipc_close(base))
        self._opened.clear()


def _dedupe(transfers: Iterable[tuple]) -> list[tuple]:
    seen, out = set(), []
    for x in transfers:
        if x not in seen:
            seen.add(x)
            out.append(x)
    return out


# ---------------------------------------------------------------------------
# the sharded algorithm


def sharded_prime_ranks(inputs: dict, n: int, k: int, ops, comm) -> dict:
    """Run the schedule. ``inputs[g]`` is rank g's local table slice (for the
    ranks local to ``comm``). Returns {top block t: ranks of P_t (global
    ranks, ascending)} for the blocks owned by local ranks."""
    nl = n - k
    if nl < 5:
        raise ValueError(f"sharding needs n - k >= 5, got n={n}, k={k}")
    own = owner_map(k)
    held: dict = {}
    for g in comm.local_ranks():
        held[(g, binary_block(g, k))] = ops.merge(inputs[g], nl)
    # (2) star blocks, one round per top axis
    for jobs in star_rounds(k):
        transfers = _dedupe((c, own[c], own[t]) for t, c0, c1 in jobs for c in (c0, c1) if own[c] != own[t])
        recv = comm.exchange(transfers, held, ops)
        for t, c0, c1 in jobs:
            o = own[t]
            if comm.is_local(o):
                a = held[(o, c0)] if (o, c0) in held else recv[(o, c0)]
                b = held[(o, c1)] if (o, c1) in held else recv[(o, c1)]
                held[(o, t)] = ops.and_(a, b)
        del recv
    # received children were temporaries; keep only owned blocks
    held = {(g, t): v for (g, t), v in held.items() if own[t] == g}
    # (3) kills from the top-axis parents (pre-reduce M)
    transfers = _dedupe((p, own[p], own[t]) for t in all_blocks(k) for p in parents(t) if own[p] != own[t])
    recv = comm.exchange(transfers, held, ops)
    kills = {}
    for t in all_blocks(k):
        o = own[t]
        if not comm.is_local(o):
            continue
        kill = None
        for p in parents(t):
            src = held[(o, p)] if (o, p) in held else recv[(o, p)]
            kill = ops.copy(src) if kill is None else ops.or_(kill, src)
        kills[t] = kill
    del recv
    ops.sync()
    comm.done_reading(ops)  # P2P: peers have read every M_t before it is reduced in place
    # (4) reduce the low dimensions, apply the kills, compact with the block offset
    out = {}
    for t in all_blocks(k):
        o = own[t]
        if comm.is_local(o):
            out[t] = ops.reduce_extract(held[(o, t)], nl, kills[t], rho(t) * 3**nl)
    return out


def concat_ranks(parts: dict) -> np.ndarray:
    """Global ascending rank list from {t: ranks} (blocks are disjoint rank ranges)."""
    arrs = [np.asarray(parts[t]) for t in sorted(parts, key=rho)]
    return np.concatenate(arrs).astype(np.int64) if arrs else np.zeros(0, dtype=np.int64)


# ---------------------------------------------------------------------------
# GPU ops (libdqmc.so + torch buffers)


class GpuOps:
    """Local compute on the current CUDA device through the C ABI."""

    def __init__(self, n_local: int, device=None):
        import torch

        from . import _lib
        from .dense import state_bytes

        self.torch = torch
        self._lib = _lib
        self.L = _lib.load()
        self.nl = n_local
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.words = state_bytes(n_local, 5) // 4
        self.rank_buf = None

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def empty_block(self):
        return self.torch.empty(self.words, dtype=self.torch.int32, device=self.device)

    def sync(self):
        self.torch.cuda.current_stream(self.device).synchronize()

    def merge(self, values, nl):
        out = self.empty_block()
        kind = self._lib.IN_U8 if values.dtype == self.torch.uint8 else self._lib.IN_WORDS
        self._lib.check(self.L.dqmc_merge_device(values.data_ptr(), kind, nl, out.data_ptr(), self._stream()))
        return out

    def _bitop(self, a, b, op, out=None):
        out = self.empty_block() if out is None else out
        self._lib.check(self.L.dqmc_bitop_device(out.data_ptr(), a.data_ptr(), b.data_ptr(), a.numel() * 4, op,
                                                 self._stream()))
        return out

    def and_(self, a, b):
        return self._bitop(a, b, 0)

    def or_(self, dst, src):
        return self._bitop(dst, src, 1, out=dst)

    def copy(self, src):
        if isinstance(src, self.torch.Tensor):
            return src.clone()
        return self._bitop(src, src, 0)  # a peer block: x & x, read over P2P

    def reduce_extract(self, block, nl, kill, offset):
        import ctypes

        cnt = ctypes.c_int64(0)
        if self.rank_buf is None:
            self.rank_buf = self.torch.empty(1 << 22, dtype=self.torch.int64, device=self.device)
        kp = kill.data_ptr() if kill is not None else None
        work = block  # reduced in place (all readers of M_t are done)
        for _ in range(2):
            self._lib.check(self.L.dqmc_reduce_extract_device(
                work.data_ptr(), nl, kp, int(offset), self.rank_buf.data_ptr(), self.rank_buf.numel(),
                ctypes.byref(cnt), 0, self._stream()))
            if cnt.value <= self.rank_buf.numel():
                break
            # REDUCE is idempotent and the kills are applied outside the block,
            # so the already-reduced block can simply be extracted again
            self.rank_buf = self.torch.empty(int(cnt.value * 1.1) + 1024, dtype=self.torch.int64, device=self.device)
        return self.rank_buf[: cnt.value].clone()


def gpu_sharded_prime_ranks_emulated(values_full, n: int, k: int) -> np.ndarray:
    """All 2^k shards on the current GPU, one after another (no collective):
    the k-GPU schedule, checked bit-exact against the 1-GPU engine."""
    import torch

    nl = n - k
    ops = GpuOps(nl)
    inputs = {g: values_full[g << nl : (g + 1) << nl] for g in range(1 << k)}
    parts = sharded_prime_ranks(inputs, n, k, ops, EmulatedComm(1 << k))
    return concat_ranks({t: v.cpu().numpy() for t, v in parts.items()})


def bench_main(args, workload, metric, unit):  # pragma: no cover - needs N GPUs
    """bench.py under torchrun (N > 1): config-4 workload sharded on the top
    log2(N) variables; device time of the whole schedule, max over ranks."""
    import json
    import os

    import torch
    import torch.distributed as dist

    from . import _lib

    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    backend = os.environ.get("DQMC_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local % ndev))
    else:  # gloo with host staging (tests: several ranks sharing one GPU)
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    k = world.bit_length() - 1
    if 1 << k != world:
        raise SystemExit("world size must be a power of two")
    n = args.n
    nl = n - k
    # this rank's slice of the frozen generator: points [rank*2^nl, (rank+1)*2^nl)
    vals = torch.empty(1 << nl, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().dqmc_gen3_range_device(vals.data_ptr(), rank << nl, 1 << nl, workload["p_on"],
                                                   workload["p_dc"], workload["seed"],
                                                   torch.cuda.current_stream().cuda_stream))
    ops = GpuOps(nl)
    # DQMC_DIST_TRANSPORT=p2p: CUDA-IPC peer reads (IpcComm); default: block send/recv
    if os.environ.get("DQMC_DIST_TRANSPORT", "sendrecv") == "p2p":
        comm = IpcComm()
    else:
        comm = DistComm(staging=backend != "nccl")

    def step():
        parts = sharded_prime_ranks({rank: vals}, n, k, ops, comm)
        return sum(int(v.numel()) for v in parts.values())

    # e2e step: this rank's slice from pinned host memory, its primes back to the host
    host_vals = torch.empty(1 << nl, dtype=torch.uint8, pin_memory=True)
    host_vals.copy_(vals.cpu())
    h2d = torch.empty_like(vals)

    def e2e_step():
        h2d.copy_(host_vals, non_blocking=True)
        parts = sharded_prime_ranks({rank: h2d}, n, k, ops, comm)
        outs = [v.cpu() for v in parts.values()]
        return sum(int(o.numel()) for o in outs)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cnt = 0
    for _ in range(args.steps):
        cnt = step()
    e1.record()
    torch.cuda.synchronize()
    # e2e (host buffers) under the same barrier + max-over-ranks rule
    dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        e2e_step()
    e3.record()
    torch.cuda.synchronize()
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps, e2.elapsed_time(e3) / 1e3 / args.steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([cnt], device=dev, dtype=torch.int64)
    dist.all_reduce(c)
    if rank == 0:
        tmax = float(t[0].item())
        te2e = float(t[1].item())
        line = {
            "metric": metric, "value": 3**n / tmax, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tmax * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (frozen generator, per-rank slice on device)",
            "config": {"workload": "BASELINE config 4 sharded on the top log2(N) variables", "n": n, "k": k,
                       "primes": int(c.item()), "backend": backend},
            "e2e": {"value": 3**n / te2e, "unit": unit, "ms_per_step": te2e * 1e3,
                    "h2d_bytes_per_step": int(1 << n), "d2h_bytes_per_step": int(c.item()) * 8},
            "gpu_launches": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0
