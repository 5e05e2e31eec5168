"""Top-k-variable sharding of the dense path over 2^k GPUs.

GPU g owns the assignment of the top k variables given by the bits of g, and
its truth-table slice [g*2^(n-k), (g+1)*2^(n-k)) (the top variables are the
most significant index bits). The 3^n cells are cut into SUPER-BLOCKS by the
top K = k + m variables: super-block d is a K-digit ternary tuple (digits
0..m-1 = variables n-K+1..n-k, the top of a GPU's own cube; digits m..K-1 =
the k GPU variables), and it holds the 3^L cells (L = n - K) of the contiguous
global rank range [rho(d)*3^L, (rho(d)+1)*3^L) in the h=5 layout. So the global
prime list is the concatenation of the super-blocks' lists in rho order.

Ownership (the interleaved rule of SURVEY.md §8(e), refined by super-block):
bit j of owner(d) is the GPU digit t_j when it is 0/1, and bit j of
h(s) = rho(s) mod 2^k when t_j is a star, s = the m local top digits. Then
  * every binary-t super-block (t = bits of g) lies on g: the whole 3^(n-k)
    cube of g is local and contiguous (slots 0..3^m-1 of g's arena);
  * a star super-block's two children along its highest star GPU axis j
    differ from it only in bit j of the owner: one is local, the other is on
    peer g XOR e_j;
  * each GPU holds ~1.5^k of the 3^k top blocks, i.e. 3^n/2^k cells:
    125.5 GB of the 1.004 TB state at n=27 on 8 GPUs (127.6 GB with the
    rounding of 3^m super-blocks; ShardPlan.budget).
The algorithm (composition verified on the reference):
  1. MERGE: each GPU merges its own cube (dqmc_merge_device); star
     super-blocks are then, level by level (number of star GPU digits), the
     AND of their two children, one read in place from the peer over NVLink
     (block-level MERGE of dense.py:174-212, merge_triple dense.py:46-48).
  2. REDUCE of the strided low groups: every rank reduces them for all its
     super-blocks in place, in one batched set of passes — its own cube over
     all n-k variables (its local-digit parents are inside it, and no other
     super-block reads it as a parent), the star super-blocks over L.
  3. Primes of super-block d = R_low(M_d) AND NOT OR_i R_A(M_{d[i->*]}) over
     its fixed top digits i (own-cube super-blocks: only the GPU digits), where
     R_A is the partial low REDUCE of step 2
     (oracle formula oracle.py:77-80 with M_parent replaced by any partial
     low REDUCE of it: a parent cleared by one of its own low parents means
     the cell's low parent along that axis is an implicant, so the cell dies
     either way; the parents must NOT carry their own top kills). One final
     pass over all of a rank's super-blocks finishes each tile's low REDUCE
     in shared memory, reads the <= K parents in place (local or peer
     pointers, a per-slot table) and applies their OR in registers: no kill
     buffers, no staging copies, and one fence between steps 2 and 3.
  4. Compaction with each super-block's global rank offset, slot by slot.
NCCL has no bitwise-AND reduction (nccl.h ops: sum/prod/max/min/avg) and the
exchange here is pure peer loads, so the only collectives are the level
fences and the one-time exchange of arena IPC handles.

The same schedule runs over all 2^k ranks inside one process
(``EmulatedComm``: one GPU checks k-GPU bit-exactness) or one process per rank
(``ProcessComm``: torch.distributed for the fences, arena handles exchanged
once). Local compute is an ``ops`` object: ``GpuOps`` (libdqmc.so) in
production; the CPU tests plug in oracle-backed ops over shared memory.
"""

from __future__ import annotations

import itertools
import json
from dataclasses import dataclass

import numpy as np

MAX_KILL = 8  # parent super-blocks the final pass can read (kMaxKill, csrc/dqmc_internal.cuh)
BALANCE = 1.02  # target max/ideal arena bytes when choosing m


def rho(d) -> int:
    """Rank of a digit tuple (digit i has weight 3^i)."""
    return sum(int(x) * 3**i for i, x in enumerate(d))


def state_bytes5(n: int) -> int:
    """dqmc_state_bytes(n, 5): 3^(n-5) blocks of 256 bits (dense.py:56-63)."""
    return 3 ** (n - 5) * 32


def _owner(d, m: int, k: int) -> int:
    hs = rho(d[:m]) % (1 << k) if k else 0
    g = 0
    for j in range(k):
        t = d[m + j]
        g |= (t if t < 2 else (hs >> j) & 1) << j
    return g


def _arena_counts(k: int, m: int) -> list[int]:
    cnt = [0] * (1 << k)
    for d in itertools.product((0, 1, 2), repeat=k + m):
        cnt[_owner(d, m, k)] += 1
    return cnt


def choose_m(n: int, k: int) -> int:
    """Smallest m whose super-block rounding keeps every GPU within BALANCE of
    the ideal 3^n / 2^k cells, subject to K = k + m <= MAX_KILL and L >= 5."""
    hi = min(MAX_KILL - k, n - k - 5)
    if k == 0 or hi <= 0:
        return 0
    for m in range(1, hi + 1):
        if max(_arena_counts(k, m)) * 2**k <= BALANCE * 3 ** (k + m):
            return m
    return hi


@dataclass(frozen=True)
class Ref:
    """A super-block's location: rank and byte offset inside its arena."""

    rank: int
    off: int


class ShardPlan:
    """The whole schedule of one sharded call, identical on every rank."""

    def __init__(self, n: int, k: int, m: int | None = None):
        if not 0 <= k <= 3:
            raise ValueError(f"k must be in 0..3 (1..8 GPUs), got {k}")
        if n - k < 5:
            raise ValueError(f"sharding needs n - k >= 5, got n={n}, k={k}")
        self.n, self.k = n, k
        self.m = choose_m(n, k) if m is None else int(m)
        self.K = k + self.m
        self.L = n - self.K
        if self.m < 0 or self.K > MAX_KILL or self.L < 5:
            raise ValueError(f"bad super-block split m={self.m} for n={n}, k={k}")
        self.world = 1 << k
        self.sb_bytes = state_bytes5(self.L)
        m = self.m
        self.blocks = sorted(itertools.product((0, 1, 2), repeat=self.K), key=rho)
        self.owner = {d: _owner(d, m, k) for d in self.blocks}
        # arena slots: the rank's own cube first (binary GPU digits = bits of g,
        # local digits in rho order: exactly dqmc_merge_device's output), then
        # its star super-blocks in rho order
        self.slot: dict[tuple, int] = {}
        nslots = [3**m] * self.world
        for d in self.blocks:
            t = d[m:]
            if 2 not in t:
                self.slot[d] = rho(d[:m])
        for d in self.blocks:
            if d not in self.slot:
                g = self.owner[d]
                self.slot[d] = nslots[g]
                nslots[g] += 1
        self.nslots = nslots
        self.slot_blocks = [[None] * nslots[g] for g in range(self.world)]  # rank -> super-block per slot
        for d in self.blocks:
            self.slot_blocks[self.owner[d]][self.slot[d]] = d
        self.merge_levels = self._merge_levels()

    # -- layout
    def ref(self, d) -> Ref:
        return Ref(self.owner[d], self.slot[d] * self.sb_bytes)

    def offset(self, d) -> int:
        """Global rank of the super-block's first cell."""
        return rho(d) * 3**self.L

    def arena_bytes(self, g: int) -> int:
        return self.nslots[g] * self.sb_bytes

    # -- schedule
    def _merge_levels(self):
        """Level w (1..k): (d, child0, child1) for every super-block with w star
        GPU digits, split along its highest star GPU digit."""
        m = self.m
        levels = []
        for w in range(1, self.k + 1):
            jobs = []
            for d in self.blocks:
                stars = [j for j in range(self.k) if d[m + j] == 2]
                if len(stars) != w:
                    continue
                j = m + max(stars)
                c0 = d[:j] + (0,) + d[j + 1 :]
                c1 = d[:j] + (1,) + d[j + 1 :]
                jobs.append((d, c0, c1))
            levels.append(jobs)
        return levels

    def parents(self, d) -> list:
        """The super-blocks d[i->*] over d's fixed digits (<= K <= MAX_KILL)."""
        return [d[:i] + (2,) + d[i + 1 :] for i in range(self.K) if d[i] != 2]

    def is_own(self, d) -> bool:
        """d lies in its owner's own cube (binary GPU digits)."""
        return 2 not in d[self.m :]

    @property
    def own_full(self) -> bool:
        """The own cube's strided low groups cover every variable above the
        super-blocks' 3^7-block C0 tile (L >= 12: both plans share that tile),
        so reduce_low can reduce the own cube over all its n-k variables."""
        return self.L >= 12 and self.m > 0

    def kill_parents(self, d) -> list:
        """The parents the extract pass reads for d. With own_full, a rank's
        own cube is reduced over all its n-k variables in place (its
        local-digit parents are inside it, and no other super-block reads it
        as a parent), so its super-blocks only need their GPU-digit parents;
        star super-blocks need every fixed digit's parent."""
        if self.own_full and self.is_own(d):
            return [d[:i] + (2,) + d[i + 1 :] for i in range(self.m, self.K) if d[i] != 2]
        return self.parents(d)

    # -- budget
    def tile_bytes(self) -> int:
        """Engine tile arrays of one super-block's final pass (20 B per C0 tile)."""
        t = max(0, self.L - 5 - 7)
        return 3**t * 20

    def peak_device_bytes(self, g: int, rank_bytes: int = 0) -> int:
        """Per-rank device peak: the arena, the rank's table slice (2^(n-k)
        uint8) and its packed words, the engine's tile arrays, and the rank
        output (0 when counting only)."""
        nl = self.n - self.k
        return self.arena_bytes(g) + (1 << nl) + (1 << nl) // 8 + self.tile_bytes() + rank_bytes

    def budget(self) -> dict:
        """Dry-run summary (bench.py --dry-run)."""
        total = state_bytes5(self.n)
        peaks = [self.peak_device_bytes(g) for g in range(self.world)]
        recv = self.peer_read_bytes()
        return {
            "n": self.n, "k": self.k, "m": self.m, "gpus": self.world, "low_vars": self.L,
            "super_blocks": len(self.blocks), "super_block_bytes": self.sb_bytes,
            "state_bytes_total": total, "ideal_bytes_per_gpu": total // self.world,
            "arena_bytes": [self.arena_bytes(g) for g in range(self.world)],
            "peak_device_bytes": peaks, "max_peak_device_bytes": max(peaks),
            "balance": max(peaks) / (total / self.world),
            "merge_levels": len(self.merge_levels),
            "peer_read_bytes": recv,
        }

    def check_budget(self, g: int, free_bytes: int, rank_bytes: int = 0) -> int:
        """Refuse before allocating, as load() does (dense.py:358-364): raise
        ResourceLimitError naming the bytes rank g needs if they exceed
        free_bytes. Returns the need."""
        need = self.peak_device_bytes(g, rank_bytes)
        if need > free_bytes:
            from . import errors

            raise errors.ResourceLimitError(
                f"sharded n={self.n} on {self.world} GPUs: rank {g} needs {need} bytes "
                f"({self.nslots[g]} super-blocks of {self.sb_bytes} bytes), only {free_bytes} bytes are free"
            )
        return need

    def peer_read_bytes(self) -> list[int]:
        """Bytes each rank reads from peers over the schedule (AND inputs + kills)."""
        out = [0] * self.world
        for jobs in self.merge_levels:
            for d, c0, c1 in jobs:
                g = self.owner[d]
                out[g] += sum(self.sb_bytes for c in (c0, c1) if self.owner[c] != g)
        for d in self.blocks:
            g = self.owner[d]
            out[g] += sum(self.sb_bytes for p in self.kill_parents(d) if self.owner[p] != g)
        return out


# ---------------------------------------------------------------------------
# the schedule


def run_schedule(plan: ShardPlan, inputs: dict, ops, comm, count_only: bool = False) -> dict:
    """Run the sharded call. ``inputs[g]`` is rank g's table slice for every
    rank local to ``comm``. Returns {d: result} for the super-blocks those
    ranks own: a (start, count) span of ops' rank output, or a count."""
    local = comm.local_ranks()
    for g in local:
        ops.ensure_arena(g, plan.arena_bytes(g))
    comm.share(ops)
    nl = plan.n - plan.k
    for g in local:
        ops.merge(inputs[g], nl, Ref(g, 0))
    comm.fence(ops)
    for jobs in plan.merge_levels:  # star super-blocks: one batched AND per level and rank
        for g in local:
            mine = [(plan.ref(d), plan.ref(c0), plan.ref(c1)) for d, c0, c1 in jobs if plan.owner[d] == g]
            ops.and_batch(mine, plan.sb_bytes)
        comm.fence(ops)
    own = 3**plan.m if plan.own_full else 0
    for g in local:  # strided low groups, in place: the own cube over all its n-k variables, the rest over L
        if own:
            ops.reduce_low(g, nl, 1, 0)
        if plan.nslots[g] > own:
            ops.reduce_low(g, plan.L, plan.nslots[g] - own, own * plan.sb_bytes)
    comm.fence(ops)  # parents are read only once every rank has reduced them
    out = {}
    for g in local:
        slots = plan.slot_blocks[g]
        kills = [[plan.ref(q) for q in plan.kill_parents(d)] for d in slots]
        res = ops.extract(g, plan.L, kills, [plan.offset(d) for d in slots], count_only)
        out.update(zip(slots, res))
    comm.fence(ops)  # nobody reads an arena once its owner may rewrite it (next call)
    return out


def ordered(parts: dict) -> list:
    """Results in global rank order (super-blocks are disjoint rank ranges)."""
    return [parts[d] for d in sorted(parts, key=rho)]


# ---------------------------------------------------------------------------
# communication


class EmulatedComm:
    """All 2^k ranks inside one process: every arena is local."""

    def __init__(self, world: int):
        self.world = world

    def local_ranks(self) -> list[int]:
        return list(range(self.world))

    def share(self, ops):
        pass

    def fence(self, ops):
        ops.sync()

    def close(self, ops):
        pass


class ProcessComm:
    """One rank per process of a torch.distributed group (NCCL on 8 GPUs;
    gloo for CPU tests and for several ranks sharing one GPU). ``share``
    exchanges each arena's handle once (CUDA IPC on GPUs, a shared-memory name
    on CPU); every later access is a peer load inside our kernels. ``fence``
    = local stream sync + barrier: no kernel ever waits on another process."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._shared = None

    def local_ranks(self) -> list[int]:
        return [self.rank]

    def share(self, ops):
        # every rank learns every arena's identity; if none changed since the
        # last call the opened peer handles are still valid (one small
        # all-gather per call), else all ranks re-export and re-open
        keys = [None] * self.world
        self.dist.all_gather_object(keys, ops.arena_key(self.rank), group=self.group)
        if self._shared == keys:
            return
        if self._shared is not None:
            ops.close_peers()
        mine = ops.export_arena(self.rank)
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        for g, h in enumerate(allh):
            if g != self.rank:
                ops.import_arena(g, h)
        self._shared = keys

    def fence(self, ops):
        ops.sync()
        self.dist.barrier(group=self.group)

    def close(self, ops):
        if self._shared is not None:
            self.fence(ops)
            ops.close_peers()
            self._shared = None


# ---------------------------------------------------------------------------
# GPU ops (libdqmc.so + torch buffers)


class GpuOps:
    """Super-block compute on the current CUDA device through the C ABI.
    Ranks of every super-block are written back to back into one device
    buffer (``out``); extract returns their (start, count) spans."""

    def __init__(self, device=None):
        import torch

        from . import _lib

        self.torch = torch
        self._lib = _lib
        self.L = _lib.load()
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.arenas: dict[int, object] = {}  # local rank -> uint8 tensor
        self.bases: dict[int, int] = {}  # rank -> device address of its arena (local or IPC-mapped)
        self._opened: list[int] = []
        self.out = None
        self.cursor = 0

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def ptr(self, ref: Ref) -> int:
        return self.bases[ref.rank] + ref.off

    def sync(self):
        self.torch.cuda.current_stream(self.device).synchronize()

    def ensure_arena(self, g: int, nbytes: int):
        a = self.arenas.get(g)
        if a is None or a.numel() < nbytes:
            self.arenas[g] = None
            a = self.torch.empty(max(nbytes, 16), dtype=self.torch.uint8, device=self.device)
            self.arenas[g] = a
        self.bases[g] = a.data_ptr()

    def arena_key(self, g: int):
        return self.arenas[g].data_ptr()

    def export_arena(self, g: int):
        import ctypes

        h = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64(0)
        self._lib.check(self.L.dqmc_ipc_get(self.arenas[g].data_ptr(), h, ctypes.byref(off)))
        return (h.raw, int(off.value))

    def import_arena(self, g: int, handle):
        import ctypes

        raw, off = handle
        p = ctypes.c_void_p()
        self._lib.check(self.L.dqmc_ipc_open(raw, ctypes.byref(p)))
        self._opened.append(int(p.value))
        self.bases[g] = int(p.value) + off

    def close_peers(self):
        for base in self._opened:
            self._lib.check(self.L.dqmc_ipc_close(base))
        self._opened.clear()

    def reset_output(self):
        self.cursor = 0

    def merge(self, values, nl: int, dst: Ref):
        kind = self._lib.IN_U8 if values.dtype == self.torch.uint8 else self._lib.IN_WORDS
        self._lib.check(self.L.dqmc_merge_device(values.data_ptr(), kind, nl, self.ptr(dst), self._stream()))

    def and_batch(self, triples, nbytes: int):
        """dst = a & b for every (dst, a, b) of one merge level: one launch."""
        if not triples:
            return
        t = self.torch
        jobs = t.tensor([[self.ptr(d), self.ptr(a), self.ptr(b)] for d, a, b in triples], dtype=t.int64)
        self._jobs = jobs.to(self.device, non_blocking=False)  # kept alive until the launch has read it
        self._lib.check(self.L.dqmc_bitop_batch_device(self._jobs.data_ptr(), len(triples), nbytes, 0,
                                                       self._stream()))

    def reduce_low(self, g: int, n: int, nstates: int, off: int):
        self._lib.check(self.L.dqmc_reduce_low_device(self.bases[g] + off, n, nstates, self._stream()))

    def extract(self, g: int, L: int, kills: list, rank_adds: list, count_only: bool):
        """Primes of rank g's nslots super-blocks: [(start, count)] spans of
        ``out`` in slot order, or counts."""
        import ctypes

        t = self.torch
        nslots = len(kills)
        key = (g, L, tuple(self.bases.items()))
        if getattr(self, "_tab_key", None) != key:  # tables depend only on the plan and the arenas
            tab = [[self.ptr(r) for r in ks] + [0] * (MAX_KILL - len(ks)) for ks in kills]
            self._tab = t.tensor(tab, dtype=t.int64).to(self.device)
            self._radd = t.tensor(rank_adds, dtype=t.int64).to(self.device)
            self._spans = t.empty((2, nslots), dtype=t.int64, device=self.device)
            self._tab_key = key
        total = ctypes.c_int64(0)
        flags = self._lib.FLAG_COUNT_ONLY if count_only else 0
        if self.out is None:
            self.out = t.empty(1 << 22, dtype=t.int64, device=self.device)
        for _ in range(2):
            free = 0 if count_only else self.out.numel() - self.cursor
            dst = None if count_only else self.out.data_ptr() + 8 * self.cursor
            self._lib.check(self.L.dqmc_extract_kills_device(
                self.bases[g], L, nslots, self._tab.data_ptr(), self._radd.data_ptr(), dst, free,
                self._spans[0].data_ptr(), self._spans[1].data_ptr(), ctypes.byref(total), flags, self._stream()))
            if count_only or total.value <= free:
                break
            # grow the output and extract again (the arena is read, not written)
            bigger = t.empty(max(2 * self.out.numel(), self.cursor + int(total.value * 1.25) + 1024),
                             dtype=t.int64, device=self.device)
            bigger[: self.cursor].copy_(self.out[: self.cursor])
            self.out = bigger
        starts, counts = self._spans.cpu().tolist()
        if count_only:
            return counts
        res = [(self.cursor + a, c) for a, c in zip(starts, counts)]
        self.cursor += int(total.value)
        return res

    def gather(self, parts: dict):
        """Device int64 ranks of the given super-blocks in global rank order."""
        spans = ordered(parts)
        if not spans:
            return self.torch.zeros(0, dtype=self.torch.int64, device=self.device)
        return self.torch.cat([self.out[s : s + c] for s, c in spans])


def gpu_sharded_prime_ranks_emulated(values_full, n: int, k: int, m: int | None = None) -> np.ndarray:
    """All 2^k ranks on the current GPU in one process (no collective): the
    k-GPU schedule, checked bit-exact against the 1-GPU engine."""
    plan = ShardPlan(n, k, m)
    nl = n - k
    ops = GpuOps()
    inputs = {g: values_full[g << nl : (g + 1) << nl] for g in range(plan.world)}
    parts = run_schedule(plan, inputs, ops, EmulatedComm(plan.world))
    return ops.gather(parts).cpu().numpy()


def dry_run(n: int, k: int) -> dict:
    return ShardPlan(n, k).budget()


# ---------------------------------------------------------------------------
# bench.py under torchrun (N > 1)


def bench_main(args, workload, metric, unit, clock_sampler=None):  # pragma: no cover - needs N GPUs
    """The workload sharded on the top log2(N) variables, one rank per GPU;
    CUDA-event time of the whole schedule, max over ranks. The same n at every
    N (total work fixed): strong scaling."""
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
    else:  # gloo (several ranks sharing one GPU in tests)
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    k = world.bit_length() - 1
    if 1 << k != world:
        raise SystemExit("world size must be a power of two")
    n = args.n
    plan = ShardPlan(n, k)
    nl = n - k
    count_only = n > 25  # config 5: 3-4e10 primes (~300 GB of ranks); the deliverable is counts
    free, _ = torch.cuda.mem_get_info()
    plan.check_budget(rank, free)
    vals = torch.empty(1 << nl, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().dqmc_gen3_range_device(vals.data_ptr(), rank << nl, 1 << nl, workload["p_on"],
                                                   workload["p_dc"], workload["seed"],
                                                   torch.cuda.current_stream().cuda_stream))
    ops = GpuOps()
    comm = ProcessComm()

    def step(src):
        ops.reset_output()
        parts = run_schedule(plan, {rank: src}, ops, comm, count_only=count_only)
        return parts

    def primes_of(parts):
        return sum(int(v) if count_only else int(v[1]) for v in parts.values())

    host_vals = torch.empty(1 << nl, dtype=torch.uint8, pin_memory=True)
    host_vals.copy_(vals.cpu())
    h2d = torch.empty_like(vals)

    for _ in range(args.warmup):
        step(vals)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = int(_lib.load().dqmc_launch_count())
    clk = None
    if clock_sampler is not None and rank == 0:  # SM clocks and throttle reasons during the timed region
        try:
            clk = clock_sampler(local % ndev)
            clk.__enter__()
        except Exception:
            clk = None
    e0.record()
    parts = None
    for _ in range(args.steps):
        parts = step(vals)
    e1.record()
    torch.cuda.synchronize()
    clocks = None
    if clk is not None:
        clk.__exit__(None, None, None)
        clocks = clk.summary()
    launches = int(_lib.load().dqmc_launch_count()) - launches0  # this rank's kernels in the timed region
    cnt = primes_of(parts)
    # e2e: this rank's slice from pinned host memory, its primes back to (pinned) host memory
    host_out = None if count_only else torch.empty(int(cnt * 1.05) + 1024, dtype=torch.int64, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    d2h = 0
    for _ in range(args.steps):
        h2d.copy_(host_vals, non_blocking=True)
        parts = step(h2d)
        if count_only:
            d2h = 8 * len(parts)
        else:
            mine = ops.gather(parts)
            if host_out is None or host_out.numel() < mine.numel():
                host_out = torch.empty(int(mine.numel() * 1.05) + 1024, dtype=torch.int64, pin_memory=True)
            host_out[: mine.numel()].copy_(mine, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            d2h = mine.numel() * 8
    e3.record()
    torch.cuda.synchronize()
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps, e2.elapsed_time(e3) / 1e3 / args.steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([cnt, d2h, launches], device=dev, dtype=torch.int64)
    dist.all_reduce(c)
    comm.close(ops)
    if rank == 0:
        tmax = float(t[0].item())
        te2e = float(t[1].item())
        b = plan.budget()
        line = {
            "metric": metric, "value": 3**n / tmax, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tmax * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (frozen generator, per-rank slice on device)",
            "config": {"workload": workload.get("name", "sharded"), "n": n, "k": k, "m": plan.m,
                       "primes": int(c[0].item()), "count_only": count_only, "backend": backend,
                       "max_peak_device_bytes": b["max_peak_device_bytes"]},
            "e2e": {"value": 3**n / te2e, "unit": unit, "ms_per_step": te2e * 1e3,
                    "h2d_bytes_per_step": int(1 << n), "d2h_bytes_per_step": int(c[1].item())},
            "gpu_launches": int(c[2].item()),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":  # pragma: no cover
    import argparse

    ap = argparse.ArgumentParser(description="per-rank byte budget of the sharded plan (no GPU needed)")
    ap.add_argument("--n", type=int, default=27)
    ap.add_argument("--k", type=int, default=3)
    a = ap.parse_args()
    print(json.dumps(dry_run(a.n, a.k), indent=1))
