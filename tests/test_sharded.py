"""Top-k sharding: the super-block plan and its byte budget,
the schedule on CPU (one process, and gloo worlds of 2 and 4 processes whose
arenas live in shared memory, the CPU stand-in for CUDA IPC), and on the GPU
the k-rank schedule compared bit-exactly with the single-GPU engine.

On CPU the per-super-block compute is done by the oracle (test
infrastructure); the code under test is the plan + schedule in
paper_2302_10083_b200.sharded, which is the same code the GPU path runs.
"""

import hashlib
import os
import socket
from multiprocessing import shared_memory

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_10083_b200 import sharded as S


class CpuOps:
    """Oracle MERGE / REDUCE over numpy arenas in POSIX shared memory: a peer
    arena is opened by name exactly as a GPU peer arena is opened by its IPC
    handle, and read in place."""

    def __init__(self):
        from oracle import oracle as O

        self.O = O
        self.shm = {}  # rank -> SharedMemory (own and opened peers)
        self.own = set()

    def ensure_arena(self, g, nbytes):
        if g in self.shm and self.shm[g].size >= nbytes:
            return
        self.shm[g] = shared_memory.SharedMemory(create=True, size=max(nbytes, 16))
        self.own.add(g)

    def arena_key(self, g):
        return self.shm[g].name

    def export_arena(self, g):
        return self.shm[g].name

    def import_arena(self, g, name):
        self.shm[g] = shared_memory.SharedMemory(name=name)

    def close_peers(self):
        for g in [g for g in self.shm if g not in self.own]:
            self.shm.pop(g).close()

    def release(self):
        self.close_peers()
        for g in list(self.own):
            self.shm[g].close()
            self.shm[g].unlink()
        self.shm.clear()
        self.own.clear()

    def sync(self):
        pass

    def words(self, ref, nbytes):
        return np.ndarray((nbytes // 8,), dtype=np.uint64, buffer=self.shm[ref.rank].buf, offset=ref.off)

    def merge(self, values, nl, dst):
        from oracle import gen as G

        st = self.O.OracleState(G.values_to_words(values), nl, 5)
        st.run_pass(self.O.MERGE)
        self.words(dst, st.words.nbytes)[:] = st.words

    def and_batch(self, triples, nbytes):
        for dst, a, b in triples:
            np.bitwise_and(self.words(a, nbytes), self.words(b, nbytes), out=self.words(dst, nbytes))

    @staticmethod
    def _split(L):
        """As the GPU: reduce_low covers the strided groups (block digits above
        the 3^min(L-5, 7)-block C0 tile), extract the C0 and in-block dims."""
        c0 = 5 + min(L - 5, 7)
        return list(range(c0 + 1, L + 1)), list(range(1, c0 + 1))

    def reduce_low(self, g, n, nstates, off):
        nb = self.O.state_bytes(n, 5)
        groups, _ = self._split(n)
        if not groups:
            return
        for s in range(nstates):
            w = self.words(S.Ref(g, off + s * nb), nb)
            st = self.O.OracleState.from_words(w.copy(), n, 5)
            st.run_pass(self.O.REDUCE, dims=groups)
            w[:] = st.words  # in place, as the GPU does

    def extract(self, g, L, kills, rank_adds, count_only):
        nb = self.O.state_bytes(L, 5)
        _, rest = self._split(L)
        res = []
        for s, (ks, add) in enumerate(zip(kills, rank_adds)):
            st = self.O.OracleState.from_words(self.words(S.Ref(g, s * nb), nb).copy(), L, 5)
            st.run_pass(self.O.REDUCE, dims=rest)  # finish the low REDUCE (not written back)
            w = st.words
            for q in ks:  # parents as they are: only partially low-reduced
                w &= ~self.words(q, nb)
            r = self.O.OracleState.from_words(w, L, 5).extract_ranks() + add
            res.append(len(r) if count_only else r)
        return res


# ---------------------------------------------------------------------------
# the plan


def test_star_block_is_the_merge_of_the_anded_tables(oracle_mod, gen_mod):
    """MERGE is an AND-homomorphism on truth tables: a cube is an implicant of
    f0 AND f1 iff it is one of both. So the '*' block of the top variable
    (dense.py:174-212, u = s & t) equals the merged array of the table
    f0 & f1 on its own, and blocks 0/1 those of f0/f1: a rank can build any
    top block from ANDed 2^(n-k)-bit tables instead of exchanging
    3^(n-k)-bit arrays."""
    MERGE = 0
    for n, seed in ((9, 1), (12, 2), (14, 3)):
        words = gen_mod.random_words(n, 0.8, seed)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: 1 << n]
        f0, f1 = bits[: 1 << (n - 1)], bits[1 << (n - 1):]
        full = oracle_mod.OracleState(words, n)
        full.run_pass(MERGE)
        top = full.words.reshape(3, -1)  # the top variable is the slowest block digit: blocks 0, 1, *

        def merged(b):
            w = np.packbits(np.pad(b, (0, (-len(b)) % 64)), bitorder="little").view(np.uint64)
            st = oracle_mod.OracleState(w, n - 1)
            st.run_pass(MERGE)
            return st.words

        assert np.array_equal(top[0], merged(f0))
        assert np.array_equal(top[1], merged(f1))
        assert np.array_equal(top[2], merged(f0 & f1))


class TestPlan:
    @pytest.mark.parametrize("n,k", [(12, 1), (13, 2), (14, 3), (24, 3), (27, 3), (24, 1)])
    def test_ownership_rules(self, n, k):
        p = S.ShardPlan(n, k)
        m = p.m
        assert p.K <= S.MAX_KILL and p.L >= 5
        # every super-block has one owner; a rank's own cube is local, contiguous, in rho order
        for d in p.blocks:
            g = p.owner[d]
            t = d[m:]
            assert all(((g >> j) & 1) == x for j, x in enumerate(t) if x != 2)
            if 2 not in t:
                assert g == sum(x << j for j, x in enumerate(t)) and p.slot[d] == S.rho(d[:m])
        # slots of a rank are distinct and dense
        for g in range(p.world):
            slots = sorted(p.slot[d] for d in p.blocks if p.owner[d] == g)
            assert slots == list(range(p.nslots[g]))
        assert sum(p.nslots) * p.sb_bytes == S.state_bytes5(n)

    @pytest.mark.parametrize("k", [1, 2, 3])
    def test_merge_children_local_or_one_peer(self, k):
        p = S.ShardPlan(17, k)
        done = {d for d in p.blocks if 2 not in d[p.m:]}
        for jobs in p.merge_levels:
            for d, c0, c1 in jobs:
                assert c0 in done and c1 in done  # children computed in an earlier level
                g = p.owner[d]
                owners = {p.owner[c0], p.owner[c1]}
                assert g in owners
                other = (owners - {g}) or {g}
                assert bin(other.pop() ^ g).count("1") <= 1  # the other child is on g XOR e_j
            done |= {d for d, _, _ in jobs}
        assert done == set(p.blocks)

    @pytest.mark.parametrize("n,k", [(16, 1), (16, 2), (16, 3), (22, 2), (24, 3)])
    def test_parents_exist_and_fit_the_kill_table(self, n, k):
        p = S.ShardPlan(n, k)
        read = set()
        for d in p.blocks:
            ps = p.parents(d)
            assert len(ps) == sum(x != 2 for x in d) <= S.MAX_KILL
            assert all(q in p.owner for q in ps)
            kp = p.kill_parents(d)
            assert set(kp) <= set(ps) and (kp == ps or (p.own_full and p.is_own(d)))
            read |= set(kp)
        # with own_full the own cubes are reduced over all their variables in place: nobody may read them
        if p.own_full:
            assert not any(p.is_own(q) for q in read)
        for g in range(p.world):  # slot lists cover each rank's arena exactly
            assert [p.slot[d] for d in p.slot_blocks[g]] == list(range(p.nslots[g]))

    def test_own_cube_full_reduce_only_with_a_shared_c0_tile(self):
        assert S.ShardPlan(27, 3).own_full and S.ShardPlan(24, 3).own_full
        assert not S.ShardPlan(16, 2).own_full  # L = 10: the own cube's C0 tile differs

    def test_super_blocks_tile_the_rank_space(self):
        p = S.ShardPlan(12, 2)
        ranges = sorted((p.offset(d), p.offset(d) + 3**p.L) for d in p.blocks)
        assert ranges[0][0] == 0 and ranges[-1][1] == 3**12
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))

    def test_config5_fits_eight_b200(self):
        """n=27 on 8 GPUs: every rank's peak (arena + table slice + words +
        tile arrays) stays under 150 GB of a B200's ~180 GB."""
        b = S.ShardPlan(27, 3).budget()
        assert b["max_peak_device_bytes"] <= 150e9
        assert b["balance"] <= 1.02
        assert sum(b["arena_bytes"]) == 3**22 * 32  # state_bytes(27, 5) = 1.004 TB in total

    @pytest.mark.parametrize("k", [1, 2, 3])
    def test_n24_arena_is_one_over_2k_of_the_state(self, k):
        p = S.ShardPlan(24, k)
        ideal = S.state_bytes5(24) / 2**k
        assert max(p.arena_bytes(g) for g in range(p.world)) <= 1.03 * ideal

    def test_over_budget_raises_before_allocating(self, pkg):
        p = S.ShardPlan(27, 3)
        need = p.peak_device_bytes(0)
        assert p.check_budget(0, need) == need
        with pytest.raises(pkg.ResourceLimitError, match=str(need)):
            p.check_budget(0, need - 1)

    def test_bad_splits(self):
        with pytest.raises(ValueError):
            S.ShardPlan(8, 4)
        with pytest.raises(ValueError):
            S.ShardPlan(7, 3)
        with pytest.raises(ValueError):
            S.ShardPlan(20, 3, m=6)  # K = 9 > MAX_KILL

    def test_dry_run_cli(self):
        import json
        import subprocess
        import sys

        r = subprocess.run([sys.executable, "-m", "paper_2302_10083_b200.sharded", "--n", "27", "--k", "3"],
                           capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr
        b = json.loads(r.stdout)
        assert b["gpus"] == 8 and b["max_peak_device_bytes"] <= 150e9


# ---------------------------------------------------------------------------
# the schedule on CPU


@pytest.mark.parametrize("n,k,m", [(8, 1, None), (9, 2, None), (10, 3, None), (11, 2, 2), (12, 3, 3), (11, 1, 0),
                                   (15, 1, 1), (16, 2, 1), (14, 1, 1)])
def test_emulated_cpu_matches_single_engine(n, k, m, oracle_mod, gen_mod):
    v = gen_mod.gen3(n, 0.7, 0.1, n)
    plan = S.ShardPlan(n, k, m)
    nl = n - k
    ops = CpuOps()
    try:
        inputs = {g: v[g << nl : (g + 1) << nl] for g in range(plan.world)}
        parts = S.run_schedule(plan, inputs, ops, S.EmulatedComm(plan.world))
        got = np.concatenate(S.ordered(parts)).astype(np.int64)
    finally:
        ops.release()
    want = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), n)
    assert np.array_equal(got, want)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, seed, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ops = CpuOps()
    try:
        from oracle import gen as G

        k = world.bit_length() - 1
        plan = S.ShardPlan(n, k, m=2)  # 3^(k+2) super-blocks keep the CPU oracle calls few
        nl = n - k
        v = G.gen3(n, 0.75, 0.05, seed)
        comm = S.ProcessComm()
        parts = S.run_schedule(plan, {rank: v[rank << nl : (rank + 1) << nl]}, ops, comm)
        comm.close(ops)
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(parts, gathered, dst=0)
        if rank == 0:
            allp = {}
            for d in gathered:
                allp.update(d)
            assert set(allp) == set(plan.blocks)
            np.save(os.path.join(outdir, "ranks.npy"), np.concatenate(S.ordered(allp)).astype(np.int64))
        dist.barrier()
    finally:
        ops.release()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 10), (4, 12)])
def test_gloo_sharded_equals_single(world, n, tmp_path, oracle_mod, gen_mod):
    mp.spawn(_worker, args=(world, _free_port(), n, 3, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "ranks.npy")
    v = gen_mod.gen3(n, 0.75, 0.05, 3)
    want = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), n)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# the schedule on the GPU


def _block_diff(got, want, plan):
    out = [f"total got {len(got)} want {len(want)}"]
    for d in plan.blocks:
        lo, hi = plan.offset(d), plan.offset(d) + 3**plan.L
        g, w = got[(got >= lo) & (got < hi)], want[(want >= lo) & (want < hi)]
        if not np.array_equal(g, w):
            out.append(f"super-block {d} (owner {plan.owner[d]}): got {len(g)} want {len(w)}")
    return "; ".join(out[:12])


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(12, 1), (14, 2), (17, 3), (20, 2), (22, 3), (21, 1)])
def test_gpu_emulated_shards_bit_exact(n, k, pkg):
    from paper_2302_10083_b200 import device

    vd = device.gen3_device(n, 0.75, 0.05, 3)
    got = S.gpu_sharded_prime_ranks_emulated(vd, n, k)
    want = pkg.prime_ranks_from_values(vd.cpu().numpy())
    assert np.array_equal(got, want), _block_diff(got, want, S.ShardPlan(n, k))


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 2, 3])
def test_gpu_emulated_config4(k, pkg, golden):
    """n=24 on 2^k emulated ranks == the reference's pins for config 4."""
    from paper_2302_10083_b200 import device

    g = golden["configs"]["4"]
    vd = device.gen3_device(24, 0.75, 0.05, 3)
    got = S.gpu_sharded_prime_ranks_emulated(vd, 24, k)
    del vd
    if len(got) != g["primes"]:
        from paper_2302_10083_b200 import device as D

        want = pkg.prime_ranks_from_values(D.gen3_device(24, 0.75, 0.05, 3).cpu().numpy())
        raise AssertionError(_block_diff(got, want, S.ShardPlan(24, k)))
    assert hashlib.sha256(got.astype("<i8").tobytes()).hexdigest()[:16] == g["ranks_sha256_prefix"]
    torch.cuda.empty_cache()


def _gpu_worker(rank, world, port, n, outdir):
    """One rank of a multi-process run sharing cuda:0: real GPU kernels, peer
    arenas opened through CUDA IPC and read in place (no kernel waits on
    another process; the level fences are host barriers)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2302_10083_b200 import _lib

        k = world.bit_length() - 1
        plan = S.ShardPlan(n, k)
        nl = n - k
        vals = torch.empty(1 << nl, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().dqmc_gen3_range_device(vals.data_ptr(), rank << nl, 1 << nl, 0.75, 0.05, 3,
                                                       torch.cuda.current_stream().cuda_stream))
        ops = S.GpuOps()
        comm = S.ProcessComm()
        for _ in range(2):  # the second call reuses the arenas and the open peer handles
            ops.reset_output()
            parts = S.run_schedule(plan, {rank: vals}, ops, comm)
        mine = {d: ops.out[s : s + c].cpu().numpy() for d, (s, c) in parts.items()}
        comm.close(ops)
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(mine, gathered, dst=0)
        if rank == 0:
            allp = {}
            for d in gathered:
                allp.update(d)
            np.save(os.path.join(outdir, "ranks.npy"), np.concatenate(S.ordered(allp)).astype(np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n", [(2, 18), (4, 19)])
def test_gpu_multiprocess_sharded(world, n, tmp_path, pkg):
    """The sharded data path with GpuOps on real kernels, ranks as processes,
    peer super-blocks read through CUDA IPC."""
    from paper_2302_10083_b200 import device

    mp.spawn(_gpu_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "ranks.npy")
    want = pkg.prime_ranks_from_values(device.gen3_device(n, 0.75, 0.05, 3).cpu().numpy())
    assert np.array_equal(got, want), _block_diff(got, want, S.ShardPlan(n, world.bit_length() - 1))


@pytest.mark.gpu
def test_bench_torchrun_two_ranks_gloo(tmp_path, pkg):
    """bench.py under torch.distributed.run (N=2) through the sharded path, gloo
    backend so both ranks can share this run's single GPU (peer reads over
    CUDA IPC)."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DQMC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1", "--nvars", "18"]
    r = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    from paper_2302_10083_b200 import device

    want = len(pkg.prime_ranks_from_values(device.gen3_device(18, 0.75, 0.05, 3).cpu().numpy()))
    assert line["n_gpus"] == 2 and line["config"]["primes"] == want and line["value"] > 0
    assert line["scaling"] == "strong" and line["e2e"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 2])
def test_gpu_emulated_n25_equals_single_gpu(k, pkg):
    """n = 25 (111.6 GB, the largest state one B200 holds; above every size the
    CPU reference runs): the 2^k-rank schedule and the single-GPU engine agree
    on every rank (north_star: 1-GPU and k-GPU runs bit-exact at larger n)."""
    from paper_2302_10083_b200 import _lib, device

    n = 25
    vd = device.gen3_device(n, 0.75, 0.05, 3)
    r, cnt = device.dense_prime_ranks_device(vd, n)
    want = r.cpu().numpy()
    del r
    _lib.load().dqmc_release()
    torch.cuda.empty_cache()
    got = S.gpu_sharded_prime_ranks_emulated(vd, n, k)
    torch.cuda.empty_cache()
    assert len(got) == cnt and np.array_equal(got, want)
