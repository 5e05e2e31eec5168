"""Top-k sharding: schedule logic, gloo multi-process runs on
CPU (world_size 2 and 4, 127.0.0.1), and the k-shard schedule on one GPU
compared bit-exactly with the single-GPU engine.

On CPU the per-block compute is done by the oracle (test infrastructure); the
code under test is the schedule + point-to-point exchange in
paper_2302_10083_b200.sharded, which is the same code the GPU path runs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_10083_b200 import sharded as S


class OracleOps:
    """CPU block ops for tests: oracle MERGE / REDUCE on h=5 blocks."""

    def __init__(self, nl):
        from oracle import oracle as O

        self.O = O
        self.nl = nl
        self.words = O.state_bytes(nl, 5) // 8

    def empty_block(self):
        return torch.empty(self.words, dtype=torch.int64)

    def sync(self):
        pass

    def merge(self, values, nl):
        from oracle import gen as G

        st = self.O.OracleState(G.values_to_words(values), nl, 5)
        st.run_pass(self.O.MERGE)
        return torch.from_numpy(st.words.view(np.int64).copy())

    def and_(self, a, b):
        return torch.bitwise_and(a, b)

    def or_(self, dst, src):
        return dst.bitwise_or_(src)

    def copy(self, src):
        return src.clone()

    def reduce_extract(self, block, nl, kill, offset):
        st = self.O.OracleState.from_words(block.numpy().view(np.uint64).copy(), nl, 5)
        st.run_pass(self.O.REDUCE)
        if kill is not None:
            st.words &= ~kill.numpy().view(np.uint64)
        return st.extract_ranks() + offset


class TestSchedule:
    @pytest.mark.parametrize("k", [1, 2, 3])
    def test_owner_map(self, k):
        own = S.owner_map(k)
        assert len(own) == 3**k
        for g in range(1 << k):
            assert own[S.binary_block(g, k)] == g
        for t, g in own.items():  # owner agrees with every fixed digit
            assert all(((g >> j) & 1) == d for j, d in enumerate(t) if d != 2)
        loads = np.bincount(list(own.values()), minlength=1 << k)
        assert loads.max() - loads.min() <= 1  # balanced to within one block

    @pytest.mark.parametrize("k", [1, 2, 3])
    def test_rounds_cover_every_star_block_once(self, k):
        seen = [t for jobs in S.star_rounds(k) for t, _, _ in jobs]
        stars = [t for t in S.all_blocks(k) if 2 in t]
        assert sorted(seen) == sorted(stars)
        done = {t for t in S.all_blocks(k) if 2 not in t}
        for jobs in S.star_rounds(k):  # children always computed in an earlier round
            for t, c0, c1 in jobs:
                assert c0 in done and c1 in done
            done |= {t for t, _, _ in jobs}

    def test_block_ranges_tile_the_rank_space(self):
        k, nl = 2, 6
        ranges = sorted((S.rho(t) * 3**nl, (S.rho(t) + 1) * 3**nl) for t in S.all_blocks(k))
        assert ranges[0][0] == 0 and ranges[-1][1] == 3 ** (nl + k)
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))

    @pytest.mark.parametrize("n,k", [(8, 1), (9, 2), (10, 3), (11, 2)])
    def test_emulated_cpu_matches_single_engine(self, n, k, oracle_mod, gen_mod):
        v = gen_mod.gen3(n, 0.7, 0.1, n)
        nl = n - k
        inputs = {g: v[g << nl : (g + 1) << nl] for g in range(1 << k)}
        parts = S.sharded_prime_ranks(inputs, n, k, OracleOps(nl), S.EmulatedComm(1 << k))
        got = S.concat_ranks({t: x for t, x in parts.items()})
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
    try:
        from oracle import gen as G

        k = world.bit_length() - 1
        nl = n - k
        v = G.gen3(n, 0.75, 0.05, seed)
        mine = v[rank << nl : (rank + 1) << nl]
        parts = S.sharded_prime_ranks({rank: mine}, n, k, OracleOps(nl), S.DistComm())
        gathered = [None] * world if rank == 0 else None
        dist.gather_object({t: np.asarray(x) for t, x in parts.items()}, gathered, dst=0)
        if rank == 0:
            allp = {}
            for d in gathered:
                allp.update(d)
            np.save(os.path.join(outdir, "ranks.npy"), S.concat_ranks(allp))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 10), (4, 12)])
def test_gloo_sharded_equals_single(world, n, tmp_path, oracle_mod, gen_mod):
    mp.spawn(_worker, args=(world, _free_port(), n, 3, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "ranks.npy")
    v = gen_mod.gen3(n, 0.75, 0.05, 3)
    want = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), n)
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(12, 1), (14, 2), (17, 3), (20, 2), (22, 3)])
def test_gpu_emulated_shards_bit_exact(n, k, pkg, gen_mod):
    from paper_2302_10083_b200 import device

    vd = device.gen3_device(n, 0.75, 0.05, 3)
    got = S.gpu_sharded_prime_ranks_emulated(vd, n, k)
    want = pkg.prime_ranks_from_values(vd.cpu().numpy())
    assert np.array_equal(got, want), _block_diff(got, want, n, k)


def _block_diff(got, want, n, k):
    nl = n - k
    out = [f"total got {len(got)} want {len(want)}"]
    for t in S.all_blocks(k):
        lo, hi = S.rho(t) * 3**nl, (S.rho(t) + 1) * 3**nl
        g, w = got[(got >= lo) & (got < hi)], want[(want >= lo) & (want < hi)]
        if not np.array_equal(g, w):
            out.append(f"block {t}: got {len(g)} want {len(w)} missing {len(np.setdiff1d(w, g))} extra {len(np.setdiff1d(g, w))}")
    return "; ".join(out)


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_emulated_config4_k3(pkg, golden):
    """n=24 on 8 emulated shards == the reference's pins for config 4."""
    import hashlib

    from paper_2302_10083_b200 import device

    g = golden["configs"]["4"]
    vd = device.gen3_device(24, 0.75, 0.05, 3)
    got = S.gpu_sharded_prime_ranks_emulated(vd, 24, 3)
    if len(got) != g["primes"]:
        want = pkg.prime_ranks_from_values(vd.cpu().numpy())
        raise AssertionError(_block_diff(got, want, 24, 3))
    assert hashlib.sha256(got.astype("<i8").tobytes()).hexdigest()[:16] == g["ranks_sha256_prefix"]


def _gpu_worker(rank, world, port, n, outdir, transport="staging"):
    """One rank of a multi-process run sharing cuda:0: real GPU block ops; the
    exchange is host-staged gloo send/recv, or P2P reads of the peers' blocks
    through CUDA IPC (no kernel waits on another process either way)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2302_10083_b200 import _lib

        k = world.bit_length() - 1
        nl = n - k
        vals = torch.empty(1 << nl, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().dqmc_gen3_range_device(vals.data_ptr(), rank << nl, 1 << nl, 0.75, 0.05, 3,
                                                       torch.cuda.current_stream().cuda_stream))
        comm = S.IpcComm() if transport == "p2p" else S.DistComm(staging=True)
        parts = S.sharded_prime_ranks({rank: vals}, n, k, S.GpuOps(nl), comm)
        gathered = [None] * world if rank == 0 else None
        dist.gather_object({t: v.cpu().numpy() for t, v in parts.items()}, gathered, dst=0)
        if rank == 0:
            allp = {}
            for d in gathered:
                allp.update(d)
            np.save(os.path.join(outdir, "ranks.npy"), S.concat_ranks(allp))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["staging", "p2p"])
@pytest.mark.parametrize("world,n", [(2, 18), (4, 19)])
def test_gpu_multiprocess_sharded(world, n, transport, tmp_path, pkg):
    """The sharded data path with GpuOps on real kernels, ranks as processes,
    over both transports (send/recv with host staging; CUDA-IPC peer reads)."""
    from paper_2302_10083_b200 import device

    mp.spawn(_gpu_worker, args=(world, _free_port(), n, str(tmp_path), transport), nprocs=world, join=True)
    got = np.load(tmp_path / "ranks.npy")
    want = pkg.prime_ranks_from_values(device.gen3_device(n, 0.75, 0.05, 3).cpu().numpy())
    assert np.array_equal(got, want), _block_diff(got, want, n, world.bit_length() - 1)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["sendrecv", "p2p"])
def test_bench_torchrun_two_ranks_gloo(transport, tmp_path, pkg):
    """bench.py under torch.distributed.run (N=2) through the sharded path, gloo
    backend (host-staged send/recv, or CUDA-IPC peer reads) so both ranks can
    share this run's single GPU."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DQMC_DIST_BACKEND="gloo", DQMC_DIST_TRANSPORT=transport)
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
