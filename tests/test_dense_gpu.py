"""Parity of the B200 engine (libdqmc.so through the C ABI) with the oracle.

Bar: bit-exact int64 rank arrays. Small sizes are compared against the
committed reference goldens and the C oracle; n=24 (BASELINE config 4) is
pinned by the reference's recorded count and rank hash, plus sortedness and a
sampled independent implicant/maximality check.
"""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rsha(r):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(r, dtype="<i8")).tobytes()).hexdigest()


def tt_of(pkg, gen_mod, n, d, s):
    return pkg.TruthTable(n, gen_mod.random_words(n, d, s))


class TestKnownAnswers:
    def test_maj3_and_frozen(self, pkg, golden):
        maj3 = pkg.TruthTable.from_indices(3, [3, 5, 6, 7])
        assert pkg.dense_prime_ranks(maj3).tolist() == [14, 16, 22]
        assert pkg.find_primes_dense(maj3) == {"*11", "1*1", "11*"}
        assert pkg.dense_prime_ranks(pkg.TruthTable.from_indices(5, [12, 14])).tolist() == [42]
        assert pkg.find_primes_dense(pkg.TruthTable.from_indices(5, [0b01100, 0b01110])) == {"0*110"}
        assert pkg.find_primes_dense(pkg.TruthTable.from_indices(6, [0b101001])) == {"100101"}
        bits = golden["known"]["cli_order_bits"]
        tt = pkg.TruthTable.from_bools(4, np.array([c == "1" for c in bits]))
        assert pkg.dense_prime_ranks(tt).tolist() == golden["known"]["cli_order_ranks"]

    def test_constant_and_empty(self, pkg):
        for n in range(1, 16):
            r = pkg.dense_prime_ranks(pkg.TruthTable.full(n))
            assert r.tolist() == [3**n - 1], n
            e = pkg.dense_prime_ranks(pkg.TruthTable.empty(n))
            assert e.dtype == np.int64 and e.shape == (0,), n

    def test_extract_equals_support_for_isolated_points(self, pkg):
        # points pairwise at Hamming distance >= 2 are their own primes
        tt = pkg.TruthTable.from_indices(4, [0, 5, 9, 14])
        assert pkg.find_primes_dense(tt) == {"0000", "1010", "1001", "0111"}


class TestSweeps:
    def test_acceptance_sweep_c1(self, pkg, golden, gen_mod):
        for n, d, s, cnt, h16 in golden["sweep_c1"]:
            r = pkg.dense_prime_ranks(tt_of(pkg, gen_mod, n, d, s))
            assert r.dtype == np.int64 and len(r) == cnt and rsha(r)[:16] == h16, (n, d, s)

    def test_configs_1_to_3(self, pkg, golden, gen_mod):
        for c in ("1", "2", "3"):
            g = golden["configs"][c]
            v = gen_mod.config_values(int(c))
            r = pkg.prime_ranks_from_values(v)
            assert len(r) == g["primes"] and rsha(r) == g["ranks_sha256"], c
            r2 = pkg.dense_prime_ranks(pkg.TruthTable(g["n"], gen_mod.values_to_words(v)))
            assert np.array_equal(r, r2)

    def test_readme_and_dc(self, pkg, golden, gen_mod):
        for e in golden["readme"]:
            r = pkg.dense_prime_ranks(tt_of(pkg, gen_mod, e["n"], e["density"], e["seed"]))
            assert len(r) == e["primes"] and rsha(r) == e["ranks_sha256"]
        for e in golden["dc_cases"]:
            r = pkg.prime_ranks_from_values(gen_mod.gen3(e["n"], e["p_on"], e["p_dc"], e["seed"]))
            assert len(r) == e["primes"] and rsha(r) == e["ranks_sha256"]

    @pytest.mark.parametrize("n", list(range(11, 21)))
    def test_vs_oracle(self, pkg, oracle_mod, gen_mod, n):
        for d in (0.0, 0.3, 0.7, 0.95, 1.0):
            w = gen_mod.random_words(n, d, n)
            got = pkg.dense_prime_ranks(pkg.TruthTable(n, w))
            want = oracle_mod.dense_prime_ranks(w, n)
            assert np.array_equal(got, want), (n, d)

    @pytest.mark.parametrize(
        "n,p_on,p_dc",
        [(21, 0.75, 0.05), (22, 0.9, 0.05), pytest.param(23, 0.6, 0.1, marks=pytest.mark.slow)],
    )
    def test_vs_oracle_large(self, pkg, oracle_mod, gen_mod, n, p_on, p_dc):
        # n=21/22/23: groups (5,4)/(5,5)/(6,5): 3- and 8-column tiles in the strided passes
        v = gen_mod.gen3(n, p_on, p_dc, 3)
        got = pkg.prime_ranks_from_values(v)
        want = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), n)
        assert np.array_equal(got, want)


class TestBitmap:
    @pytest.mark.parametrize("n", [5, 6, 9, 12, 13, 15, 17, 19])
    def test_final_bitmap_equals_reference_state(self, pkg, oracle_mod, gen_mod, n):
        w = gen_mod.random_words(n, 0.7, 5)
        st = oracle_mod.OracleState(w, n, 5)
        st.run_merge_reduce()
        got = pkg.prime_bitmap(pkg.TruthTable(n, w))
        assert np.array_equal(got, st.words)


class TestContract:
    def test_split_and_optimized_accepted(self, pkg, gen_mod):
        tt = tt_of(pkg, gen_mod, 9, 0.5, 21)
        base = pkg.dense_prime_ranks(tt)
        for h in range(1, 10):
            assert np.array_equal(pkg.dense_prime_ranks(tt, h=h), base)
            assert np.array_equal(pkg.dense_prime_ranks(tt, h=h, optimized=False), base)

    def test_mem_cap_exact(self, pkg):
        tt = pkg.TruthTable.empty(12)
        need = pkg.state_bytes(12, 5)
        with pytest.raises(pkg.ResourceLimitError) as exc:
            pkg.dense_prime_ranks(tt, h=5, mem_cap=need - 1)
        assert str(need) in str(exc.value) and "bytes" in str(exc.value)
        pkg.dense_prime_ranks(tt, h=5, mem_cap=need)  # exactly at the cap is fine
        with pytest.raises(pkg.ResourceLimitError):
            pkg.run_engine("dense", pkg.TruthTable.full(14), mem_cap=1000)

    def test_run_engine_and_count(self, pkg, gen_mod):
        tt = tt_of(pkg, gen_mod, 16, 0.5, 42)
        r = pkg.run_engine("dense", tt)
        assert len(r) == 68460  # pkg/README.md:54-55
        assert pkg.count_primes(tt) == 68460

    def test_repeated_calls_stable(self, pkg, gen_mod):
        outs = [pkg.dense_prime_ranks(tt_of(pkg, gen_mod, 18, 0.8, 1)) for _ in range(3)]
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
        small = pkg.dense_prime_ranks(tt_of(pkg, gen_mod, 7, 0.5, 2))
        again = pkg.dense_prime_ranks(tt_of(pkg, gen_mod, 18, 0.8, 1))
        assert np.array_equal(outs[0], again) and len(small) > 0


class TestPipelinedHostPath:
    @pytest.mark.parametrize("n", [13, 17, 20, 23])
    def test_pipelined_equals_plain(self, pkg, oracle_mod, gen_mod, n):
        """The host API pipelines the final stage (chunked, copied out over
        PCIe while the next chunk computes) once it has a size hint of at
        least 4M ranks (n = 20, 23 here; n = 13, 17 stay on the plain path).
        n = 23 runs the piece-major plan."""
        from paper_2302_10083_b200 import _lib

        _lib.load().dqmc_release()  # no size hint: the first call takes the plain path
        v = gen_mod.gen3(n, 0.8, 0.05, 11)
        want = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), n)
        first = pkg.prime_ranks_from_values(v)  # plain; sets the hint
        second = pkg.prime_ranks_from_values(v)  # pipelined
        assert np.array_equal(first, want) and np.array_equal(second, want)
        # a larger output than the hint (grow path): denser table, same n
        v2 = gen_mod.gen3(n, 0.95, 0.0, 12)
        got = pkg.prime_ranks_from_values(v2)
        assert np.array_equal(got, oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v2), n))


class TestDevice:
    def test_gen3_device_matches_oracle(self, pkg, gen_mod):
        from paper_2302_10083_b200 import device

        for n, pon, pdc, s in ((16, 0.9, 0.05, 1), (20, 0.75, 0.05, 3), (12, 0.5, 0.0, 0)):
            v = device.gen3_device(n, pon, pdc, s).cpu().numpy()
            assert np.array_equal(v, gen_mod.gen3(n, pon, pdc, s))

    def test_device_entry_point(self, pkg, golden, gen_mod):
        import torch

        from paper_2302_10083_b200 import device

        g = golden["configs"]["2"]
        v = device.gen3_device(16, 0.90, 0.05, 1)
        r, cnt = device.dense_prime_ranks_device(v, 16)
        assert cnt == g["primes"] and rsha(r.cpu().numpy()) == g["ranks_sha256"]
        words = torch.from_numpy(gen_mod.values_to_words(gen_mod.config_values(2)).view(np.int64)).cuda()
        r2, cnt2 = device.dense_prime_ranks_device(words, 16)
        assert cnt2 == cnt and torch.equal(r, r2)
        _, c3 = device.dense_prime_ranks_device(v, 16, count_only=True)
        assert c3 == cnt


@pytest.mark.slow
class TestFullSize:
    def test_config4_n24(self, pkg, golden, oracle_mod, gen_mod):
        """BASELINE config 4 at full size: pinned by the reference's count and hash."""
        from paper_2302_10083_b200 import device

        g = golden["configs"]["4"]
        v = device.gen3_device(24, 0.75, 0.05, 3)
        r, cnt = device.dense_prime_ranks_device(v, 24)
        host = r.cpu().numpy()
        assert cnt == g["primes"]
        assert rsha(host)[:16] == g["ranks_sha256_prefix"]
        assert host[:3].tolist() == g["first"] and host[-3:].tolist() == g["last"]
        assert np.all(np.diff(host) > 0)  # unique, ascending
        # independent implicant + maximality check on sampled primes
        on = gen_mod.config_values(4) != 0
        rng = np.random.default_rng(7)
        for r0 in rng.choice(host, 200, replace=False):
            imp, mx = oracle_mod.is_prime_cube(int(r0), 24, on)
            assert imp and mx, int(r0)
        # and through the host API (same arrays)
        hr = pkg.prime_ranks_from_values(v.cpu().numpy())
        assert np.array_equal(hr, host)

    def test_config4_n24_reference_layout_plan(self, pkg, golden):
        """The bitmap-keeping plan (reference layout, no piece-major group 0,
        no sparse pass-C stores) counts the same primes as the default plan,
        and a default call after it (reusing the state buffer, whose stale
        contents pass D must mask) is still exact."""
        import ctypes

        import torch

        from paper_2302_10083_b200 import _lib, device

        g = golden["configs"]["4"]
        v = device.gen3_device(24, 0.75, 0.05, 3)
        cnt = ctypes.c_int64(0)
        _lib.check(_lib.load().dqmc_primes_device(v.data_ptr(), _lib.IN_U8, 24, None, 0, ctypes.byref(cnt),
                                                  _lib.FLAG_KEEP_BITMAP | _lib.FLAG_COUNT_ONLY,
                                                  torch.cuda.current_stream().cuda_stream))
        assert cnt.value == g["primes"]
        r, c2 = device.dense_prime_ranks_device(v, 24)
        assert c2 == g["primes"] and rsha(r.cpu().numpy())[:16] == g["ranks_sha256_prefix"]
        # a different table in between leaves different stale rows behind
        w = device.gen3_device(24, 0.5, 0.1, 9)
        device.dense_prime_ranks_device(w, 24, count_only=True)
        r, c3 = device.dense_prime_ranks_device(v, 24)
        assert c3 == g["primes"] and rsha(r.cpu().numpy())[:16] == g["ranks_sha256_prefix"]


    @pytest.mark.parametrize("p_on,p_dc", [(0.99, 0.0), (0.5, 0.1)])
    def test_n24_zero_skip_vs_reference_layout(self, pkg, p_on, p_dc):
        """The n=24 plan's zero-skip flags (pass C -> D items / E tiles) and the
        per-tile sparse/round final stage give the same rank list as the
        reference-layout plan (no flags, no piece-major group) at the config-5
        density and at a sparser one."""
        import ctypes

        import torch

        from paper_2302_10083_b200 import _lib, device

        v = device.gen3_device(24, p_on, p_dc, 4)
        r1, c1 = device.dense_prime_ranks_device(v, 24)
        out = torch.empty(c1 + 1024, dtype=torch.int64, device="cuda")
        cnt = ctypes.c_int64(0)
        _lib.check(_lib.load().dqmc_primes_device(v.data_ptr(), _lib.IN_U8, 24, out.data_ptr(), out.numel(),
                                                  ctypes.byref(cnt), _lib.FLAG_KEEP_BITMAP,
                                                  torch.cuda.current_stream().cuda_stream))
        assert cnt.value == c1
        assert bool(out[:c1].eq(r1).all())
        del out, r1
        torch.cuda.empty_cache()

    @pytest.mark.parametrize("p_on,p_dc,seed", [(0.75, 0.05, 3), (0.9, 0.0, 5), (0.99, 0.0, 4)])
    def test_n24_gather_finish_equals_pass_d(self, pkg, golden, p_on, p_dc, seed):
        """The two ways the n=24 plan finishes a state (include/dqmc.h,
        dqmc_gather_threshold): the lower group's REDUCE as its own read+write
        pass D, or gathered in the final stage from the unreduced state. Both
        forced on the same table, sparse to config-5 density: identical rank
        lists (config 4: the reference's count and hash), and the device-side
        choice reports what it did."""
        import ctypes

        from paper_2302_10083_b200 import _lib, device

        L = _lib.load()
        v = device.gen3_device(24, p_on, p_dc, seed)
        prev = L.dqmc_gather_threshold(-1)

        def info():
            nzb, tot, g = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
            _lib.check(L.dqmc_last_gather(ctypes.byref(nzb), ctypes.byref(tot), ctypes.byref(g)))
            return nzb.value, tot.value, g.value

        try:
            L.dqmc_gather_threshold(0)  # never: pass D
            r0, c0 = device.dense_prime_ranks_device(v, 24)
            nzb, tot, g = info()
            assert tot == 3**19 and 0 < nzb <= tot and g == 0
            L.dqmc_gather_threshold(1000)  # always: gather finish
            r1, c1 = device.dense_prime_ranks_device(v, 24)
            assert info() == (nzb, tot, 1)
            assert c1 == c0 and bool(r1.eq(r0).all())
            if (p_on, seed) == (0.75, 3):
                g4 = golden["configs"]["4"]
                assert c1 == g4["primes"] and rsha(r1.cpu().numpy())[:16] == g4["ranks_sha256_prefix"]
            del r0
            L.dqmc_gather_threshold(prev)  # the default choice follows the block density
            r2, c2 = device.dense_prime_ranks_device(v, 24)
            assert info()[2] == (1 if nzb * 1000 <= tot * prev else 0)
            assert c2 == c1 and bool(r2.eq(r1).all())
        finally:
            L.dqmc_gather_threshold(prev)


@pytest.mark.slow
class TestLargestSingleGpu:
    def test_n25_sampled(self, pkg, oracle_mod, gen_mod):
        """n=25: 3^20 = 3.5e9 blocks (> 2^31) and a 111.6 GB state on one GPU.
        No CPU reference fits, so: unique ascending int64 output, every sampled
        prime is an implicant with no implicant one-widening parent, and every
        sampled non-listed cube is not prime (independent checks, oracle.py:23-48)."""
        from paper_2302_10083_b200 import device

        n = 25
        v = device.gen3_device(n, 0.75, 0.05, 3)
        r, cnt = device.dense_prime_ranks_device(v, n)
        host = r.cpu().numpy()
        del r
        assert cnt == len(host) and cnt > 0 and np.all(np.diff(host) > 0)
        assert host[0] >= 0 and host[-1] < 3**n
        on = v.cpu().numpy() != 0
        rng = np.random.default_rng(25)
        for r0 in rng.choice(host, 150, replace=False):
            imp, mx = oracle_mod.is_prime_cube(int(r0), n, on)
            assert imp and mx, int(r0)
        # non-listed cubes: low-weight candidates near listed primes (the interesting ones)
        listed = set(host.tolist())
        checked = 0
        for r0 in rng.choice(host, 400, replace=False):
            s = oracle_mod.unrank(int(r0), n)
            i = int(rng.integers(0, n))
            for ch in "01*":
                t = s[:i] + ch + s[i + 1 :]
                rt = oracle_mod.rank(t)
                if rt in listed or t.count("*") > 8:
                    continue
                imp, mx = oracle_mod.is_prime_cube(rt, n, on)
                assert not (imp and mx), t
                checked += 1
        assert checked > 100


class TestAsyncAndGraph:
    """DQMC_FLAG_ASYNC (stream-ordered, no host sync) and CUDA-graph replay
    give the synchronous results bit for bit."""

    def test_async_matches_sync(self, pkg):
        import torch
        from paper_2302_10083_b200 import device

        for n, dtype in ((14, "u8"), (18, "u8"), (16, "words")):
            v = device.gen3_device(n, 0.6, 0.1, n)
            if dtype == "words":
                v = (v.view(-1, 8).ne(0).to(torch.int64) << torch.arange(8, device=v.device)).sum(1).to(torch.uint8)
                v = v.view(torch.int64) if v.numel() >= 8 else v
            ref, cnt = device.dense_prime_ranks_device(v, n)
            ref = ref.clone()
            out = torch.full((cnt + 100,), -7, dtype=torch.int64, device="cuda")
            c = torch.zeros(1, dtype=torch.int64, device="cuda")
            for _ in range(3):  # back-to-back, no host sync in between
                device.enqueue_prime_ranks(v, n, out, c)
            assert int(c.item()) == cnt
            assert torch.equal(out[:cnt], ref)

    def test_async_flags_short_output(self, pkg):
        import torch
        from paper_2302_10083_b200 import device

        v = device.gen3_device(16, 0.7, 0.0, 2)
        _, cnt = device.dense_prime_ranks_device(v, 16)
        out = torch.empty(cnt - 1, dtype=torch.int64, device="cuda")
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        device.enqueue_prime_ranks(v, 16, out, c)
        assert int(c.item()) == -(cnt + 1)

    def test_graph_replay_and_refill(self, pkg):
        import torch
        from paper_2302_10083_b200 import _lib, device

        n = 20
        v = device.gen3_device(n, 0.75, 0.05, 3)
        g = device.PrimesGraph(v, n)
        for _ in range(2):
            g.replay()
        ref, cnt = device.dense_prime_ranks_device(v, n)
        assert torch.equal(g.ranks(), ref)
        # refill the captured input in place with another function, replay
        _lib.check(_lib.load().dqmc_gen3_device(v.data_ptr(), n, 0.7, 0.05, 9,
                                                torch.cuda.current_stream().cuda_stream))
        g.replay()
        ref2, cnt2 = device.dense_prime_ranks_device(v, n)
        assert cnt2 != cnt
        if cnt2 <= g.out.numel():
            assert torch.equal(g.ranks(), ref2)
        else:
            with pytest.raises(RuntimeError):
                g.ranks()

    @pytest.mark.slow
    def test_graph_n24_finish_follows_the_data(self, pkg, golden):
        """One captured graph of the n=24 plan holds both ways to finish a
        state; which one runs is decided on the device at every replay
        (DESIGN.md 3c). Captured on a dense table (pass D), replayed on it,
        then on BASELINE config 4 refilled in place (gather finish): each
        replay equals the direct call / the reference's count and hash."""
        import ctypes

        import torch
        from paper_2302_10083_b200 import _lib, device

        L = _lib.load()

        def gathered():
            nzb, tot, g = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
            _lib.check(L.dqmc_last_gather(ctypes.byref(nzb), ctypes.byref(tot), ctypes.byref(g)))
            return g.value

        n = 24
        v = device.gen3_device(n, 0.99, 0.0, 4)
        ref, cnt = device.dense_prime_ranks_device(v, n)
        want = rsha(ref.cpu().numpy())
        del ref
        torch.cuda.empty_cache()
        g = device.PrimesGraph(v, n, headroom=1.0)
        g.replay()
        r = g.ranks()
        assert r.numel() == cnt and rsha(r.cpu().numpy()) == want
        assert gathered() == 0
        _lib.check(L.dqmc_gen3_device(v.data_ptr(), n, 0.75, 0.05, 3, torch.cuda.current_stream().cuda_stream))
        g.replay()
        r = g.ranks()
        g4 = golden["configs"]["4"]
        assert r.numel() == g4["primes"] and rsha(r.cpu().numpy())[:16] == g4["ranks_sha256_prefix"]
        assert gathered() == 1
        del g, r
        torch.cuda.empty_cache()


class TestJobStream:
    """dqmc_submit_* / dqmc_collect: three calls in flight, results identical to
    the synchronous call, edge cases of the job protocol."""

    def test_stream_matches_sync(self, pkg, gen_mod):
        tabs = [gen_mod.gen3(n, 0.7, 0.05, s) for n, s in ((16, 1), (16, 2), (16, 3), (18, 4), (18, 5), (16, 6))]
        want = [pkg.prime_ranks_from_values(t) for t in tabs]
        got = list(pkg.stream_prime_ranks(tabs))
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)

    def test_stream_n24_zero_skip_plan(self, pkg, golden):
        """The job stream at n = 24 (zero-skip flags, per-tile scratch slots,
        async count publication): config 4 twice, then the config-5 density (whose
        tiles overflow their slots), then config 4 again, each equal to the
        synchronous engine."""
        from paper_2302_10083_b200 import device

        g = golden["configs"]["4"]
        v4 = device.gen3_device(24, 0.75, 0.05, 3).cpu().numpy()
        v5 = device.gen3_device(24, 0.99, 0.0, 4)
        r5, c5 = device.dense_prime_ranks_device(v5, 24)
        h5 = rsha(r5.cpu().numpy())
        del r5
        got = list(pkg.stream_prime_ranks([v4, v4, v5.cpu().numpy(), v4]))
        for i in (0, 1, 3):
            assert len(got[i]) == g["primes"] and rsha(got[i])[:16] == g["ranks_sha256_prefix"]
        assert len(got[2]) == c5 and rsha(got[2]) == h5

    @pytest.mark.parametrize("threads", [0, 1, 5])
    def test_stream_packed_transfer(self, pkg, oracle_mod, gen_mod, threads):
        """Results of 4M+ ranks leave the device as 4-byte tile offsets and are
        widened to int64 by the host pool (n = 20 here: ~6M ranks): different
        tables back to back, any pool size, equal to the oracle."""
        from paper_2302_10083_b200 import _lib

        prev = _lib.load().dqmc_host_threads(threads)
        try:
            tabs = [gen_mod.gen3(20, 0.8, 0.05, s) for s in (21, 22, 23, 24)]
            got = list(pkg.stream_prime_ranks(tabs))
            for t, g in zip(tabs, got):
                assert g.dtype == np.int64 and len(g) >= 1 << 22
                assert np.array_equal(g, oracle_mod.dense_prime_ranks(gen_mod.values_to_words(t), 20))
        finally:
            _lib.load().dqmc_host_threads(prev)

    def test_truth_tables_and_repeat(self, pkg, gen_mod):
        t = pkg.TruthTable(17, gen_mod.random_words(17, 0.6, 9))
        want = pkg.dense_prime_ranks(t)
        for r in pkg.stream_prime_ranks([t] * 5):
            assert np.array_equal(r, want)

    def test_output_outgrows_the_hint(self, pkg, gen_mod):
        # a sparse table first (small hint), then a dense one of the same n:
        # the second job overflows its hinted output and is recomputed
        small = gen_mod.gen3(18, 0.05, 0.0, 1)
        big = gen_mod.gen3(18, 0.8, 0.1, 2)
        want = [pkg.prime_ranks_from_values(x) for x in (small, big, big)]
        got = list(pkg.stream_prime_ranks([small, small, big, big]))
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[0])
        assert np.array_equal(got[2], want[1]) and np.array_equal(got[3], want[2])

    def test_protocol_errors(self, pkg, gen_mod):
        t = gen_mod.gen3(12, 0.5, 0.0, 1)
        a, b, c = pkg.submit(t), pkg.submit(t), pkg.submit(t)
        with pytest.raises(ValueError):
            pkg.submit(t)  # a fourth outstanding job
        with pytest.raises(ValueError):
            b.result()  # out of order
        ra, rb, rc = a.result(), b.result(), c.result()
        assert np.array_equal(ra, rb) and np.array_equal(ra, rc) and np.array_equal(ra, pkg.prime_ranks_from_values(t))


class TestWorkspaceSafety:
    """Entry points sharing the engine workspace stay ordered, and captured
    graphs refuse to replay over reallocated buffers."""

    def test_graph_refuses_after_release(self, pkg):
        from paper_2302_10083_b200 import _lib, device

        v = device.gen3_device(16, 0.7, 0.05, 4)
        g = device.PrimesGraph(v, 16)
        g.replay()
        _lib.load().dqmc_release()
        with pytest.raises(RuntimeError, match="reallocated or released"):
            g.replay()

    def test_jobs_and_device_calls_interleaved(self, pkg, gen_mod):
        import torch
        from paper_2302_10083_b200 import device

        n = 18
        tabs = [gen_mod.gen3(n, 0.7, 0.05, s) for s in (11, 12, 13)]
        want = [pkg.prime_ranks_from_values(t) for t in tabs]
        dv = device.gen3_device(n, 0.6, 0.1, 21)
        dref, dcnt = device.dense_prime_ranks_device(dv, n)
        dref = dref.clone()
        jobs = [pkg.submit(t) for t in tabs]  # three jobs queued on the host-API stream
        out = torch.empty(dcnt + 64, dtype=torch.int64, device="cuda")
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):  # a caller-stream call while the jobs are in flight
            device.enqueue_prime_ranks(dv, n, out, c)
        got = [j.result() for j in jobs]
        s.synchronize()
        assert int(c.item()) == dcnt and torch.equal(out[:dcnt], dref)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)

    def test_bitmap_dropped_by_later_calls(self, pkg, gen_mod):
        t = pkg.TruthTable(16, gen_mod.random_words(16, 0.6, 3))
        bm = pkg.prime_bitmap(t)
        assert bm.any()
        # a host call on the pipelined path (count hint present) reuses the state
        pkg.dense_prime_ranks(t)
        pkg.dense_prime_ranks(t)
        with pytest.raises(ValueError, match="no bitmap held"):
            _download_only(pkg)


def _download_only(pkg):
    from paper_2302_10083_b200 import _lib

    out = np.zeros(pkg.state_bytes(16, 5) // 8, dtype=np.uint64)
    _lib.check(_lib.load().dqmc_bitmap_download(out.ctypes.data, out.nbytes))
