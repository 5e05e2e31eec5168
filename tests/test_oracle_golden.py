"""Pin the CPU oracle (and the restated generators) to the reference's goldens.

Golden vectors come from tests/golden/golden.json, produced by running the
reference package itself (tests/golden/make_golden.py) plus the survey's
recorded n=24 reference run. Nothing here needs a GPU.
"""

import hashlib
import os

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rsha(r):
    return sha(np.asarray(r, dtype="<i8"))


class TestGenerators:
    def test_configs_tt_hash(self, golden, gen_mod):
        for c in ("1", "2", "3"):
            g = golden["configs"][c]
            v = gen_mod.config_values(int(c))
            assert sha(v) == g["tt_sha256"], c
            assert (int((v == 1).sum()), int((v == 2).sum()), int((v == 0).sum())) == (g["on"], g["dc"], g["off"])

    def test_random_function_words(self, golden, gen_mod):
        for e in golden["generator"]:
            assert sha(gen_mod.random_words(e["n"], e["density"], e["seed"])) == e["words_sha256"]

    def test_readme_gen_bits(self, gen_mod):
        # pkg/README.md:136-137: gen (5, .3, 7) -> bits
        w = gen_mod.random_words(5, 0.3, 7)
        bits = "".join(str((int(w[0]) >> i) & 1) for i in range(32))
        assert bits == "01000100101000000000010000100001"

    def test_config4_tt_prefix(self, golden, gen_mod):
        g = golden["configs"]["4"]
        v = gen_mod.config_values(4)
        assert sha(v)[:16] == g["tt_sha256_prefix"]
        assert (int((v == 1).sum()), int((v == 2).sum()), int((v == 0).sum())) == (g["on"], g["dc"], g["off"])


class TestDenseOracle:
    def test_configs_1_to_3(self, golden, oracle_mod, gen_mod):
        for c in ("1", "2", "3"):
            g = golden["configs"][c]
            v = gen_mod.config_values(int(c))
            r = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), g["n"])
            assert len(r) == g["primes"] and rsha(r) == g["ranks_sha256"], c
            assert r[:5].tolist() == g["first"] and r[-5:].tolist() == g["last"]
        w1 = gen_mod.values_to_words(gen_mod.config_values(1))
        assert golden["configs"]["1"]["ranks"] == oracle_mod.dense_prime_ranks(w1, 10).tolist()

    def test_acceptance_sweep_c1(self, golden, oracle_mod, gen_mod):
        # test_acceptance.py:56-72: n 1..10 x 7 densities x 20 seeds
        for n, d, s, cnt, h16 in golden["sweep_c1"]:
            r = oracle_mod.dense_prime_ranks(gen_mod.random_words(n, d, s), n)
            assert len(r) == cnt and rsha(r)[:16] == h16, (n, d, s)

    def test_readme_and_known(self, golden, oracle_mod, gen_mod):
        for e in golden["readme"]:
            r = oracle_mod.dense_prime_ranks(gen_mod.random_words(e["n"], e["density"], e["seed"]), e["n"])
            assert len(r) == e["primes"] and rsha(r) == e["ranks_sha256"]
        k = golden["known"]
        maj3 = np.array([0b11101000], dtype=np.uint64)  # support {3,5,6,7}
        assert oracle_mod.dense_prime_ranks(maj3, 3).tolist() == k["maj3"] == [14, 16, 22]
        w = np.zeros(1, dtype=np.uint64)
        w[0] = (1 << 12) | (1 << 14)
        assert oracle_mod.dense_prime_ranks(w, 5).tolist() == k["n5_12_14"] == [42]

    def test_dc_cases(self, golden, oracle_mod, gen_mod):
        for e in golden["dc_cases"]:
            v = gen_mod.gen3(e["n"], e["p_on"], e["p_dc"], e["seed"])
            assert sha(v) == e["tt_sha256"]
            r = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(v), e["n"])
            assert len(r) == e["primes"] and rsha(r) == e["ranks_sha256"]

    def test_state_layout_pins(self, golden, oracle_mod, gen_mod):
        # DenseState.words byte-for-byte after load / MERGE / REDUCE (dense.py:296-337)
        for e in golden["states"]:
            st = oracle_mod.OracleState(gen_mod.random_words(e["n"], e["density"], e["seed"]), e["n"], e["h"])
            assert sha(st.words) == e["loaded"]
            st.run_pass(oracle_mod.MERGE)
            assert sha(st.words) == e["merged"]
            st.run_pass(oracle_mod.REDUCE)
            assert sha(st.words) == e["reduced"]

    def test_split_and_unroll_invariance(self, oracle_mod, gen_mod):
        w = gen_mod.random_words(9, 0.5, 21)
        base = oracle_mod.dense_prime_ranks(w, 9, 5)
        for h in range(1, 10):
            assert np.array_equal(oracle_mod.dense_prime_ranks(w, 9, h), base), h
            assert np.array_equal(oracle_mod.dense_prime_ranks(w, 9, h, optimized=False), base), h

    def test_bad_split(self, oracle_mod):
        with pytest.raises(ValueError):
            oracle_mod.dense_prime_ranks(np.zeros(1, dtype=np.uint64), 3, 4)

    @pytest.mark.slow
    @pytest.mark.skipif(not os.environ.get("DQMC_BIG_ORACLE"), reason="needs ~40 GB host RAM; set DQMC_BIG_ORACLE=1")
    def test_config4_full(self, golden, oracle_mod, gen_mod):
        g = golden["configs"]["4"]
        r = oracle_mod.dense_prime_ranks(gen_mod.values_to_words(gen_mod.config_values(4)), 24)
        assert len(r) == g["primes"] and rsha(r)[:16] == g["ranks_sha256_prefix"]
        assert r[:3].tolist() == g["first"] and r[-3:].tolist() == g["last"]


class TestDefinitionOracle:
    def test_matches_dense_oracle(self, oracle_mod, gen_mod):
        for n in range(1, 11):
            for d in (0.2, 0.5, 0.8, 1.0):
                for s in range(3):
                    w = gen_mod.random_words(n, d, s)
                    assert np.array_equal(oracle_mod.definition_prime_ranks(w, n), oracle_mod.dense_prime_ranks(w, n))

    def test_naive_small(self, oracle_mod, gen_mod):
        for n in range(1, 6):
            for s in range(3):
                w = gen_mod.random_words(n, 0.5, s)
                got = set(oracle_mod.unrank(int(r), n) for r in oracle_mod.definition_prime_ranks(w, n))
                assert got == oracle_mod.naive_primes(w, n)

    def test_prime_cube_checker(self, oracle_mod, gen_mod):
        w = gen_mod.random_words(8, 0.6, 1)
        on = oracle_mod.tt_bools(w, 8)
        primes = set(oracle_mod.dense_prime_ranks(w, 8).tolist())
        rng = np.random.default_rng(0)
        for r in rng.integers(0, 3**8, 300):
            imp, mx = oracle_mod.is_prime_cube(int(r), 8, on)
            assert (imp and mx) == (int(r) in primes)
