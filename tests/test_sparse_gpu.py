"""The sparse engine on the GPU (reference sparse.py:80-314)
against the reference's pins: the acceptance sweep c1 (dense = sparse =
oracle for n=1..10 x 7 densities x 20 seeds, golden counts and hashes from the
reference), README counts, config 1/2 goldens, known answers, agreement with
the dense engine at larger n, and the memory-cap refusal."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rsha(r):
    return hashlib.sha256(np.asarray(r, dtype="<i8").tobytes()).hexdigest()


def tt_of(pkg, gen_mod, n, density, seed):
    return pkg.TruthTable(n, gen_mod.random_words(n, density, seed))


def test_acceptance_sweep_c1(pkg, golden, gen_mod):
    for n, d, s, cnt, h16 in golden["sweep_c1"]:
        r = pkg.sparse_prime_ranks(tt_of(pkg, gen_mod, n, d, s))
        assert r.dtype == np.int64 and len(r) == cnt and rsha(r)[:16] == h16, (n, d, s)


def test_known_answers(pkg, golden):
    maj3 = pkg.TruthTable.from_indices(3, [3, 5, 6, 7])
    assert pkg.sparse_prime_ranks(maj3).tolist() == [14, 16, 22]
    assert pkg.find_primes_sparse(pkg.TruthTable.from_indices(5, [12, 14])) == {"0*110"}
    for n in range(1, 13):  # constant-1 -> the all-star cube (test_acceptance.py:84-90)
        assert pkg.find_primes_sparse(pkg.TruthTable.full(n)) == {"*" * n}
        e = pkg.sparse_prime_ranks(pkg.TruthTable.empty(n))
        assert e.dtype == np.int64 and e.shape == (0,)


def test_readme_and_configs(pkg, golden, gen_mod):
    for e in golden["readme"]:
        r = pkg.sparse_prime_ranks(tt_of(pkg, gen_mod, e["n"], e["density"], e["seed"]))
        assert len(r) == e["primes"] and rsha(r) == e["ranks_sha256"], e
    for c in ("1", "2"):
        g = golden["configs"][c]
        v = gen_mod.config_values(int(c))
        r = pkg.sparse_prime_ranks(pkg.TruthTable.from_values(g["n"], v))
        assert len(r) == g["primes"] and rsha(r) == g["ranks_sha256"], c


@pytest.mark.parametrize("n,density", [(12, 0.1), (14, 0.3), (16, 0.05), (18, 0.02), (17, 0.5)])
def test_sparse_equals_dense(pkg, gen_mod, n, density):
    tt = tt_of(pkg, gen_mod, n, density, n)
    assert np.array_equal(pkg.sparse_prime_ranks(tt), pkg.dense_prime_ranks(tt))
    assert np.array_equal(pkg.run_engine("sparse", tt), pkg.run_engine("dense", tt))


def test_mem_cap(pkg, gen_mod):
    tt = tt_of(pkg, gen_mod, 14, 0.5, 3)
    with pytest.raises(pkg.ResourceLimitError, match="bytes"):
        pkg.sparse_prime_ranks(tt, mem_cap=0)
    with pytest.raises(pkg.ResourceLimitError, match="sparse level table needs"):
        pkg.sparse_prime_ranks(tt, mem_cap=4096)  # level 0 alone needs 2^14 slots
    assert len(pkg.sparse_prime_ranks(tt, mem_cap=1 << 30)) == len(pkg.dense_prime_ranks(tt))
