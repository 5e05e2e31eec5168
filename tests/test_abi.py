"""C-ABI boundary checks that run without a GPU.

* libdqmc.so loads and exports every function include/dqmc.h declares;
* size helpers agree with the reference formulas (dense.py:56-63);
* argument validation and resource errors behave as the reference's
  (ValueError / ResourceLimitError naming the bytes) before any GPU use;
* with no CUDA device a compute call fails loudly — there is no CPU fallback.
"""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(REPO, "include", "dqmc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dqmc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(pkg):
    from paper_2302_10083_b200 import _lib

    L = _lib.load()
    declared = header_functions()
    assert declared, "no functions parsed from include/dqmc.h"
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_abi_version_and_sizes(pkg):
    from paper_2302_10083_b200 import _lib

    L = _lib.load()
    assert L.dqmc_abi_version() == 5
    for h in range(1, 10):
        assert L.dqmc_block_bits(h) == pkg.block_bits_for(h)
    for n in range(1, 28):
        for h in range(1, min(n, 8) + 1):
            assert L.dqmc_state_bytes(n, h) == 3 ** (n - h) * pkg.block_bits_for(h) // 8
    # tests/test_dense.py:72-84 pins
    assert pkg.block_bits_for(1) == 64 and pkg.block_bits_for(3) == 64
    assert pkg.block_bits_for(4) == 128 and pkg.block_bits_for(5) == 256
    assert pkg.state_bytes(3, 1) == 72 and pkg.state_bytes(20, 5) == 3**15 * 32


def test_gather_threshold_and_launch_count(pkg):
    """The tuning knob of the n=24 plan's finish (include/dqmc.h) is plain host
    state: set/query round trip, clamped to 0..1000, no device needed; nothing
    has run, so there is no gather report and no launch has been counted."""
    import ctypes

    from paper_2302_10083_b200 import _lib

    L = _lib.load()
    prev = L.dqmc_gather_threshold(-1)
    try:
        assert 0 <= prev <= 1000
        assert L.dqmc_gather_threshold(0) == prev
        assert L.dqmc_gather_threshold(5000) == 0
        assert L.dqmc_gather_threshold(-1) == 1000
    finally:
        L.dqmc_gather_threshold(prev)
    assert L.dqmc_gather_threshold(-1) == prev
    if not pkg_has_device():
        a, b, g = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
        assert L.dqmc_last_gather(ctypes.byref(a), ctypes.byref(b), ctypes.byref(g)) == _lib.DQMC_ERR_INVALID
        assert L.dqmc_launch_count() == 0


def pkg_has_device() -> bool:
    import torch

    return torch.cuda.is_available()


def test_plan_covers_every_axis(pkg):
    from paper_2302_10083_b200 import _lib

    for n in range(1, 28):
        p = _lib.plan(n)
        assert p["ne"] == max(n, 5) and p["H"] == p["ne"] - 5
        assert p["g"] + p["T"] == p["H"] and p["g"] <= 7
        assert sum(p["r"]) == p["T"] and all(0 < r <= 6 for r in p["r"][: p["m"]])
        a = p["g"]
        for k in range(p["m"]):
            assert p["a"][k] == a
            a += p["r"][k]
        masks = [p["ib_C"], p["ib_E"]] + p["ib_D"][: max(0, p["m"] - 1)]
        acc = 0
        for m in masks:
            assert acc & m == 0  # each in-block axis reduced exactly once
            acc |= m
        assert acc == 31
        assert p["rank_sub"] == (243 - 3**n if n < 5 else 0)


def test_validation_before_gpu(pkg):
    tt = pkg.TruthTable.empty(3)
    with pytest.raises(ValueError):
        pkg.dense_prime_ranks(tt, h=0)
    with pytest.raises(ValueError):
        pkg.dense_prime_ranks(tt, h=4)
    tt12 = pkg.TruthTable.empty(12)
    need = pkg.state_bytes(12, 5)
    with pytest.raises(pkg.ResourceLimitError) as exc:
        pkg.dense_prime_ranks(tt12, h=5, mem_cap=0)
    assert str(need) in str(exc.value) and "bytes" in str(exc.value)
    with pytest.raises(ValueError):
        pkg.TruthTable(3, np.zeros(2, dtype=np.uint64))
    with pytest.raises(ValueError):
        pkg.run_engine("fastest", tt)


def test_no_device_fails_loudly(pkg):
    from paper_2302_10083_b200 import _lib

    if _lib.load().dqmc_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    with pytest.raises(RuntimeError, match="CUDA device required"):
        pkg.dense_prime_ranks(pkg.TruthTable.full(4))
    res = _lib.DqmcResult()
    w = np.zeros(16, dtype=np.uint64)
    rc = _lib.load().dqmc_primes_tt(w.ctypes.data, 10, 0, 0, 0, ctypes.byref(res))
    assert rc == _lib.DQMC_ERR_NODEVICE


def test_ternary_helpers(pkg):
    assert pkg.rank("1*0**") == 223  # SPEC.md rank example
    assert pkg.unrank(223, 5) == "1*0**"
    assert pkg.index_to_rank(np.array([7]), 3).tolist() == [13]
    assert pkg.unrank_many(np.array([14, 16, 22]), 3) == ["*11", "1*1", "11*"]
    assert pkg.ranks_to_text(np.array([14]), 3, wildcard="-") == "-11\n"
    assert pkg.rank_weights(np.array([26, 0]), 3).tolist() == [3, 0]


def test_count_primes_cap_validated_like_load(pkg):
    # dense.py:358-364: a cap that cannot hold the state raises before any
    # allocation (0 and negative caps included), naming the bytes
    tt = pkg.TruthTable.full(12)
    for cap in (0, -5):
        with pytest.raises(pkg.ResourceLimitError, match=str(pkg.state_bytes(12, 5))):
            pkg.count_primes(tt, mem_cap=cap)


def test_sparse_cap_validated_before_the_device(pkg):
    # sparse.py:105-111: an explicit cap <= 0 cannot hold the level-0 table
    tt = pkg.TruthTable.full(10)
    with pytest.raises(pkg.ResourceLimitError, match="sparse level table needs 16384 bytes"):
        pkg.sparse_prime_ranks(tt, mem_cap=0)
    assert pkg.ENGINES == ("dense", "sparse")
    with pytest.raises(ValueError, match="oracle"):
        pkg.run_engine("oracle", tt)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_widen_host_matches_numpy(pkg, threads):
    """The host half of the packed rank transfer (csrc/dqmc_hostpack.cpp):
    rank = tile's first rank + 4-byte offset, every tile boundary, empty
    tiles, unaligned output and chunk-relative positions, any pool size."""
    from paper_2302_10083_b200 import _lib

    L = _lib.load()
    prev = L.dqmc_host_threads(threads)
    try:
        rng = np.random.default_rng(7 + threads)
        tile_cells, rank_add = 3**12, -162
        for ntiles, mean in ((1, 5), (50, 3), (3000, 40), (2000, 700)):
            cnt = rng.poisson(mean, ntiles).astype(np.int64)
            cnt[rng.random(ntiles) < 0.2] = 0  # zero tiles
            t0, add = 17, 12345  # a chunk in the middle of a call
            pos = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
            total = int(cnt.sum())
            end = add + total
            off = np.zeros(end + 5, dtype=np.uint32)
            off[add:end] = rng.integers(0, tile_cells, total, dtype=np.uint32)
            for shift in (0, 1, 3):  # output alignment relative to 64 bytes
                buf = np.full(end + 16, -7, dtype=np.int64)
                out = buf[shift:]
                L.dqmc_widen_host(off.ctypes.data, out.ctypes.data, pos.ctypes.data, add, end, t0, t0 + ntiles,
                                  tile_cells, rank_add)
                tile_of = np.repeat(np.arange(ntiles, dtype=np.int64), cnt)
                want = (t0 + tile_of) * tile_cells + rank_add + off[add:end].astype(np.int64)
                assert np.array_equal(out[add:end], want)
                assert np.all(out[:add] == -7) and np.all(out[end:] == -7)  # nothing outside the chunk
    finally:
        L.dqmc_host_threads(prev)
