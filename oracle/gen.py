"""Seeded synthetic truth tables for the BASELINE configs (CPU, numpy).

TEST INFRASTRUCTURE ONLY. This module is part of the oracle: it is imported by
tests/, bench.py's CPU-baseline leg and __graft_entry__.smoke() as the checker.
The product path generates inputs on the GPU (paper_2302_10083_b200.gen) and is
checked against this file.

Restates the reference's frozen counter-based generator:
  splitmix64 output mix            -> ttio.py:331-338 (_mix)
  x -> mix(seed + (x+1)*GAMMA)     -> ttio.py:341-343 (_point_values)
  include iff (u >> 11) < floor(density * 2^53)
                                   -> ttio.py:365-374 (random_function)
and the survey's three-way / S-box extensions of it (SURVEY.md §8(d),
Appendix A "Generators used"):
  gen3(n, p_on, p_dc, seed): v = 2 where u53 < int((p_on+p_dc)*2^53),
                             then v = 1 where u53 < int(p_on*2^53), else 0
  sbox_complement(seed):     perm = stable argsort of _point_values(0,1024,seed);
                             v = 1 everywhere except v[x | perm[x] << 10] = 0
Don't-care semantics: the function handed to the engine is
on ∪ dc, i.e. TruthTable.from_bools(n, v != 0) (ternary.py:210-218).
"""

from __future__ import annotations

import numpy as np

U = np.uint64
GAMMA = U(0x9E3779B97F4A7C15)
_CHUNK = 1 << 22


def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (ttio.py:331-338)."""
    x = x.copy()
    x ^= x >> U(30)
    x *= U(0xBF58476D1CE4E5B9)
    x ^= x >> U(27)
    x *= U(0x94D049BB133111EB)
    x ^= x >> U(31)
    return x


def point_values(lo: int, hi: int, seed: int) -> np.ndarray:
    """Generator value of points lo..hi-1 (ttio.py:341-343)."""
    x = np.arange(lo, hi, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(U(seed & ((1 << 64) - 1)) + (x + U(1)) * GAMMA)


def threshold53(p: float) -> int:
    return int(p * (1 << 53))


def gen3(n: int, p_on: float, p_dc: float, seed: int) -> np.ndarray:
    """uint8 values in {0 off, 1 on, 2 don't-care}, one per point x."""
    size = 1 << n
    out = np.empty(size, dtype=np.uint8)
    t_on = U(threshold53(p_on))
    t_any = U(threshold53(p_on + p_dc))  # float64 sum, as SURVEY §8(d)
    for lo in range(0, size, _CHUNK):
        hi = min(size, lo + _CHUNK)
        u = point_values(lo, hi, seed) >> U(11)
        v = np.zeros(hi - lo, dtype=np.uint8)
        v[u < t_any] = 2
        v[u < t_on] = 1
        out[lo:hi] = v
    return out


def sbox_complement(seed: int = 2) -> np.ndarray:
    """n=20 CNF case: f(x||y) = 0 iff y = P(x), P a seeded bijection on 10 bits."""
    perm = np.argsort(point_values(0, 1024, seed), kind="stable").astype(np.int64)
    v = np.ones(1 << 20, dtype=np.uint8)
    x = np.arange(1024, dtype=np.int64)
    v[x | (perm << 10)] = 0
    return v


def values_to_words(values: np.ndarray) -> np.ndarray:
    """on ∪ dc bitmap as little-endian uint64 words, TruthTable layout
    (ternary.py:187-196, 210-218): bit x of the stream is f(x)."""
    vals = np.asarray(values) != 0
    packed = np.packbits(vals, bitorder="little")
    packed = np.pad(packed, (0, (-len(packed)) % 8))
    return packed.view(np.uint64).copy()


def random_words(n: int, density: float, seed: int) -> np.ndarray:
    """TruthTable words of random_function(n, density, seed) (ttio.py:346-378)."""
    return values_to_words(gen3(n, density, 0.0, seed))


# BASELINE.json configs, restated
CONFIGS = {
    1: dict(n=10, kind="gen3", p_on=0.5, p_dc=0.0, seed=0),
    2: dict(n=16, kind="gen3", p_on=0.90, p_dc=0.05, seed=1),
    3: dict(n=20, kind="sbox", seed=2),
    4: dict(n=24, kind="gen3", p_on=0.75, p_dc=0.05, seed=3),
    5: dict(n=27, kind="gen3", p_on=0.99, p_dc=0.0, seed=4),
}


def config_values(cfg: int | dict, n: int | None = None) -> np.ndarray:
    """uint8 values of a BASELINE config; n overrides the size (same distribution)."""
    c = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    nn = c["n"] if n is None else n
    if c["kind"] == "sbox":
        if nn != 20:
            raise ValueError("the S-box config is defined at n=20 only")
        return sbox_complement(c["seed"])
    return gen3(nn, c["p_on"], c["p_dc"], c["seed"])
