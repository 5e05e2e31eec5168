"""Engine dispatch seam, mirroring run_engine (bench.py:94-108).

The reference has no plugin system: its operator API is run_engine's string
dispatch over ENGINES (bench.py:35). This module registers the B200 engines
under the same names: "dense" (the hot path) and "sparse" (the level walk,
SURVEY.md §8(f4)). "oracle" is the reference's definition-level checker and
stays out of scope, so asking for it is an error that names
the engine.
"""

from __future__ import annotations

import numpy as np

from .dense import dense_prime_ranks
from .sparse import sparse_prime_ranks

ENGINES = ("dense", "sparse")


def run_engine(engine: str, tt, h: int | None = None, optimized: bool = True, mem_cap: int | None = None) -> np.ndarray:
    """Prime implicant ranks from the named engine, ascending (bench.py:94-108)."""
    if engine == "dense":
        return dense_prime_ranks(tt, h=h, optimized=optimized, mem_cap=mem_cap)
    if engine == "sparse":  # h and optimized do not apply (bench.py:104-105)
        return sparse_prime_ranks(tt, mem_cap=mem_cap)
    raise ValueError(f"unknown engine {engine!r}; expected one of {', '.join(ENGINES)}")
