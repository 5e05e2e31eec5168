"""Engine dispatch seam, mirroring run_engine (bench.py:94-108).

The reference has no plugin system: its operator API is run_engine's string
dispatch over ENGINES (bench.py:35). This module registers the B200 engine
under the same name "dense" so callers of run_engine("dense", ...) get the
GPU path; "sparse" and "oracle" belong to the reference and are out of scope
here, so asking for them is an error that names the engine.
"""

from __future__ import annotations

import numpy as np

from .dense import dense_prime_ranks

ENGINES = ("dense",)


def run_engine(engine: str, tt, h: int | None = None, optimized: bool = True, mem_cap: int | None = None) -> np.ndarray:
    """Prime implicant ranks from the named engine, ascending (bench.py:94-108)."""
    if engine == "dense":
        return dense_prime_ranks(tt, h=h, optimized=optimized, mem_cap=mem_cap)
    raise ValueError(f"unknown engine {engine!r}; expected one of {', '.join(ENGINES)}")
