"""BASELINE.json workloads as device-side generators.

Product-side definitions; the oracle restates the same generators on the CPU
(oracle/gen.py) and the tests compare the two byte for byte.

  1: n=10, p_on=.5,  p_dc=0,   seed 0   (= random_function(10, .5, 0))
  2: n=16, p_on=.90, p_dc=.05, seed 1
  3: n=20, S-box complement, seed 2    (v = 0 iff y = P(x), x/y the low/high 10 bits)
  4: n=24, p_on=.75, p_dc=.05, seed 3   (the bench workload)
  5: n=27, p_on=.99, p_dc=0,   seed 4   (1.0 TB state: sharded only)
"""

from __future__ import annotations

import numpy as np

from . import _lib

CONFIGS = {
    1: dict(n=10, kind="gen3", p_on=0.5, p_dc=0.0, seed=0),
    2: dict(n=16, kind="gen3", p_on=0.90, p_dc=0.05, seed=1),
    3: dict(n=20, kind="sbox", seed=2),
    4: dict(n=24, kind="gen3", p_on=0.75, p_dc=0.05, seed=3),
    5: dict(n=27, kind="gen3", p_on=0.99, p_dc=0.0, seed=4),
}


def config_values_host(cfg: int, n: int | None = None) -> np.ndarray:
    """uint8 values (0 off, 1 on, 2 dc) of a BASELINE config, generated on the
    GPU and copied to the host; n overrides the size (same distribution)."""
    if cfg not in CONFIGS:
        raise ValueError(f"unknown config {cfg}; expected one of {sorted(CONFIGS)}")
    c = CONFIGS[cfg]
    nn = c["n"] if n is None else int(n)
    L = _lib.load()
    if c["kind"] == "sbox":
        if nn != 20:
            raise ValueError("the S-box config is defined at n=20 only")
        out = np.empty(1 << 20, dtype=np.uint8)
        _lib.check(L.dqmc_gen_sbox_host(out.ctypes.data, int(c["seed"])))
        return out
    if not 1 <= nn <= 31:
        raise ValueError(f"n must be in 1..31, got {nn}")
    out = np.empty(1 << nn, dtype=np.uint8)
    _lib.check(L.dqmc_gen3_host(out.ctypes.data, nn, float(c["p_on"]), float(c["p_dc"]), int(c["seed"])))
    return out


def config_values_device(cfg: int, n: int | None = None, device: int = 0):
    """The same values as a uint8 CUDA tensor (generated in place)."""
    import torch

    if cfg not in CONFIGS:
        raise ValueError(f"unknown config {cfg}; expected one of {sorted(CONFIGS)}")
    c = CONFIGS[cfg]
    nn = c["n"] if n is None else int(n)
    if c["kind"] == "sbox":
        if nn != 20:
            raise ValueError("the S-box config is defined at n=20 only")
        out = torch.empty(1 << 20, dtype=torch.uint8, device=f"cuda:{device}")
        stream = torch.cuda.current_stream(out.device).cuda_stream
        _lib.check(_lib.load().dqmc_gen_sbox_device(out.data_ptr(), int(c["seed"]), stream))
        return out
    from .device import gen3_device

    return gen3_device(nn, c["p_on"], c["p_dc"], c["seed"], device=device)
