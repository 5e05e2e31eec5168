"""Command-line front end of the GPU engine.

Mirrors the dense-path subset of the reference CLI
(/root/reference/pkg/src/implicants/cli.py:1-337):

  primes  all prime implicants of one function, one string per line,
          wildcard count descending then rank ascending (cli.py:131-138);
          the ordering runs on the GPU (dqmc_order_by_weight)
  verify  run independent GPU engines on the same input and compare
          (cli.py:141-177): "dense" = the fused multi-pass plan
          (dense_prime_ranks), "sparse" = the level walk over device hash
          sets (sparse_prime_ranks, csrc/dqmc_sparse.cu), "state" = the
          per-dimension device DenseState (the reference's layer structure,
          csrc/dqmc_state.cu)
  bench   timed runs over sweeps of generated inputs, JSONL reports with the
          reference's BenchReport fields (bench.py:38-56)

Inputs: --input PATH in the 'bits' text format (one '0'/'1' per point, index 0
first, whitespace ignored; ttio.py format "bits") or generated on the device
from --n/--density/--seed with the reference's frozen generator (ttio.py:331-378),
optionally with --dc (three-valued table, don't-care = on), or
--config K for a BASELINE.json workload (configs.py).
Other text formats (hex/minterms/pla) are out of scope.

Exit codes (cli.py:320-333): 0 success, 1 bad input or usage, 2 resource
limit exceeded, 3 verify found disagreeing engines.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

from . import _lib
from .dense import dense_prime_ranks, prime_ranks_from_values
from .sparse import sparse_prime_ranks
from . import errors
from .ternary import TruthTable, ranks_to_text

_CORRUPT_ENV = "IMPLICANTS_VERIFY_CORRUPT"  # same fault-injection hook as cli.py:40-42
ENGINES = ("dense", "sparse", "state")


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        self.exit(1, f"{self.prog}: error: {message}\n")


def generate_values(n: int, density: float, seed: int, dc: float = 0.0) -> np.ndarray:
    """2^n uint8 values (0 off, 1 on, 2 dc) from the frozen generator, built on the GPU."""
    if not 1 <= n <= 31:
        raise ValueError(f"n must be in 1..31, got {n}")
    if not 0.0 <= density <= 1.0 or not 0.0 <= dc <= 1.0 - density + 1e-12:
        raise ValueError("density and dc must be probabilities with density + dc <= 1")
    out = np.empty(1 << n, dtype=np.uint8)
    _lib.check(_lib.load().dqmc_gen3_host(out.ctypes.data, n, float(density), float(dc), int(seed)))
    return out


def read_bits(text: str) -> TruthTable:
    """The reference's 'bits' format (ttio.py:1-20): n from the length."""
    bits = "".join(text.split())
    if not bits or any(c not in "01" for c in bits):
        raise errors.ParseError("bits format expects only '0'/'1' characters")
    n = len(bits).bit_length() - 1
    if len(bits) != 1 << n or n < 1:
        raise errors.ParseError(f"bits format needs 2^n characters, got {len(bits)}")
    return TruthTable.from_bools(n, np.frombuffer(bits.encode(), dtype=np.uint8) == ord("1"))


def order_for_listing(ranks: np.ndarray, n: int) -> np.ndarray:
    """Wildcard count descending, rank ascending (cli.py:133-135), on the GPU."""
    r = np.ascontiguousarray(ranks, dtype=np.int64)
    out = np.empty_like(r)
    _lib.check(_lib.load().dqmc_order_by_weight(r.ctypes.data, len(r), n, out.ctypes.data))
    return out


def _state_engine(tt: TruthTable, h: int | None) -> np.ndarray:
    from .state import extract_ranks, load

    st = load(tt, h=h, mirror=False)
    st.run_merge_reduce()
    return extract_ranks(st)


def _input(args):
    """(n, truth table or None, values or None)."""
    if args.input:
        with open(args.input) if args.input != "-" else sys.stdin as fh:
            tt = read_bits(fh.read())
        return tt.n, tt, None
    if args.config is not None:
        from .configs import CONFIGS, config_values_host

        v = config_values_host(args.config, args.n)
        return (args.n or CONFIGS[args.config]["n"]), None, v
    if args.n is None or args.density is None:
        raise errors.ParseError("provide --input PATH, --config K, or both --n and --density to generate")
    v = generate_values(args.n, args.density, args.seed, args.dc)
    return args.n, None, v


def _run(engine: str, n: int, tt, values, args) -> np.ndarray:
    if engine == "dense":
        if tt is not None:
            return dense_prime_ranks(tt, h=args.h, optimized=args.unroll == "on", mem_cap=args.mem_cap)
        return prime_ranks_from_values(values, h=args.h, mem_cap=args.mem_cap)
    if engine == "sparse":
        if tt is None:
            tt = TruthTable.from_values(n, values)
        return sparse_prime_ranks(tt, mem_cap=args.mem_cap)
    if engine == "state":
        if tt is None:
            tt = TruthTable.from_values(n, values)
        return _state_engine(tt, args.h)
    raise ValueError(f"unknown engine {engine!r}; expected one of {', '.join(ENGINES)}")


def _cmd_primes(args) -> int:
    n, tt, v = _input(args)
    ranks = _run(args.algo, n, tt, v, args)
    if args.count_only:
        sys.stdout.write(f"{len(ranks)}\n")
        return 0
    text = ranks_to_text(order_for_listing(ranks, n), n, wildcard=args.wildcard_char)
    if args.output and args.output != "-":
        with open(args.output, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _cmd_verify(args) -> int:
    n, tt, v = _input(args)
    algos = [a.strip() for a in args.algo.split(",")]
    results = {}
    for a in algos:
        r = _run(a, n, tt, v, args)
        if os.environ.get(_CORRUPT_ENV) == a and len(r):
            r = r[1:]
        results[a] = r
    base = results[algos[0]]
    bad = [a for a in algos[1:] if not np.array_equal(results[a], base)]
    if bad:
        for a in bad:
            d1 = np.setdiff1d(base, results[a])[:5]
            d2 = np.setdiff1d(results[a], base)[:5]
            sys.stderr.write(f"MISMATCH {algos[0]} vs {a}: only-{algos[0]} {d1.tolist()} only-{a} {d2.tolist()}\n")
        return 3
    sys.stdout.write(f"OK {len(base)} primes agree across {', '.join(algos)}\n")
    return 0


def _sweep(text: str) -> list[int]:
    out = []
    for part in text.split(","):
        if ".." in part:
            a, _, b = part.partition("..")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def _cmd_bench(args) -> int:
    lines = []
    for n in _sweep(args.n_sweep):
        for d in [float(x) for x in args.densities.split(",")]:
            v = generate_values(n, d, args.seed, args.dc)
            best, cnt, err = float("inf"), -1, None
            for _ in range(max(1, args.reps)):
                try:
                    t0 = time.perf_counter()
                    r = _run(args.algo, n, None, v, args)
                    best = min(best, time.perf_counter() - t0)
                    cnt = len(r)
                except errors.ResourceLimitError as exc:
                    err = str(exc)
                    break
            rep = {"engine": args.algo, "n": n, "density": d, "seed": args.seed,
                   "seconds": 0.0 if err else best, "peak_bytes": int(_lib.load().dqmc_device_bytes(n)),
                   "prime_count": cnt}
            if err:
                rep["error"] = err
            lines.append(json.dumps(rep))
    text = "\n".join(lines) + "\n"
    if args.output and args.output != "-":
        with open(args.output, "a", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _add_common(p):
    g = p.add_argument_group("input (file or generated)")
    g.add_argument("--input", "-i", metavar="PATH", help="truth table in 'bits' format, '-' for stdin")
    g.add_argument("--n", type=int, help="variable count (generated input)")
    g.add_argument("--density", type=float, help="P(on) for generated input")
    g.add_argument("--dc", type=float, default=0.0, help="P(don't care) for generated input (counted as on)")
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--config", type=int, choices=(1, 2, 3, 4, 5), help="BASELINE.json workload (--n overrides its size)")
    e = p.add_argument_group("engine")
    e.add_argument("--h", type=int, help="dense split, validated as the reference (result independent of it)")
    e.add_argument("--unroll", choices=("on", "off"), default="on")
    e.add_argument("--mem-cap", type=int, metavar="BYTES")


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="python -m paper_2302_10083_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    p = sub.add_parser("primes", help="list all prime implicants")
    _add_common(p)
    p.add_argument("--algo", choices=ENGINES, default="dense")
    p.add_argument("--wildcard-char", choices=("*", "-"), default="*")
    p.add_argument("--output", "-o")
    p.add_argument("--count-only", action="store_true", help="print only the number of primes")
    p.set_defaults(func=_cmd_primes)
    p = sub.add_parser("verify", help="compare engines on one input")
    _add_common(p)
    p.add_argument("--algo", default="dense,sparse", help="comma list of engines (dense, sparse, state)")
    p.set_defaults(func=_cmd_verify)
    p = sub.add_parser("bench", help="time the engine over generated inputs (JSONL)")
    p.add_argument("--n", dest="n_sweep", required=True, help="e.g. 16..22 or 20,24")
    p.add_argument("--densities", default="0.5")
    p.add_argument("--dc", type=float, default=0.0)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--algo", choices=ENGINES, default="dense")
    p.add_argument("--h", type=int)
    p.add_argument("--unroll", choices=("on", "off"), default="on")
    p.add_argument("--mem-cap", type=int)
    p.add_argument("--output", "-o")
    p.set_defaults(func=_cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except errors.ResourceLimitError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 2
    except (errors.ParseError, ValueError, OSError) as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 1


if __name__ == "__main__":  # pragma: no cover
    sys.exit(main())
