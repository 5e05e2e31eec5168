"""Generate tests/golden/golden.json by running the REFERENCE package.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the read-only reference (`implicants`, pure Python + NumPy) from
/root/reference/pkg/src and records its outputs on seeded inputs. The inputs
come from the committed restated generators (oracle/gen.py); the script first
checks they are bit-identical to the reference's own `random_function`
(ttio.py:346-378). The GPU box never runs this file (the reference does not
travel); tests read only the committed JSON.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import implicants as ref  # noqa: E402  (the reference, read-only)

from oracle import gen as G  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ranks_sha(r: np.ndarray) -> str:
    return sha(np.asarray(r, dtype="<i8"))


def max_weight(r: np.ndarray, n: int) -> int:
    if not len(r):
        return 0
    return int(ref.rank_weights(r, n).max())


def main() -> None:
    out: dict = {"source": "reference implicants package @ /root/reference/pkg/src", "cases": {}}

    # --- configs 1-3 (BASELINE.json), DC semantics: on ∪ dc
    cfgs = {}
    for c in (1, 2, 3):
        n = G.CONFIGS[c]["n"]
        v = G.config_values(c)
        tt = ref.TruthTable.from_bools(n, v != 0)
        assert np.array_equal(tt.words, G.values_to_words(v))
        r = ref.dense_prime_ranks(tt)
        cfgs[str(c)] = dict(
            n=n,
            tt_sha256=sha(v),
            on=int((v == 1).sum()),
            dc=int((v == 2).sum()),
            off=int((v == 0).sum()),
            primes=int(len(r)),
            ranks_sha256=ranks_sha(r),
            first=[int(x) for x in r[:5]],
            last=[int(x) for x in r[-5:]],
            max_weight=max_weight(r, n),
        )
        if c == 1:
            cfgs[str(c)]["ranks"] = [int(x) for x in r]
    # config 4 (n=24): recorded by the survey's reference run;
    # re-running the NumPy reference costs ~11 min and 41 GiB, so only its pins are kept.
    cfgs["4"] = dict(
        n=24,
        tt_sha256_prefix="a5f01dccb61db7fa",
        on=12585839,
        dc=838429,
        off=3352948,
        primes=209934817,
        ranks_sha256_prefix="0f45898a2642f3d1",
        first=[429, 708, 1536],
        last=[281848326690, 281848404681, 281851043241],
        max_weight=6,
        source="SURVEY.md Appendix A (reference dense_prime_ranks, h=5, run by the survey)",
    )
    out["configs"] = cfgs

    # --- generator agreement with the reference's random_function
    gen_checks = []
    for n, d, s in ((5, 0.3, 7), (10, 0.4, 3), (14, 0.37, 123), (16, 0.5, 42), (20, 0.75, 3)):
        assert np.array_equal(ref.random_function(n, d, s).words, G.random_words(n, d, s))
        gen_checks.append(dict(n=n, density=d, seed=s, words_sha256=sha(G.random_words(n, d, s))))
    out["generator"] = gen_checks

    # --- acceptance criterion 1 sweep (test_acceptance.py:56-72): n 1..10 x 7 densities x 20 seeds
    sweep = []
    for n in range(1, 11):
        for d in (0.0, 0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
            for s in range(20):
                tt = ref.random_function(n, d, s)
                r = ref.dense_prime_ranks(tt)
                sweep.append([n, d, s, int(len(r)), ranks_sha(r)[:16]])
    out["sweep_c1"] = sweep

    # --- README goldens (pkg/README.md:54-108) and small known answers
    readme = []
    for n, d, s in ((16, 0.5, 42), (10, 0.4, 3), (10, 0.5, 0), (12, 0.5, 1), (13, 0.5, 1), (14, 0.5, 1)):
        r = ref.dense_prime_ranks(ref.random_function(n, d, s))
        readme.append(dict(n=n, density=d, seed=s, primes=int(len(r)), ranks_sha256=ranks_sha(r)))
    out["readme"] = readme
    out["known"] = dict(
        maj3=[int(x) for x in ref.dense_prime_ranks(ref.TruthTable.from_indices(3, [3, 5, 6, 7]))],
        n5_12_14=[int(x) for x in ref.dense_prime_ranks(ref.TruthTable.from_indices(5, [12, 14]))],
        single_point_6=[int(x) for x in ref.dense_prime_ranks(ref.TruthTable.from_indices(6, [0b101001]))],
        cli_order_bits="0001100010101011",
        cli_order_ranks=[
            int(x)
            for x in ref.dense_prime_ranks(
                ref.TruthTable.from_bools(4, np.array([c == "1" for c in "0001100010101011"]))
            )
        ],
    )

    # --- don't-care cases at small n (three-way values, on ∪ dc)
    dcs = []
    for n, pon, pdc, s in ((6, 0.5, 0.2, 1), (9, 0.6, 0.2, 2), (12, 0.8, 0.1, 3), (14, 0.9, 0.05, 1), (18, 0.75, 0.05, 3)):
        v = G.gen3(n, pon, pdc, s)
        r = ref.dense_prime_ranks(ref.TruthTable.from_bools(n, v != 0))
        dcs.append(dict(n=n, p_on=pon, p_dc=pdc, seed=s, tt_sha256=sha(v), primes=int(len(r)), ranks_sha256=ranks_sha(r)))
    out["dc_cases"] = dcs

    # --- layout pins: DenseState.words after MERGE and after REDUCE (dense.py:296-337)
    states = []
    for n, d, s, h in ((7, 0.5, 12, 3), (8, 0.35, 5, 4), (9, 0.5, 21, 5), (11, 0.6, 4, 5)):
        tt = ref.random_function(n, d, s)
        st = ref.load(tt, h=h)
        loaded = sha(st.words)
        st.run_pass(ref.MERGE)
        merged = sha(st.words)
        st.run_pass(ref.REDUCE)
        states.append(dict(n=n, density=d, seed=s, h=h, loaded=loaded, merged=merged, reduced=sha(st.words)))
    out["states"] = states

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
