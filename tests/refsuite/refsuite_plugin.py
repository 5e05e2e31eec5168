"""pytest plugin: the reference's OWN test files run against this engine.

Loaded with ``-p refsuite_plugin`` (tests/refsuite on PYTHONPATH) in a subprocess whose rootdir is
baseline/_ref (the reference package installed there by
tools/stage_reference.sh, with its tests/ directory staged beside it; nothing
of the reference is committed to this repository). Before the reference's
test modules are imported, the reference package's dense path
(implicants.dense: load, DenseState, extract_ranks, extract_strings,
dense_prime_ranks, find_primes_dense — dense.py:127-428) is rebound to the
device implementation (paper_2302_10083_b200.state / .dense), and our errors
adopt the reference's exception classes. The sparse and oracle engines stay
the reference's own, so acceptance criterion 1 (dense = sparse = oracle)
compares our GPU engine against two independent CPU constructions.
"""

import os
import sys
import types

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(REPO, "baseline", "_ref")

sys.path.insert(0, REF)
if REPO not in sys.path:
    sys.path.insert(1, REPO)

import implicants  # noqa: E402  (the reference, from baseline/_ref)
import implicants.bench  # noqa: E402
import implicants.dense  # noqa: E402

from paper_2302_10083_b200 import dense as _dense  # noqa: E402
from paper_2302_10083_b200 import errors as _errors  # noqa: E402
from paper_2302_10083_b200 import state as _state  # noqa: E402

_errors.adopt(implicants.errors)

DEVICE_API = {
    "load": _state.load,
    "DenseState": _state.DenseState,
    "extract_ranks": _state.extract_ranks,
    "extract_strings": _state.extract_strings,
    "dense_prime_ranks": _dense.dense_prime_ranks,
    "find_primes_dense": _dense.find_primes_dense,
}
for _name, _obj in DEVICE_API.items():
    for _mod in (implicants, implicants.dense, implicants.bench):
        if hasattr(_mod, _name):
            setattr(_mod, _name, _obj)

# the reference's tests import their helpers as `tests.conftest`
_tests = types.ModuleType("tests")
_tests.__path__ = [os.path.join(REF, "tests")]
sys.modules["tests"] = _tests


def pytest_terminal_summary(terminalreporter):
    for n, o in DEVICE_API.items():
        bound = getattr(implicants.dense, n)
        terminalreporter.write_line(f"device engine bound: implicants.dense.{n} -> {bound.__module__}.{bound.__qualname__}")
