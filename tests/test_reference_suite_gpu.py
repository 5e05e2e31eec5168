"""the reference's own dense-path tests, unmodified, against
the device DenseState and engine (tests/refsuite/refsuite_plugin.py binds
implicants.dense to this package before they are imported).

Runs /root/reference/pkg/tests/test_dense.py (all of it: triples, layout,
passes, end-to-end; :41-249) and test_acceptance.py criteria 1-4 and 7
(:56-159, :209-225) from the copy tools/stage_reference.sh stages in
baseline/_ref. Criteria 5/6 are CPU wall-clock/RSS envelopes of the reference
and 8 is text-format I/O: not this path. Skips when the reference has not
been staged.
"""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")


def _run(files, kexpr=None):
    if not os.path.isdir(os.path.join(REF, "tests")) or not os.path.isdir(os.path.join(REF, "implicants")):
        pytest.skip("reference not staged in baseline/_ref (tools/stage_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "tests", "refsuite"), REPO, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-p", "no:cacheprovider", "-q", "-rA",
           "--rootdir", REF, "-c", os.path.join(REF, "pyproject.toml"), *[os.path.join(REF, "tests", f) for f in files]]
    if kexpr:
        cmd += ["-k", kexpr]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    return r


@pytest.mark.gpu
def test_reference_test_dense_on_device():
    r = _run(["test_dense.py"])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "device engine bound: implicants.dense.load -> paper_2302_10083_b200.state.load" in r.stdout
    assert " failed" not in r.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
def test_reference_acceptance_on_device():
    r = _run(["test_acceptance.py"], "criterion_1 or criterion_2 or criterion_3 or criterion_4 or criterion_7")
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "device engine bound: implicants.dense.dense_prime_ranks" in r.stdout
    last = r.stdout.strip().splitlines()[-1]
    assert "5 passed" in last, last
