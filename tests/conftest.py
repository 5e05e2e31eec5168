"""Shared fixtures. GPU tests are marked @pytest.mark.gpu."""

import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(REPO, "tests", "golden", "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def gen_mod():
    from oracle import gen as G

    return G


@pytest.fixture(scope="session")
def pkg():
    import paper_2302_10083_b200 as P

    return P


@pytest.fixture(autouse=True)
def _release_after_large_tests(request):
    """The engine caches its device workspace between calls (state, scratch:
    111 GB after the n=25 test). Large tests hand it back, so the tests after
    them (and the processes the multi-process tests spawn) start with the
    GPU's memory free."""
    yield
    if request.node.get_closest_marker("slow") is None and request.node.get_closest_marker("gpu") is None:
        return
    if "paper_2302_10083_b200._lib" not in sys.modules:
        return
    try:
        import torch

        from paper_2302_10083_b200 import _lib

        _lib.load().dqmc_release()  # cheap: buffers come back on the next call
        torch.cuda.empty_cache()
    except Exception:  # pragma: no cover - no GPU / library not built
        pass
