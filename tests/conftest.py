"""Shared fixtures.  `-m gpu` tests need a CUDA device (a B200); everything
else runs on CPU.  The oracles (tests/oracle_bindings.py) are test-only."""
import json
import os
import sys

import pytest

TESTS = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(TESTS)
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: minutes of CPU or GPU time")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle_bindings import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("compiled reference oracle/_ref missing")
    return RefLib()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(TESTS, "golden", "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def egs():
    import paper_1710_03647_b200 as egs
    return egs
