import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ns():
    """The product package with its sm_100a library loaded (built if absent)."""
    import paper_2503_05934_b200 as ns
    from paper_2503_05934_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    ns.lib()
    return ns


@pytest.fixture(scope="session")
def cuda(ns):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a host without CUDA")
    return torch.device("cuda:0")
