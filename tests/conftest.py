import os
import sys

import pytest

# The quick sort hands arrays / segments of up to 2^19 keys to the merge layer
# (its base case, quicksort.cu qs_base_max).  The tests lower that to one tile
# so that every partition path also runs at test sizes; the default policy is
# checked by tests/test_gpu_quicksort.py::test_quick_sort_default_base_case
# (a child process without this variable), the bench and smoke().
os.environ.setdefault("NSB_QS_BASE_MAX", "16384")

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
