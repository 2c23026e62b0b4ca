import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
EPS = 2.220446049250313e-16


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def unhex(lst) -> np.ndarray:
    return np.array([float.fromhex(s) for s in lst])


@pytest.fixture(scope="session")
def ref_vectors():
    with open(os.path.join(GOLDEN, "ref_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def nodes_truth():
    with open(os.path.join(GOLDEN, "nodes_truth.json")) as f:
        return json.load(f)
