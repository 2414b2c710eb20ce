import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_fixtures():
    import json
    with open(os.path.join(GOLDEN, "reference_fixtures.json")) as f:
        return json.load(f)["fixtures"]


@pytest.fixture(scope="session")
def ref_vectors():
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, "ref_vectors.npz")))


@pytest.fixture(scope="session")
def verify_vectors():
    import json
    with open(os.path.join(GOLDEN, "verify_vectors.json")) as f:
        return json.load(f)
