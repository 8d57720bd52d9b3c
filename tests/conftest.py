import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large (App. B full-size) oracle pins")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "appendix_b.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle_hashes():
    import json
    p = os.path.join(ROOT, "tests", "golden", "oracle_hashes.json")
    with open(p) as f:
        return json.load(f)
