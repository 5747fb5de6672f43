import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def golden_small():
    import json

    import numpy as np
    with open(os.path.join(GOLDEN, "small_cases.json")) as f:
        manifest = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, "small_cases.npz")))
    return manifest["cases"], arrays


def load_digests(cfg):
    import json
    path = os.path.join(GOLDEN, f"digests_{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_lf5():
    import json
    with open(os.path.join(GOLDEN, "small_cases.json")) as f:
        return json.load(f)["lf5"]
