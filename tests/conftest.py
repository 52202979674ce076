import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run on the GPU box")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    out = {}
    for name in ("hashes", "runs", "traces"):
        with open(os.path.join(d, name + ".json")) as f:
            out[name] = json.load(f)
    return out


@pytest.fixture(scope="session")
def ctx():
    import paper_2410_14047_b200 as D
    return D.Context(0)


@pytest.fixture(scope="session")
def golden_fasst():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "fasst_stats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_influence():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "influence.json")) as f:
        return json.load(f)
