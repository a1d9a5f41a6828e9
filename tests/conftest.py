import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    return load


# parity metrics recorded by the GPU tests (first L-trace divergence, max |dx|, trace-column errors,
# gradient-check margins); written as JSON when FOE_PARITY_REPORT names a path (profiles/ keeps the
# committed copy of a driver-style run)
_REPORT: dict = {}


@pytest.fixture(scope="session")
def parity_report():
    return _REPORT


def pytest_sessionfinish(session, exitstatus):
    import json
    path = os.environ.get("FOE_PARITY_REPORT")
    if path and _REPORT:
        with open(path, "w") as fh:
            json.dump(_REPORT, fh, indent=1, sort_keys=True, default=float)
