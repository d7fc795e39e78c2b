import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# tests/_ref_suite holds the reference's own test files (tools/ref_suite.py);
# they run through tests/test_ref_suite.py in a child, never collected directly
collect_ignore_glob = [] if os.environ.get("QADIC_REF_SUITE") == "1" else ["_ref_suite/*"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size parity runs")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def golden_scalars():
    with open(os.path.join(GOLDEN, "golden_scalars.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_fdiv_scans():
    """Reports of the reference's own exhaustive FDIV scans (make_fdiv_scans.py)."""
    with open(os.path.join(GOLDEN, "fdiv_scans.json")) as fh:
        return json.load(fh)


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))
