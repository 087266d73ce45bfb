import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a extension)")
    config.addinivalue_line("markers", "slow: larger parity sweeps")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "cases.json")) as f:
        manifest = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden_v1.npz")))
    return manifest, arrays


@pytest.fixture(scope="session")
def native_lib():
    from paper_2602_04936_b200 import _build, _native

    if _build.needs_build():
        _build.build_native()
    return _native.load()


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_04936_b200 import _build

    if _build.needs_build():
        _build.build_native()
    return torch.device("cuda:0")
