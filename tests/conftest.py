import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgebq_b200.so")
    config.addinivalue_line("markers", "slow: long-running (full 2^32 sweeps on CPU)")


@pytest.fixture(scope="session")
def fixtures():
    with gzip.open(os.path.join(GOLDEN, "fixtures.json.gz"), "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kernel_arrays():
    return dict(np.load(os.path.join(GOLDEN, "kernels.npz")))


@pytest.fixture(scope="session")
def fuzz_arrays():
    return dict(np.load(os.path.join(GOLDEN, "decode_fuzz.npz")))


@pytest.fixture(scope="session")
def golden_record():
    with open(os.path.join(GOLDEN, "golden_record.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sweeps_fixture():
    with open(os.path.join(GOLDEN, "sweeps.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_15037_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


def pytest_sessionstart(session):
    """Refuse to test a stale CUDA library (sources newer than the built .so)."""
    try:
        from paper_2407_15037_b200 import _build
    except Exception:  # pragma: no cover
        return
    import os

    if os.path.exists(_build.LIB) and not _build.up_to_date():
        raise RuntimeError("libgebq_b200.so is older than its sources: run "
                           "`python -m paper_2407_15037_b200._build` first")
