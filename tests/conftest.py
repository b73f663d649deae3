import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


# the reference's own tests run against the drop-in only through
# tests/test_gpu_reference_suite.py (a GPU subprocess)
collect_ignore = ["reference_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the CUDA library")


@pytest.fixture(scope="session")
def oracle():
    from tests.oracle_bind import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test on a machine without a GPU")
    return torch.device("cuda", 0)
