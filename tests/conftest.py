import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2410_00425_b200 import _native

    _native.ensure_device()
    return torch.device("cuda", torch.cuda.current_device())


@pytest.fixture(scope="session")
def pose_golden():
    import numpy as np

    return dict(np.load(os.path.join(ROOT, "tests", "golden", "pose_golden.npz")))
