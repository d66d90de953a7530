import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# The GPU tests run up to 8 ranks as threads on ONE device, each with its own stream and side
# stream.  With CUDA's default 8 hardware work queues, streams share queues, and work queued
# behind another rank's spinning peer-exchange kernel cannot start (a false dependency that
# deadlocks the exchange: fastusp.h, peer-memory transport).  One queue per stream; must be set
# before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def fu():
    """The product package; building it if the in-tree library is missing."""
    import paper_2602_10940_b200 as fu
    fu.build()
    return fu
