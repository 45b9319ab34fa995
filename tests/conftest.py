import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# Co-located ranks on one GPU (tests/test_gpu_colocated.py): one hardware queue
# per CUDA stream, so a rank's spinning flag barrier never blocks another rank's
# producer kernel queued behind it. Read when the CUDA context is created, i.e.
# before any test touches the GPU.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")
