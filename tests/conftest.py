import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liboffsim_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if any(item.get_closest_marker("gpu") for item in items) and not _cuda_available():
        skip = pytest.mark.skip(reason="no CUDA device in this container")
        for item in items:
            if item.get_closest_marker("gpu"):
                item.add_marker(skip)
