import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) when selected without a GPU: the driver runs
    # `-m gpu` only on a B200 box.
    pass


@pytest.fixture(autouse=True)
def _release_device_memory():
    """GPU tests build engines with arenas of tens of GB: after each test, return what torch's caching
    allocator still holds to the device, so later tests (and the spawned tensor-parallel ranks) see it."""
    yield
    if "torch" in sys.modules:
        import gc
        torch = sys.modules["torch"]
        gc.collect()
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.empty_cache()
