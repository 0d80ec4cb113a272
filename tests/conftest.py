import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")
    # Test infrastructure: make sure the in-tree library is built (nvcc cross-compiles without a
    # GPU) and up to date before any test loads it. The product binding itself never builds:
    # it raises if libdvstream.so is missing.
    from paper_2403_01876_b200 import build
    build.build()
    build.build_fast()
    build.build_c_smoke()


def pytest_collection_modifyitems(config, items):
    # GPU tests never silently pass without a device: they fail loudly if selected without one.
    pass


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """After every GPU test, hand the caching allocator's blocks back to the driver: the full-size
    tests hold tens of GB, and the multi-process tests that follow (2 ranks x 77 GB of C5 stage
    caches) need the device's memory, not this process's cache."""
    yield
    if request.node.get_closest_marker("gpu") is not None:
        import gc

        import torch
        if torch.cuda.is_available():
            gc.collect()
            torch.cuda.synchronize()
            torch.cuda.empty_cache()


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture
def golden():
    import json

    def load(name):
        with open(os.path.join(GOLDEN, name)) as f:
            return json.load(f)
    return load
