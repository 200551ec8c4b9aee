import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # compile libnnqs.so (nvcc cross-compiles without a GPU) before any test module
    # imports the package; the package itself refuses to import without it
    import __graft_entry__
    __graft_entry__.build()
