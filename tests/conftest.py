"""Shared pytest setup. `-m gpu` tests need a B200 and call the CUDA operator through the
C ABI (libfdmoe.so); everything else runs on CPU (oracle pinning, host logic, ABI surface)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running CPU reference comparisons")
