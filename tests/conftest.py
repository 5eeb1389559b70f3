import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libpipefill.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")
    config.addinivalue_line("markers", "gpu_timing: timing-dependent GPU test (runs after all parity tests)")


def pytest_collection_modifyitems(session, config, items):
    """Parity tests first, timing-dependent ones last: under `-x` a timing test that trips on
    a fresh box must not hide the kernel and executor parity tests behind it."""
    items.sort(key=lambda it: 1 if it.get_closest_marker("gpu_timing") else 0)
