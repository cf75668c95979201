import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: larger parity cases")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "gpu" in item.keywords and "timeout" not in item.keywords:
            item.add_marker(pytest.mark.timeout(900))
