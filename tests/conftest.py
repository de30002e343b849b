import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libwfk.so)")
    config.addinivalue_line("markers", "slow: longer CPU case")


def pytest_collection_modifyitems(config, items):
    # a GPU test on a box without CUDA is a setup error, not a skip: the driver
    # runs -m gpu only on a B200
    pass
