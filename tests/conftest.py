import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_1703_06065_b200 import bcur
    return bcur.default_context()

from impls import impl  # noqa: E402,F401  (parametrized oracle / gpu fixture)
