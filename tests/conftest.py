import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--bfla-variant", default="",
                     help="run the GPU tests against libbfla_<variant>.so (an A/B or debug build) instead of libbfla.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    variant = config.getoption("--bfla-variant")
    if variant:
        from paper_2605_12193_b200 import _lib

        _lib.use_variant(variant)


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle
