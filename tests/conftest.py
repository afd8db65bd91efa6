import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running statistical test")


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Reference

    if not Reference.available:
        pytest.skip("oracle/_ref/libescg_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def escg():
    import paper_2508_16639_b200 as e

    return e
