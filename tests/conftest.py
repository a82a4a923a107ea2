import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle
    from oracle import build as obuild
    obuild.build_oracle()
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle
    from oracle import build as obuild
    obuild.build_ref()
    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt .so)")
    return pyoracle.Oracle("reference")
