import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _cuda_devices():
    try:
        from paper_2605_16684_b200 import capi
        return capi.lib().esdg_b200_device_count()
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    # `-m gpu` on a box without a GPU must fail loudly, not silently pass:
    # only plain collection without -m gpu skips them.
    if "gpu" in (config.getoption("-m") or ""):
        return
    if _cuda_devices() == 0:
        skip = pytest.mark.skip(reason="no CUDA device")
        for item in items:
            if "gpu" in item.keywords:
                item.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle as po
    return po.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle as po
    if not po.reference_available():
        pytest.skip("oracle/_ref/libesdg_ref.so not built (reference tree absent)")
    return po.Oracle("reference")
