import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _have_gpu() -> bool:
    import paper_2406_06911_b200 as adx
    return adx.lib().adx_device_count() > 0


def pytest_collection_modifyitems(config, items):
    gpu_items = [it for it in items if "gpu" in it.keywords]
    if not gpu_items:
        return
    try:
        ok = _have_gpu()
    except ImportError as exc:  # library not built: fail loudly, never fall back
        raise pytest.UsageError(str(exc))
    if not ok:
        skip = pytest.mark.skip(reason="no CUDA device visible")
        for it in gpu_items:
            it.add_marker(skip)
