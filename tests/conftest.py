import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu():
    try:
        import paper_2402_17993_b200 as ff

        return ff.Device.count() > 0
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly on a GPU box; here (no device) they are skipped only
    # when explicitly deselected by -m "not gpu".
    pass


@pytest.fixture(scope="session")
def oracle():
    from oracle import ffo

    ffo.lib()
    return ffo
