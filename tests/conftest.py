import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running oracle check")


def pytest_sessionstart(session):
    # build the CUDA library (nvcc cross-compiles without a GPU) before any test
    # imports the binding; load build.py by path (the package needs the .so)
    import importlib.util
    spec = importlib.util.spec_from_file_location("gicp_build", os.path.join(ROOT, "paper_2308_07173_b200",
                                                                             "build.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.build()


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
